"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel family of the library on an emulated world (p ranks on cuda:0, one
cooperative launch per collective), small sizes, every output checked
against the oracle. Run one tool per process:

    compute-sanitizer --tool memcheck --error-exitcode 99 python tools/sanitize.py --p 4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--ctas", type=int, default=8)
    a = ap.parse_args()
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200.communicator import emulated_world

    p = a.p
    w = emulated_world(p, 0)
    w.set_param("ctas", a.ctas)
    w.set_timeout_ms(600_000)  # instrumented kernels are slow
    rng = np.random.default_rng(0)
    bad = []
    ran = 0

    def eq(name, got, want):
        nonlocal ran
        ran += 1
        g, wv = np.ascontiguousarray(got), np.ascontiguousarray(want)
        if g.shape != wv.shape or not np.array_equal(g.view(np.uint8), wv.view(np.uint8)):
            bad.append(name)

    pow2 = p & (p - 1) == 0
    algos = ["direct", "ring"] + (["recursive"] if pow2 else [])
    for n in (5, 4096 + 8, 70000):  # LL (direct, small), flag protocol, multi-unit slices
        ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
        want_ag = oracle.ring_all_gather(ag_in)
        for algo in algos:
            outs = pkg.run_ranks(p, lambda c: pkg.all_gather(c, ag_in[c.rank], algorithm=algo))
            for r in range(p):
                eq(f"ag_{algo}_{n}_{r}", outs[r], want_ag[r])
            order = "recursive" if algo == "recursive" else "ring"
            want = (oracle.rechalf_reduce_scatter(rs_in) if algo == "recursive" else oracle.ring_reduce_scatter(rs_in))
            outs = pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, rs_in[c.rank], algorithm=algo, order=order))
            for r in range(p):
                eq(f"rs_{algo}_{n}_{r}", outs[r], want[r])
        # bf16 device tensors
        bf = [oracle.f32_to_bf16(x) for x in rs_in]
        for algo in algos:
            fn = {"ring": oracle.ring_reduce_scatter, "recursive": oracle.rechalf_reduce_scatter,
                  "direct": lambda xs, d: oracle.direct_reduce_scatter(xs, d, order="ring")}[algo]
            want = fn(bf, "bf16")
            outs = pkg.run_ranks(p, lambda c: pkg.reduce_scatter(
                c, torch.from_numpy(bf[c.rank].view(np.int16)).view(torch.bfloat16).cuda(), algorithm=algo)
                .view(torch.int16).cpu().numpy().view(np.uint16))
            for r in range(p):
                eq(f"rs_bf16_{algo}_{n}_{r}", outs[r], want[r])
        # hierarchical
        for N in [g for g in (2, 4) if p % g == 0 and 1 < g < p]:
            for inter in ["ring"] + (["recursive"] if N & (N - 1) == 0 else []):
                plan = pkg.HierPlan(topo=pkg.Topology(N, p // N), inter_alg=inter)
                outs = pkg.run_ranks(p, lambda c: pkg.hier_all_gather(plan, c, ag_in[c.rank]))
                want = oracle.hier_all_gather(ag_in, N, p // N, inter)
                for r in range(p):
                    eq(f"hier_ag_{N}_{inter}_{n}_{r}", outs[r], want[r])
                outs = pkg.run_ranks(p, lambda c: pkg.hier_reduce_scatter(plan, c, rs_in[c.rank]))
                want = oracle.hier_reduce_scatter(rs_in, N, p // N, inter)
                for r in range(p):
                    eq(f"hier_rs_{N}_{inter}_{n}_{r}", outs[r], want[r])
    # push / pull data-movement variants of the flag protocol
    n = 4096 + 8
    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    w.set_param("ll_max", 0)
    for v in (0, 1, 2, 3):
        w.set_param("ag_variant", v)
        for algo in algos:
            if v >= 2 and algo != "direct":
                continue
            outs = pkg.run_ranks(p, lambda c: pkg.all_gather(c, ag_in[c.rank], algorithm=algo))
            for r in range(p):
                eq(f"agv{v}_{algo}_{r}", outs[r], oracle.ring_all_gather(ag_in)[r])
    w.set_param("ag_variant", -1)
    for v in (0, 1, 5):
        w.set_param("rs_variant", v)
        for algo in algos:
            if v == 5 and algo != "direct":
                continue
            order = "recursive" if algo == "recursive" else "ring"
            want = (oracle.rechalf_reduce_scatter(rs_in) if algo == "recursive" else oracle.ring_reduce_scatter(rs_in))
            outs = pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, rs_in[c.rank], algorithm=algo, order=order))
            for r in range(p):
                eq(f"rsv{v}_{algo}_{r}", outs[r], want[r])
    w.set_param("rs_variant", -1)
    w.set_param("ll_max", -1)
    # shuffles and the standalone add
    x = rng.standard_normal(2 * 2 * 33).astype(np.float32)
    eq("shuffle_l2g", pkg.shuffle_local_major_to_global(x, 2, 2, 33), oracle.shuffle_local_major_to_global(x, 2, 2, 33))
    eq("shuffle_g2l", pkg.shuffle_global_to_local_major(x, 2, 2, 33), oracle.shuffle_global_to_local_major(x, 2, 2, 33))
    acc = rng.standard_normal(1001).astype(np.float32)
    oth = rng.standard_normal(1001).astype(np.float32)
    eq("reduce_inplace", pkg.reduce_inplace(acc.copy(), oth), np.add(acc, oth, dtype=np.float32))
    torch.cuda.synchronize()
    w.check()
    print(f"SANITIZE WORKLOAD {'OK' if not bad else 'FAIL ' + ','.join(bad[:10])}: {ran} checks, p={p}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
