"""Real-mode parity worker: one process per GPU (launched by torchrun from
tests/test_gpu_multiproc.py). Every rank builds the same seeded inputs for all
ranks, runs each collective through the public API over CUDA-IPC peer memory,
and checks its own output bit-for-bit against the oracle (test
infrastructure). Exit code 0 = all checks passed on this rank."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402


def main() -> int:
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # one process per GPU, never more ranks than devices (ranks spinning on
    # each other's flags from one GPU can deadlock the device)
    if local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: local rank {local} >= {torch.cuda.device_count()} visible GPUs")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2504_18658_b200 as pkg

    comm = pkg.init_from_torch()
    p = world
    failures = []

    def sync_point(name):
        # device errors are sticky and async: surface them per section, and
        # verify every rank completed the same number of collectives
        torch.cuda.synchronize()
        try:
            comm.world.check()
        except Exception as exc:  # noqa: BLE001
            failures.append(f"{name}:{type(exc).__name__}")
            raise
        eps = [None] * p
        dist.all_gather_object(eps, comm.epoch())
        if len(set(eps)) != 1:
            failures.append(f"{name}:epochs{eps}")
            raise RuntimeError(f"epoch divergence after {name}: {eps}")

    def check(name, got, want):
        g = np.ascontiguousarray(got)
        w = np.ascontiguousarray(want)
        if g.shape != w.shape or not np.array_equal(g.view(np.uint8), w.view(np.uint8)):
            failures.append(name)

    rng = np.random.default_rng(1234)
    pow2 = p & (p - 1) == 0
    for n in (1, 37, 4096, 300_000):
        ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
        want_ag = oracle.ring_all_gather(ag_in)[rank]
        algos = [("ring", pkg.ring_all_gather), ("direct", pkg.direct_all_gather)]
        if pow2:
            algos.append(("recursive", pkg.recdbl_all_gather))
        for name, fn in algos:
            check(f"ag_{name}_n{n}", fn(comm, ag_in[rank]), want_ag)
        check(f"rs_ring_n{n}", pkg.ring_reduce_scatter(comm, rs_in[rank]), oracle.ring_reduce_scatter(rs_in)[rank])
        check(f"rs_direct_ring_n{n}", pkg.direct_reduce_scatter(comm, rs_in[rank], order="ring"),
              oracle.ring_reduce_scatter(rs_in)[rank])
        if pow2:
            want = oracle.rechalf_reduce_scatter(rs_in)[rank]
            check(f"rs_rechalf_n{n}", pkg.rechalf_reduce_scatter(comm, rs_in[rank]), want)
            check(f"rs_direct_rec_n{n}", pkg.direct_reduce_scatter(comm, rs_in[rank], order="recursive"), want)

    sync_point("flat")
    # copy-engine all-gather (ag_variant 5): symmetric outputs, mixed with
    # kernel calls on the same group (separate counters must not interfere)
    from paper_2504_18658_b200 import _lib as _L

    if _L.lib().pccl_ce_available(torch.cuda.current_device()):
        w = comm.world
        for n in (1, 37, 4096, 300_000, 1 << 21):
            ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
            want = oracle.ring_all_gather(ag_in)[rank]
            x = torch.from_numpy(ag_in[rank]).cuda()
            out = w.empty(n * p, torch.float32)
            for it in range(3):
                for algo in (["ring", "recursive"] if pow2 else ["ring"]):
                    for variant in (5, -1):
                        w.set_param("ag_variant", variant)
                        out.fill_(float("nan"))
                        pkg.all_gather_into_tensor(out, x, comm, algorithm=algo)
                        check(f"ce_ag_{algo}_v{variant}_n{n}_{it}", out.cpu().numpy(), want)
            # in place: my block already sits in the output
            w.set_param("ag_variant", 5)
            out.zero_()
            out[rank * n:(rank + 1) * n].copy_(x)
            pkg.all_gather_into_tensor(out, out[rank * n:(rank + 1) * n], comm, algorithm="ring")
            check(f"ce_ag_inplace_n{n}", out.cpu().numpy(), want)
        # an output the peers cannot write into does not qualify: every rank
        # gets Unsupported (no silent per-rank fallback, no launch)
        w.set_param("ag_variant", 5)
        try:
            pkg.all_gather_into_tensor(torch.empty(4096 * p, device=x.device), torch.zeros(4096, device=x.device),
                                       comm, algorithm="ring")
            failures.append("ce_ag_unregistered_accepted")
        except pkg.errors.Unsupported:
            pass
        w.set_param("ag_variant", -1)
    sync_point("copy_engine")
    # direct RS, pipelined push (rs_variant 5) in every fold order, fp32 + bf16
    comm.world.set_param("rs_variant", 5)
    for n in (37, 4096, 300_000):
        rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
        for order in ["ring", "rank"] + (["recursive"] if pow2 else []):
            want = oracle.direct_reduce_scatter(rs_in, "f32", order)[rank]
            got = pkg.direct_reduce_scatter(comm, torch.from_numpy(rs_in[rank]).cuda(), order=order)
            check(f"rs_pp_{order}_n{n}", got.cpu().numpy(), want)
        bf = [oracle.f32_to_bf16(x) for x in rs_in]
        xb = torch.from_numpy(bf[rank].view(np.int16)).view(torch.bfloat16).cuda()
        got = pkg.direct_reduce_scatter(comm, xb, order="ring")
        check(f"rs_pp_bf16_n{n}", got.view(torch.int16).cpu().numpy().view(np.uint16),
              oracle.direct_reduce_scatter(bf, "bf16", "ring")[rank])
    comm.world.set_param("rs_variant", -1)
    sync_point("rs_pipelined_push")
    # LL128 line protocol (ag_variant 8) over real NVLink: sizes from one word
    # to a full region, alternated with LL and flag-protocol calls
    for words in (1, 15, 61, 4099, 100_000, (1 << 14) * 15):
        ag_in = [rng.standard_normal(words * 2).astype(np.float32) for _ in range(p)]
        want = oracle.ring_all_gather(ag_in)[rank]
        for variant in (8, -1, 8):
            comm.world.set_param("ag_variant", variant)
            got = pkg.direct_all_gather(comm, torch.from_numpy(ag_in[rank]).cuda())
            check(f"ll128_v{variant}_w{words}", got.cpu().numpy(), want)
    comm.world.set_param("ag_variant", -1)
    # LL128 reduce-scatter: the direct fold in every order over line streams
    for words in (1, 61, 4099, (1 << 14) * 15):
        rs_in = [rng.standard_normal(words * 2 * p).astype(np.float32) for _ in range(p)]
        for order in ["ring", "rank"] + (["recursive"] if pow2 else []):
            want = oracle.direct_reduce_scatter(rs_in, "f32", order)[rank]
            for variant in (8, -1):
                comm.world.set_param("rs_variant", variant)
                got = pkg.direct_reduce_scatter(comm, torch.from_numpy(rs_in[rank]).cuda(), order=order)
                check(f"ll128_rs_{order}_v{variant}_w{words}", got.cpu().numpy(), want)
    comm.world.set_param("rs_variant", -1)
    sync_point("ll128")
    # NVLS multicast segment (switch-executed AG stores / RS loads)
    from paper_2504_18658_b200 import nvls as NV

    if NV.nvls_supported(comm.world):  # one multicast member per device
        seg = NV.create_nvls_segment(comm.world, 16 << 20)
        try:
            for n in (8, 4096, 300_000):
                for dt in (torch.float32, torch.bfloat16):
                    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
                    xs = [torch.from_numpy(a).to(dt) for a in ag_in]
                    out = seg.tensor(0, n * p, dt)
                    for _ in range(2):
                        out.fill_(float("nan"))
                        NV.nvls_all_gather(comm, seg, xs[rank].cuda(), out)
                        check(f"nvls_ag_{dt}_n{n}", out.cpu().view(torch.uint8).numpy(),
                              torch.cat(xs).view(torch.uint8).numpy())
                    # RS: integer-valued inputs are exact in any summation order
                    vals = [torch.from_numpy(rng.integers(-30, 31, n * p).astype(np.float32)).to(dt) for _ in range(p)]
                    x = seg.tensor(1 << 20, n * p, dt)
                    x.copy_(vals[rank])
                    y = torch.empty(n, dtype=dt, device="cuda")
                    for _ in range(2):
                        NV.nvls_reduce_scatter(comm, seg, x, y)
                        want = sum(v.float() for v in vals)[rank * n:(rank + 1) * n].to(dt)
                        check(f"nvls_rs_{dt}_n{n}", y.cpu().float().numpy(), want.float().numpy())
            # bf16 standard normal: fp32 accumulation in the switch, one rounding
            n = 65536
            vals = [torch.randn(n * p, generator=torch.Generator().manual_seed(q)).to(torch.bfloat16) for q in range(p)]
            x = seg.tensor(1 << 20, n * p, torch.bfloat16)
            x.copy_(vals[rank])
            y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
            NV.nvls_reduce_scatter(comm, seg, x, y)
            ref = sum(v.float() for v in vals)[rank * n:(rank + 1) * n]
            bound = p * 2.0 ** -8 * sum(v.float().abs() for v in vals)[rank * n:(rank + 1) * n]
            if not bool(((y.cpu().float() - ref).abs() <= bound).all()):
                failures.append("nvls_rs_bf16_normal_bound")
        finally:
            seg.close()
    sync_point("nvls")
    # pipelined host path (slices of every chunk / block, copies overlapped
    # with the collectives): small slice size so several slices run
    from paper_2504_18658_b200 import collectives as C

    saved = (C.PIPE_MIN_BYTES, C.PIPE_SLICE_BYTES)
    C.PIPE_MIN_BYTES, C.PIPE_SLICE_BYTES = 256 << 10, 64 << 10
    try:
        n = 200_003
        rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
        ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        pinned = torch.from_numpy(rs_in[rank]).pin_memory()
        check("pipe_rs_ring", pkg.ring_reduce_scatter(comm, rs_in[rank]), oracle.ring_reduce_scatter(rs_in)[rank])
        check("pipe_rs_direct_pinned", pkg.direct_reduce_scatter(comm, pinned).numpy(),
              oracle.ring_reduce_scatter(rs_in)[rank])
        if pow2:
            check("pipe_rs_rechalf", pkg.rechalf_reduce_scatter(comm, pinned).numpy(),
                  oracle.rechalf_reduce_scatter(rs_in)[rank])
        want_ag = oracle.ring_all_gather(ag_in)[rank]
        check("pipe_ag_ring", pkg.ring_all_gather(comm, ag_in[rank]), want_ag)
        check("pipe_ag_direct_pinned", pkg.direct_all_gather(comm, torch.from_numpy(ag_in[rank]).pin_memory()).numpy(),
              want_ag)
    finally:
        C.PIPE_MIN_BYTES, C.PIPE_SLICE_BYTES = saved

    sync_point("pipelined_host")
    # bf16 on device tensors, both through staging and through symmetric buffers
    n = 65536 + 8
    ins = [oracle.f32_to_bf16(rng.standard_normal(n * p).astype(np.float32)) for _ in range(p)]
    dev_in = torch.from_numpy(ins[rank].view(np.int16)).view(torch.bfloat16).cuda()
    sym_in = comm.world.empty(n * p, torch.bfloat16)
    sym_in.copy_(dev_in)
    sym_out = comm.world.empty(n, torch.bfloat16)
    for algo, ref in [("ring", oracle.ring_reduce_scatter)] + ([("recursive", oracle.rechalf_reduce_scatter)] if pow2 else []):
        want = ref(ins, "bf16")[rank]
        got = pkg.reduce_scatter(comm, dev_in, algorithm=algo)
        check(f"bf16_{algo}_staged", got.view(torch.int16).cpu().numpy().view(np.uint16), want)
        got = pkg.reduce_scatter(comm, sym_in, algorithm=algo, out=sym_out)
        check(f"bf16_{algo}_symmetric", got.view(torch.int16).cpu().numpy().view(np.uint16), want)
    want = oracle.direct_reduce_scatter(ins, "bf16", "ring")[rank]
    got = pkg.reduce_scatter(comm, sym_in, algorithm="direct", out=sym_out)
    check("bf16_direct_symmetric", got.view(torch.int16).cpu().numpy().view(np.uint16), want)

    sync_point("bf16")
    # hierarchical virtual nodes
    grids = [(N, p // N) for N in (1, 2, 4, 8) if p % N == 0]
    for N, M in grids:
        for inter in ("ring", "recursive"):
            if inter == "recursive" and N & (N - 1):
                continue
            plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=inter)
            ag_in = [rng.standard_normal(1000).astype(np.float32) for _ in range(p)]
            check(f"hier_ag_{N}x{M}_{inter}", pkg.hier_all_gather(plan, comm, ag_in[rank]),
                  oracle.hier_all_gather(ag_in, N, M, inter)[rank])
            rs_in = [rng.standard_normal(1000 * p).astype(np.float32) for _ in range(p)]
            check(f"hier_rs_{N}x{M}_{inter}", pkg.hier_reduce_scatter(plan, comm, rs_in[rank]),
                  oracle.hier_reduce_scatter(rs_in, N, M, inter)[rank])

    sync_point("hier")
    # hierarchical launch variants: intra phase ring / direct x chained /
    # separate phase launches, aligned (chain eligible) and odd sizes, fp32
    # and bf16 (the direct intra RS folds with the ring's rounding points)
    for intra, chain in ((1, 1), (1, 0), (0, 0), (0, 1)):
        comm.world.set_param("hier_intra", intra)
        comm.world.set_param("hier_chain", chain)
        for N, M in [(N, M) for N, M in grids if N > 1 and M > 1]:
            for inter in ("ring", "recursive"):
                if inter == "recursive" and N & (N - 1):
                    continue
                plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=inter)
                tag = f"{N}x{M}_{inter}_intra{intra}_chain{chain}"
                for n in (37, 1000, 65536):
                    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
                    check(f"hierv_ag_{tag}_{n}", pkg.hier_all_gather(plan, comm, ag_in[rank]),
                          oracle.hier_all_gather(ag_in, N, M, inter)[rank])
                    rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
                    check(f"hierv_rs_{tag}_{n}", pkg.hier_reduce_scatter(plan, comm, rs_in[rank]),
                          oracle.hier_reduce_scatter(rs_in, N, M, inter)[rank])
                    bf = [oracle.f32_to_bf16(x) for x in rs_in]
                    got = pkg.hier_reduce_scatter(plan, comm, torch.from_numpy(bf[rank].view(np.int16)).view(
                        torch.bfloat16).cuda())
                    check(f"hierv_rs_bf16_{tag}_{n}", got.view(torch.int16).cpu().numpy().view(np.uint16),
                          oracle.hier_reduce_scatter(bf, N, M, inter, "bf16")[rank])
    comm.world.set_param("hier_intra", -1)
    comm.world.set_param("hier_chain", 1)
    sync_point("hier_variants")
    # back-to-back reuse + barrier
    for it in range(30):
        x = torch.full((4096 * p,), float(it + rank), device="cuda")
        y = pkg.reduce_scatter(comm, x, algorithm=["direct", "ring", "recursive" if pow2 else "ring"][it % 3])
        if float(y[0]) != sum(it + q for q in range(p)):
            failures.append(f"reuse_{it}")
    comm.barrier()

    sync_point("reuse")
    # random launch skew between ranks: the device handshakes absorb it
    import random
    import time

    rnd = random.Random(rank)
    x = torch.full((8192 * p,), float(rank + 1), device="cuda")
    for it in range(40):
        torch.cuda.synchronize()
        time.sleep(rnd.random() * 0.003)
        algo = ["direct", "ring", "recursive" if pow2 else "direct"][it % 3]
        y = pkg.reduce_scatter(comm, x, algorithm=algo)
        z = pkg.all_gather(comm, y, algorithm=algo)
        if float(y[0]) != p * (p + 1) / 2 or float(z[-1]) != p * (p + 1) / 2:
            failures.append(f"skew_{it}")

    sync_point("skew")
    # CUDA graph: capture collectives, replay, interleave with eager calls
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    gin = comm.world.empty(4096 * p, torch.float32)
    gout = comm.world.empty(4096, torch.float32)
    gag = comm.world.empty(4096 * p, torch.float32)
    gin.copy_(torch.arange(4096 * p, dtype=torch.float32, device="cuda") * (rank + 1))
    side = torch.cuda.Stream()
    ga = _lib.ALGOS["recursive" if pow2 else "ring"]

    def gstep(s):
        _lib.check(L.pccl_reduce_scatter(comm.handle, ga, 0, gin.data_ptr(), gout.data_ptr(), 4096, 0, s))
        _lib.check(L.pccl_all_gather(comm.handle, _lib.ALGOS["direct"], gout.data_ptr(), gag.data_ptr(), 4096, 0, s))

    torch.cuda.synchronize()
    gstep(side.cuda_stream)
    side.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        gstep(side.cuda_stream)
        gstep(side.cuda_stream)
    with torch.cuda.stream(side):  # replay() launches on the current stream
        for _ in range(20):
            graph.replay()
    gstep(side.cuda_stream)
    sync_point("graph")
    tot = p * (p + 1) / 2
    want = torch.arange(4096 * p, dtype=torch.float32, device="cuda") * tot
    if not torch.equal(gout, want[rank * 4096:(rank + 1) * 4096]) or not torch.equal(gag, want):
        failures.append("cuda_graph")

    # BASELINE configs at FULL size over real NVLink: every
    # rank regenerates its peers' seeded inputs on its own GPU and checks its
    # whole output bit for bit against the reduction-order restatement
    # (bench.expected_rs, pinned against the oracle by tests/test_bench.py)
    if os.environ.get("PCCL_TEST_FULLSIZE", "1") == "1":
        import bench

        rig = bench.Rig(True, p, rank, torch.device("cuda", torch.cuda.current_device()), dist, comm=comm)
        MiB = 1 << 20
        # C1: all-gather fp32, 64 MiB output, ring
        n = 64 * MiB // 4 // p
        bi, bo = rig.sym(n, torch.float32), rig.sym(n * p, torch.float32)
        sd = rig.new_seed()
        rig.fill(bi, sd)
        rig.ag("ring", bi, bo, n, 0)()
        if not rig.verify_ag(bi, bo, sd, n, torch.float32):
            failures.append("full_c1_ag_f32_64MiB_ring")
        # C2: reduce-scatter bf16, 128 MiB input, recursive halving (+ direct)
        n = 128 * MiB // 2 // p
        bi, bo = rig.sym(n * p, torch.bfloat16), rig.sym(n, torch.bfloat16)
        sd = rig.new_seed()
        rig.fill(bi, sd)
        for algo in (["recursive"] if pow2 else []) + ["direct", "ring"]:
            order = "recursive" if algo == "recursive" else "ring"
            rig.rs(algo, order, bi, bo, n, 1)()
            if not rig.verify_rs(bi, bo, sd, n, torch.bfloat16, algo, order):
                failures.append(f"full_c2_rs_bf16_128MiB_{algo}")
        # C3: hierarchical AG + RS fp32, 256 MiB, every virtual grouping
        n = 256 * MiB // 4 // p
        ai, ao = rig.sym(n, torch.float32), rig.sym(n * p, torch.float32)
        ri, ro = rig.sym(n * p, torch.float32), rig.sym(n, torch.float32)
        sa, sr = rig.new_seed(), rig.new_seed()
        rig.fill(ai, sa)
        rig.fill(ri, sr)
        for N in [g for g in (2, 4) if p % g == 0 and 1 < g < p]:
            for inter in ["ring"] + (["recursive"] if N & (N - 1) == 0 else []):
                rig.hier("ag", N, p // N, inter, ai, ao, n, 0)()
                if not rig.verify_ag(ai, ao, sa, n, torch.float32):
                    failures.append(f"full_c3_hier_ag_{N}x{p // N}_{inter}")
                rig.hier("rs", N, p // N, inter, ri, ro, n, 0)()
                if not rig.verify_rs(ri, ro, sr, n, torch.float32, "hierarchical", grid=(N, p // N), inter=inter):
                    failures.append(f"full_c3_hier_rs_{N}x{p // N}_{inter}")
        del ai, ao, ri, ro, bi, bo
        # C5: GPT-3-style 7B per-layer shapes, bf16, direct AG + RS
        n7 = bench.P7 // p
        prm, full = rig.sym(n7, torch.bfloat16), rig.sym(n7 * p, torch.bfloat16)
        sd = rig.new_seed()
        rig.fill(prm, sd)
        rig.ag("direct", prm, full, n7, 1)()
        if not rig.verify_ag(prm, full, sd, n7, torch.bfloat16):
            failures.append("full_c5_ag_bf16_direct")
        del prm, full
        grad, gsh = rig.sym(n7 * p, torch.bfloat16), rig.sym(n7, torch.bfloat16)
        sd = rig.new_seed()
        rig.fill(grad, sd)
        rig.rs("direct", "ring", grad, gsh, n7, 1)()
        if not rig.verify_rs(grad, gsh, sd, n7, torch.bfloat16, "direct", "ring"):
            failures.append("full_c5_rs_bf16_direct")
        del grad, gsh
        sync_point("fullsize")

    # zero-copy for torch-owned tensors: register caching-allocator buffers
    # collectively (CUDA IPC of the containing allocation + offset), then the
    # collectives bind them without staging; and the symmetric heap
    w = comm.world
    n = 300_001
    xr = torch.randn(n * p, device="cuda")
    yr = torch.empty(n, device="cuda")
    zr = torch.empty(n * p, device="cuda")
    with w.register(xr), w.register(yr), w.register(zr):
        w.set_param("staged_bytes", 0)
        all_x = [torch.empty_like(xr) for _ in range(p)]
        dist.all_gather(all_x, xr)
        for algo in ["direct", "ring"] + (["recursive"] if pow2 else []):
            order = "recursive" if algo == "recursive" else "ring"
            pkg.reduce_scatter(comm, xr, algorithm=algo, order=order, out=yr)
            want = oracle.rechalf_reduce_scatter([a.cpu().numpy() for a in all_x])[rank] if algo == "recursive" \
                else oracle.ring_reduce_scatter([a.cpu().numpy() for a in all_x])[rank]
            check(f"registered_rs_{algo}", yr.cpu().numpy(), want)
            pkg.all_gather(comm, yr, algorithm=algo, out=zr)
            all_y = [torch.empty_like(yr) for _ in range(p)]
            dist.all_gather(all_y, yr)
            check(f"registered_ag_{algo}", zr.cpu().numpy(), torch.cat(all_y).cpu().numpy())
        torch.cuda.synchronize()
        if w.get_param("staged_bytes") != 0:
            failures.append(f"registered buffers staged {w.get_param('staged_bytes')} B")
    heap = w.heap(64 << 20)
    a = heap.empty(n * p, torch.float32)
    b = heap.empty(n, torch.float32)
    a.copy_(xr)
    w.set_param("staged_bytes", 0)
    pkg.reduce_scatter(comm, a, algorithm="direct", out=b)
    torch.cuda.synchronize()
    check("heap_rs_direct", b.cpu().numpy(), oracle.ring_reduce_scatter([t.cpu().numpy() for t in all_x])[rank])
    if w.get_param("staged_bytes") != 0:
        failures.append("heap buffers staged")
    del a, b
    sync_point("registration")

    # point-to-point over the mailbox rings (transport/base.py:140-152)
    nxt, prv = (rank + 1) % p, (rank - 1) % p
    big = np.full((5 << 20) // 4 + 3, rank + 0.5, np.float32)  # > one 2 MiB ring: fragments
    got = comm.sendrecv(nxt, 21, big.tobytes()) if p == 2 else None
    if p > 2:
        comm.send(nxt, 21, big.tobytes())
        got = comm.recv(prv, 21)
    if np.frombuffer(got, np.float32)[0] != prv + 0.5 or len(got) != big.nbytes:
        failures.append("p2p_big_ring")
    for it in range(20):
        comm.send(nxt, 100 + it, torch.full((4096,), float(rank * 1000 + it), device="cuda"))
    for it in reversed(range(20)):  # out of tag order
        t = torch.empty(4096, device="cuda")
        comm.recv_into(prv, 100 + it, t)
        if not bool((t == prv * 1000 + it).all()):
            failures.append(f"p2p_tag_{it}")
    sync_point("p2p")

    # online calibration: every rank must resolve "auto" identically afterwards
    from paper_2504_18658_b200 import selector, tuning

    tuned = tuning.autotune(comm, "reduce_scatter", 4 << 20, iters=3, warmup=1)
    pick = selector.choose_algorithm("reduce_scatter", p, 4 << 20)
    picks = [None] * p
    dist.all_gather_object(picks, (pick, sorted(tuned)))
    if len(set(map(str, picks))) != 1 or pick not in tuned or not all(v > 0 for v in tuned.values()):
        failures.append(f"autotune {picks} {tuned}")
    sync_point("autotune")

    # cross-rank length mismatch must raise LengthMismatch (device-side check)
    from paper_2504_18658_b200.errors import LengthMismatch

    # a multi-step collective whose buffers are aligned differently on one
    # rank (here rank 0's output sits 4 bytes into its allocation) cuts other
    # slices there: detected through the call signature on every rank, and
    # the world recovers after a collective flag reset
    n = 4096
    xin = torch.ones(n * p, device="cuda")
    buf = torch.empty(n + 4, device="cuda")
    yout = buf[1:1 + n] if rank == 0 else buf[:n]
    try:
        pkg.ring_reduce_scatter(comm, xin, out=yout)
        torch.cuda.synchronize()
        comm.world.check()
        failures.append("alignment_mismatch_not_detected")
    except LengthMismatch:
        pass
    torch.cuda.synchronize()
    dist.barrier()
    comm.world.reset_flags()
    dist.barrier()
    y2 = pkg.ring_reduce_scatter(comm, xin)  # the world works again
    torch.cuda.synchronize()
    if not torch.equal(y2, torch.full((n,), float(p), device="cuda")):
        failures.append("after_alignment_mismatch_reset")

    try:
        pkg.direct_all_gather(comm, np.zeros(4 if rank == 0 else 2, np.float32))
        failures.append("mismatch_not_detected")
    except LengthMismatch:
        pass

    torch.cuda.synchronize()
    print(f"[rank {rank}] {'OK' if not failures else 'FAIL ' + ','.join(failures)}", flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    try:
        code = main()
    except Exception:
        traceback.print_exc()
        code = 2
    os._exit(code)
