"""Randomised real-mode fuzz of the collective protocols (one process per GPU,
launched by tests/test_gpu_multiproc.py or by hand under torchrun).

Every iteration all ranks draw the same random call — collective, algorithm,
fold order, dtype, size (LL-sized to 16 MiB, ragged), buffer kind (symmetric,
unregistered, 4-byte misaligned), hierarchical grid — and check their own
output against values recomputed on the device. Inputs are small integers
(|x| <= 30) so every fold order is exact in fp32 / bf16 / fp16 and results
must match bit-for-bit. Every few iterations a burst of calls is captured in
a CUDA graph and replayed. Exit code 0 = no mismatch on this rank.

    torchrun --nproc-per-node 4 tests/mp_fuzz.py --iters 2000 --seed 1
"""
import argparse
import os
import random
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

DTYPES = [torch.float32, torch.bfloat16, torch.float16]


def values(it: int, q: int, start: int, n: int, dtype, dev):
    i = torch.arange(start, start + n, device=dev, dtype=torch.int64)
    return ((i * 7 + q * 13 + it * 5) % 61 - 30).to(dtype)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if local >= torch.cuda.device_count():  # one process per GPU, never shared
        raise SystemExit(f"rank {rank}: local rank {local} >= {torch.cuda.device_count()} visible GPUs")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg

    from paper_2504_18658_b200 import _lib, collectives as C

    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    ce = bool(_lib.lib().pccl_ce_available(dev.index))
    C.PIPE_MIN_BYTES, C.PIPE_SLICE_BYTES = 64 << 10, 16 << 10  # host buffers: sliced path, many slices
    from paper_2504_18658_b200 import nvls as NV

    seg = NV.create_nvls_segment(w, 64 << 20) if NV.nvls_supported(w) else None
    rng = random.Random(a.seed)  # same stream on every rank: SPMD calls
    pow2 = p & (p - 1) == 0
    grids = [(N, p // N) for N in (2, 4) if p % N == 0 and 1 < N < p]
    failures = []
    pool = {}

    def sym(n, dtype, slot):
        """Symmetric buffer of >= n elements, reused per (slot, dtype)."""
        key = (slot, dtype)
        t = pool.get(key)
        if t is None or t.numel() < n:
            t = w.empty(max(n, 1), dtype)
            pool[key] = t
        return t[:n]

    def one_call(it):
        coll = rng.choice(["ag", "rs", "rs", "hier"] if grids else ["ag", "rs"])
        if rng.random() < 0.15:  # NVLS (switch multicast) on the same world group, interleaved
            dtype = rng.choice(DTYPES)
            n = rng.choice([8, 1000, 40000, 1 << 18])
            if seg is None:
                return torch.zeros(1), torch.zeros(1), "nvls unsupported"
            if rng.random() < 0.5:
                x = values(it, rank, 0, n, dtype, dev)
                y = seg.tensor(1 << 20, n * p, dtype)
                NV.nvls_all_gather(comm, seg, x, y)
                want = torch.cat([values(it, q, 0, n, dtype, dev) for q in range(p)])
                return y.clone(), want, f"nvls ag {dtype} n={n}"
            x = seg.tensor(1 << 20, n * p, dtype)
            x.copy_(values(it, rank, 0, n * p, dtype, dev))
            y = torch.empty(n, dtype=dtype, device=dev)
            NV.nvls_reduce_scatter(comm, seg, x, y)
            want = sum(values(it, q, rank * n, n, torch.float32, dev) for q in range(p)).to(dtype)
            return y, want, f"nvls rs {dtype} n={n}"
        dtype = rng.choice(DTYPES)
        es = torch.empty(0, dtype=dtype).element_size()
        n = rng.choice([1, 3, 64, 1000, 4096, 40000, 262144, 1 << 20, (4 << 20) // es])
        if coll != "ag":
            n = max(1, n // p)
        algo = rng.choice(["direct", "ring"] + (["recursive"] if pow2 else []))
        order = rng.choice(["ring", "rank"] + (["recursive"] if pow2 else []))
        kind = rng.choice(["sym", "plain", "misaligned", "host"] if coll != "hier" else ["sym", "plain", "misaligned"])
        w.set_param("item_kib", rng.choice([0, 0, 16, 64]))  # direct kernels: static slices / work items
        w.set_param("rs_variant", rng.choice([-1, -1, 5, 7, 8]))  # 5: pipelined push (direct), 7: work items (recursive), 8: LL128
        # hierarchical: intra phase auto / ring / direct, chained or separate
        # phase launches, CTA count default or forced (chaining needs <= 128)
        w.set_param("hier_intra", rng.choice([-1, 0, 1]))
        w.set_param("hier_chain", rng.choice([1, 1, 0]))
        w.set_param("ctas", rng.choice([0, 0, 0, 24, 96, 160]))
        # 5: copy engine (ring / recursive into a registered output; every rank
        # takes the same choice, a call that does not qualify is an error)
        use_ce = ce and coll == "ag" and kind == "sym" and algo != "direct" and rng.random() < 0.4
        w.set_param("ag_variant", 5 if use_ce else (8 if coll == "ag" and rng.random() < 0.3 else -1))
        total_in = n if coll == "ag" else n * p
        total_out = n * p if coll == "ag" else n
        if kind == "sym":
            x, y = sym(total_in, dtype, "in"), sym(total_out, dtype, "out")
        elif kind == "plain":
            x = torch.empty(total_in, dtype=dtype, device=dev)
            y = torch.empty(total_out, dtype=dtype, device=dev)
        elif kind == "misaligned":
            x = torch.empty(total_in + 2, dtype=dtype, device=dev)[1:1 + total_in]
            y = torch.empty(total_out + 2, dtype=dtype, device=dev)[1:1 + total_out]
        else:  # pinned host input -> fresh host output (the reference-shaped path)
            x = torch.empty(total_in, dtype=dtype, pin_memory=True)
            y = None
        x.copy_(values(it, rank, 0, total_in, dtype, dev))
        if kind == "host":
            if coll == "ag":
                y = pkg.all_gather(comm, x, algorithm=algo).to(dev)
                want = torch.cat([values(it, q, 0, n, dtype, dev) for q in range(p)])
            else:
                y = pkg.reduce_scatter(comm, x, algorithm=algo, order=order).to(dev)
                want = sum(values(it, q, rank * n, n, torch.float32, dev) for q in range(p)).to(dtype)
            return y, want, f"{coll} {algo}/{order} {dtype} n={n} host"
        if coll == "ag":
            pkg.all_gather(comm, x, algorithm=algo, out=y)
            want = torch.cat([values(it, q, 0, n, dtype, dev) for q in range(p)])
            what = f"ag {algo} {dtype} n={n} {kind}"
        elif coll == "rs":
            pkg.reduce_scatter(comm, x, algorithm=algo, order=order, out=y)
            acc = sum(values(it, q, rank * n, n, torch.float32, dev) for q in range(p))
            want = acc.to(dtype)
            what = f"rs {algo}/{order} {dtype} n={n} {kind}"
        else:
            N, M = rng.choice(grids)
            inter = rng.choice(["ring"] + (["recursive"] if N & (N - 1) == 0 else []))
            plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=inter)
            if rng.random() < 0.5:
                xin = x[:n] if kind != "sym" else sym(n, dtype, "hin")
                xin.copy_(values(it, rank, 0, n, dtype, dev))
                yo = torch.empty(n * p, dtype=dtype, device=dev)
                pkg.hier_all_gather(plan, comm, xin, out=yo)
                y = yo
                want = torch.cat([values(it, q, 0, n, dtype, dev) for q in range(p)])
                what = f"hier ag {N}x{M} {inter} {dtype} n={n}"
            else:
                y = torch.empty(n, dtype=dtype, device=dev)
                pkg.hier_reduce_scatter(plan, comm, x, out=y)
                want = sum(values(it, q, rank * n, n, torch.float32, dev) for q in range(p)).to(dtype)
                what = f"hier rs {N}x{M} {inter} {dtype} n={n}"
        return y, want, what

    for it in range(a.iters):
        if it % 25 == 24:
            w.set_param("ag_variant", -1)
            w.set_param("rs_variant", -1)
            w.set_param("item_kib", 0)
            # CUDA graph: capture three fixed calls on a side stream, replay, verify
            side = torch.cuda.Stream(dev)
            n = rng.choice([256, 8192, 1 << 18])
            gx = sym(n * p, torch.float32, "gx")
            gy = sym(n, torch.float32, "gy")
            gz = sym(n * p, torch.float32, "gz")
            gx.copy_(values(it, rank, 0, n * p, torch.float32, dev))
            torch.cuda.synchronize()
            pkg.reduce_scatter(comm, gx, algorithm="direct", out=gy)  # size the segments before capture
            pkg.all_gather(comm, gy, algorithm="direct", out=gz)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                pkg.reduce_scatter(comm, gx, algorithm="direct", out=gy)
                pkg.all_gather(comm, gy, algorithm="direct", out=gz)
            with torch.cuda.stream(side):
                for _ in range(3):
                    g.replay()
            torch.cuda.synchronize()
            full = sum(values(it, q, 0, n * p, torch.float32, dev) for q in range(p))
            if not torch.equal(gz, full):
                failures.append(f"it {it}: graph rs+ag n={n}")
            continue
        y, want, what = one_call(it)
        if not torch.equal(y, want):
            bad = (y != want).nonzero()
            failures.append(f"it {it}: {what}: {bad.numel()} wrong, first at {bad[:1].tolist()}")
            if len(failures) > 5:
                break
        if it % 50 == 0:
            torch.cuda.synchronize()
            w.check()
    torch.cuda.synchronize()
    w.check()
    if seg is not None:
        seg.close()
    eps = [None] * p
    dist.all_gather_object(eps, comm.epoch())
    if len(set(eps)) != 1:
        failures.append(f"epochs diverged {eps}")
    print(f"[rank {rank}] {'FUZZ OK' if not failures else 'FUZZ FAIL ' + '; '.join(failures[:5])} ({a.iters} iters)",
          flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    try:
        code = main()
    except Exception:
        traceback.print_exc()
        code = 2
    os._exit(code)
