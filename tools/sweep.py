"""Message-size sweep (BASELINE configs[3], C4): busbw of every algorithm and
CTA count vs NCCL, real mode under torchrun. Writes
gpurun_out/sweep_p{p}.csv (all points) and, with --write-table, the measured
selector table paper_2504_18658_b200/data/flat_calibration.csv rows for this p.

    torchrun --nproc-per-node N tools/sweep.py [--min-mib 1 --max-mib 1024]
"""
import argparse
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-mib", type=float, default=1)
    ap.add_argument("--max-mib", type=float, default=1024)
    ap.add_argument("--ctas", default="8,16,32,64,128")
    ap.add_argument("--colls", default="ag_f32,rs_bf16")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--write-table", action="store_true")
    ap.add_argument("--no-hier", action="store_true", help="skip the hierarchical N x M groupings (C4)")
    args = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    stream = torch.cuda.current_stream(dev)
    sizes = []
    s = args.min_mib
    while s <= args.max_mib:
        sizes.append(int(s * (1 << 20)))
        s *= 2
    rows = []
    maxS = max(sizes)

    def timeit(f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters * 1e-3], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    for coll in args.colls.split(","):
        kind, dt = coll.split("_")
        dtype = torch.bfloat16 if dt == "bf16" else torch.float32
        es = 2 if dt == "bf16" else 4
        code = _lib.DTYPES[dt]
        big_in = w.empty(maxS // es, dtype)
        big_out = w.empty(maxS // es, dtype)
        big_in.normal_()
        nin = torch.empty(maxS // es, dtype=dtype, device=dev).normal_()
        nout = torch.empty(maxS // es, dtype=dtype, device=dev)
        for S in sizes:
            n = S // es // p
            if n == 0:
                continue
            for algo in ("direct", "ring", "recursive"):
                if algo == "recursive" and p & (p - 1):
                    continue
                a = _lib.ALGOS[algo]
                o = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]
                w.ensure_staging(int(L.pccl_staging_bytes(0 if kind == "ag" else 1, a, p, n, code)))
                for ctas in map(int, args.ctas.split(",")):
                    w.set_param("ctas", ctas)
                    if kind == "ag":
                        f = lambda: _lib.check(L.pccl_all_gather(comm.handle, a, big_in.data_ptr(), big_out.data_ptr(),  # noqa
                                                                n, code, stream.cuda_stream))
                    else:
                        f = lambda: _lib.check(L.pccl_reduce_scatter(comm.handle, a, o, big_in.data_ptr(),  # noqa
                                                                    big_out.data_ptr(), n, code, stream.cuda_stream))
                    t = timeit(f)
                    w.check()
                    rows.append(dict(coll=coll, p=p, S=S, algo=algo, ctas=ctas, us=t * 1e6,
                                     busbw=S * (p - 1) / p / t / 1e9))
            w.set_param("ctas", 0)
            # hierarchical virtual groupings (C4: N x M in {2x4, 4x2, 2x2}), auto CTAs
            grids = [] if args.no_hier else [(N, p // N) for N in (2, 4) if p % N == 0 and 1 < N < p]
            for N, M in grids:
                for inter in ["ring"] + (["recursive"] if N & (N - 1) == 0 else []):
                    ia = _lib.ALGOS[inter]
                    w.ensure_staging(int(L.pccl_staging_bytes(0 if kind == "ag" else 1, 3, p, n, code)))
                    hf = L.pccl_hier_all_gather if kind == "ag" else L.pccl_hier_reduce_scatter
                    f = lambda: _lib.check(hf(w.handle, N, M, ia, big_in.data_ptr(), big_out.data_ptr(), n, code,  # noqa
                                              stream.cuda_stream))
                    t = timeit(f)
                    w.check()
                    rows.append(dict(coll=coll, p=p, S=S, algo=f"hier{N}x{M}_{inter}", ctas=0, us=t * 1e6,
                                     busbw=S * (p - 1) / p / t / 1e9))
            if kind == "ag":
                f = lambda: dist.all_gather_into_tensor(nout[: n * p], nin[:n])  # noqa
            else:
                f = lambda: dist.reduce_scatter_tensor(nout[:n], nin[: n * p])  # noqa
            t = timeit(f)
            rows.append(dict(coll=coll, p=p, S=S, algo="nccl", ctas=0, us=t * 1e6, busbw=S * (p - 1) / p / t / 1e9))
            if rank == 0:
                best = max((r for r in rows if r["coll"] == coll and r["S"] == S and r["algo"] != "nccl"
                            and not r["algo"].startswith("hier")), key=lambda r: r["busbw"])
                hier = [r for r in rows if r["coll"] == coll and r["S"] == S and r["algo"].startswith("hier")]
                nc = rows[-1]
                print(f"p={p} {coll:8s} S={S / 2**20:8.2f} MiB  best {best['algo']:9s} ctas={best['ctas']:3d} "
                      f"{best['busbw']:7.1f} GB/s ({best['us']:8.1f} us)   NCCL {nc['busbw']:7.1f} GB/s ({nc['us']:8.1f} us)"
                      f"  ratio {best['busbw'] / nc['busbw']:.2f}"
                      + "".join(f"  {h['algo']} {h['busbw']:.1f}" for h in hier), flush=True)
    if rank == 0:
        os.makedirs("gpurun_out", exist_ok=True)
        with open(f"gpurun_out/sweep_p{p}.csv", "w", newline="") as fh:
            wr = csv.DictWriter(fh, fieldnames=list(rows[0].keys()))
            wr.writeheader()
            wr.writerows(rows)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
