"""Small-message latency breakdown (torchrun, real mode).

Per size: eager per-call device time (events over K back-to-back C-ABI
calls), host time per call (enqueue only), the same K calls captured in one
CUDA graph and replayed, and NCCL eager / graph for comparison.

    torchrun --nproc-per-node N tools/latency.py [--sizes 65536,1048576] [--k 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="65536,1048576,4194304")
    ap.add_argument("--k", type=int, default=200)
    ap.add_argument("--algos", default="direct,recursive")
    ap.add_argument("--colls", default="ag,rs")
    ap.add_argument("--pdl", default="1", help="comma list of PDL settings to compare (param pdl)")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--api", choices=["c", "python"], default="c",
                    help="c: ctypes calls of the C ABI; python: the package's public functions")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    side = torch.cuda.Stream(dev)

    def tmax(x):
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def measure(fn, k):
        with torch.cuda.stream(side):
            for _ in range(5):
                fn(side.cuda_stream)
            side.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0 = time.perf_counter()
            e0.record(side)
            for _ in range(k):
                fn(side.cuda_stream)
            e1.record(side)
            h1 = time.perf_counter()
            side.synchronize()
            dev_us = e0.elapsed_time(e1) * 1e3 / k
            host_us = (h1 - h0) * 1e6 / k
            # graph: the same k calls captured once
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(k):
                    fn(side.cuda_stream)
            g.replay()
            side.synchronize()
            dist.barrier()
            e0.record(side)
            g.replay()
            e1.record(side)
            side.synchronize()
            graph_us = e0.elapsed_time(e1) * 1e3 / k
        return tmax(dev_us), tmax(host_us), tmax(graph_us)

    for coll in a.colls.split(","):
        for S in map(int, a.sizes.split(",")):
            n = S // 4 // p
            if coll == "ag":
                x, y = w.empty(n, torch.float32), w.empty(n * p, torch.float32)
            else:
                x, y = w.empty(n * p, torch.float32), w.empty(n, torch.float32)
            for algo, pdl in [(x, int(q)) for x in a.algos.split(",") for q in a.pdl.split(",")]:
                w.set_param("pdl", pdl)
                al = _lib.ALGOS[algo]
                w.ensure_staging(int(L.pccl_staging_bytes(0 if coll == "ag" else 1, al, p, n, 0)))
                if a.api == "python":
                    op = pkg.all_gather if coll == "ag" else pkg.reduce_scatter
                    fn = lambda s, op=op, algo=algo: op(comm, x, algorithm=algo, out=y)  # noqa: E731
                elif coll == "ag":
                    fn = lambda s: _lib.check(L.pccl_all_gather(comm.handle, al, x.data_ptr(), y.data_ptr(), n, 0, s))  # noqa: E731
                else:
                    fn = lambda s: _lib.check(L.pccl_reduce_scatter(comm.handle, al, 0, x.data_ptr(), y.data_ptr(), n, 0, s))  # noqa: E731
                d, h, g = measure(fn, a.k)
                if rank == 0:
                    print(f"p={p} {a.api:6s} {coll} {S >> 10:7d} KiB {algo:10s} pdl={pdl} eager {d:7.2f} us/call (host enqueue {h:6.2f}) "
                          f"graph {g:7.2f} us/call", flush=True)
            if a.no_nccl:
                continue
            nx = torch.empty_like(x)
            ny = torch.empty_like(y)
            if coll == "ag":
                fn = lambda s: dist.all_gather_into_tensor(ny, nx)  # noqa: E731
            else:
                fn = lambda s: dist.reduce_scatter_tensor(ny, nx)  # noqa: E731
            try:
                d, h, g = measure(fn, a.k)
                if rank == 0:
                    print(f"p={p} {coll} {S >> 10:7d} KiB {'NCCL':10s} eager {d:7.2f} us/call (host enqueue {h:6.2f}) "
                          f"graph {g:7.2f} us/call", flush=True)
            except Exception as exc:  # noqa: BLE001
                if rank == 0:
                    print(f"NCCL graph capture failed: {exc!r}"[:200], flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
