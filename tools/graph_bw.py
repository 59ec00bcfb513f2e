"""Eager launches vs CUDA-graph replay for the bulk collectives (torchrun, real
mode): K back-to-back calls issued eagerly, and the same K calls captured in
one CUDA graph and replayed, for our kernels and for NCCL. On these boxes an
eagerly launched kernel that touched peer memory pays ~3.6 us more at its
boundary than the same kernel inside a graph (tools/pdl_probe.cu), which is
most of the inter-collective gap (tools/trace_seq.py).

    torchrun --nproc-per-node 4 tools/graph_bw.py [--sizes 64,128,256] [--k 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256")
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--algos", default="direct,ring,recursive")
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

    def timed(fn, graph: bool) -> float:
        with torch.cuda.stream(side):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(a.k):
                    fn()
            torch.cuda.synchronize()
            run = g.replay
        else:
            def run():
                for _ in range(a.k):
                    fn()
        best = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                fn()  # device-side rendezvous
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(side)
                run()
                e1.record(side)
            e1.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3 / a.k], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best.append(float(t.item()))
        return min(best)

    lines = []
    for smib in map(int, a.sizes.split(",")):
        S = smib << 20
        for coll, dtype, code in (("rs_bf16", torch.bfloat16, 1), ("ag_f32", torch.float32, 0)):
            es = torch.empty(0, dtype=dtype).element_size()
            n = S // es // p
            x = w.empty(n * p if coll.startswith("rs") else n, dtype)
            y = w.empty(n if coll.startswith("rs") else n * p, dtype)
            x.normal_()
            for algo in a.algos.split(","):
                al = _lib.ALGOS[algo]
                o = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]
                w.ensure_staging(int(L.pccl_staging_bytes(1 if coll.startswith("rs") else 0, al, p, n, code)))

                def fn(al=al, o=o):
                    st = torch.cuda.current_stream(dev).cuda_stream
                    if coll.startswith("rs"):
                        _lib.check(L.pccl_reduce_scatter(comm.handle, al, o, x.data_ptr(), y.data_ptr(), n, code, st))
                    else:
                        _lib.check(L.pccl_all_gather(comm.handle, al, x.data_ptr(), y.data_ptr(), n, code, st))

                te, tg = timed(fn, False), timed(fn, True)
                bw = lambda t: S * (p - 1) / p / t / 1e9  # noqa: E731
                lines.append(f"p={p} {coll:7s} {smib:5d} MiB {algo:9s} eager {te * 1e6:7.1f} us {bw(te):6.1f} GB/s"
                             f"   graph {tg * 1e6:7.1f} us {bw(tg):6.1f} GB/s")
            nx = torch.empty_like(x)
            ny = torch.empty_like(y)
            nx.normal_()

            def nfn():
                if coll.startswith("rs"):
                    dist.reduce_scatter_tensor(ny, nx)
                else:
                    dist.all_gather_into_tensor(ny, nx)

            te, tg = timed(nfn, False), timed(nfn, True)
            bw = lambda t: S * (p - 1) / p / t / 1e9  # noqa: E731
            lines.append(f"p={p} {coll:7s} {smib:5d} MiB {'NCCL':9s} eager {te * 1e6:7.1f} us {bw(te):6.1f} GB/s"
                         f"   graph {tg * 1e6:7.1f} us {bw(tg):6.1f} GB/s")
            del x, y, nx, ny
    if rank == 0:
        print("\n".join(lines), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
