"""NVLS collectives vs unicast kernels vs NCCL (torchrun, real mode): busbw
per CTA count for the switch-executed AG / RS, and NCCL on the same bytes
(run once with NCCL_ALGO=NVLS to compare against NCCL's own NVLS path).

    torchrun --nproc-per-node 4 tools/nvls_tune.py [--ctas 16,32,64,128,148]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", default="16,32,64,128,148")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import nvls as NV

    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world

    def timeit(f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        dist.barrier()
        f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters / 1e3], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    def bw(S, t):
        return S * (p - 1) / p / t / 1e9

    seg = NV.create_nvls_segment(w, 512 << 20)
    out = []
    for S, coll, dt in ((128 << 20, "rs", torch.bfloat16), (64 << 20, "ag", torch.float32),
                        (384 << 20, "rs", torch.bfloat16), (384 << 20, "ag", torch.bfloat16)):
        es = torch.empty(0, dtype=dt).element_size()
        n = S // es // p
        if coll == "rs":
            x = seg.tensor(0, n * p, dt)
            x.normal_()
            y = torch.empty(n, dtype=dt, device=dev)
            f = lambda: NV.nvls_reduce_scatter(comm, seg, x, y)  # noqa: E731
            ni, no = torch.randn(n * p, device=dev).to(dt), torch.empty(n, dtype=dt, device=dev)
            fn = lambda: dist.reduce_scatter_tensor(no, ni)  # noqa: E731
        else:
            x = torch.randn(n, device=dev).to(dt)
            y = seg.tensor(0, n * p, dt)
            f = lambda: NV.nvls_all_gather(comm, seg, x, y)  # noqa: E731
            ni, no = torch.randn(n, device=dev).to(dt), torch.empty(n * p, dtype=dt, device=dev)
            fn = lambda: dist.all_gather_into_tensor(no, ni)  # noqa: E731
        for c in map(int, a.ctas.split(",")):
            w.set_param("ctas", c)
            out.append(f"p={p} nvls {coll} {dt} {S >> 20} MiB ctas={c:4d}: {bw(S, timeit(f)):7.1f} GB/s")
        w.set_param("ctas", 0)
        out.append(f"p={p} NCCL {coll} {dt} {S >> 20} MiB (NCCL_ALGO={os.environ.get('NCCL_ALGO', 'default')}): "
                   f"{bw(S, timeit(fn)):7.1f} GB/s")
    seg.close()
    if rank == 0:
        print("\n".join(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
