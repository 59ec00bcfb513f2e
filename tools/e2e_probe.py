"""Break down the end-to-end (host buffers) path: H2D, collective, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    rank, p = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))); torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    comm = pkg.init_from_torch(device=dev.index)
    n = (128 << 20) // 2 // p
    x = torch.empty(n * p, dtype=torch.bfloat16).normal_().pin_memory()
    d = torch.empty(n * p, dtype=torch.bfloat16, device=dev)
    h = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    def t(f, k=5):
        f(); torch.cuda.synchronize(); dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k): f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / k * 1e3
    r = {}
    r["h2d_128MiB_ms"] = t(lambda: d.copy_(x, non_blocking=True))
    r["d2h_32MiB_ms"] = t(lambda: h.copy_(d[:n], non_blocking=True))
    r["api_e2e_ms"] = t(lambda: pkg.rechalf_reduce_scatter(comm, x))
    y = comm.world.empty(n, torch.bfloat16); s = comm.world.empty(n * p, torch.bfloat16)
    r["device_only_ms"] = t(lambda: pkg.rechalf_reduce_scatter(comm, s, out=y))
    r["device_torch_ms"] = t(lambda: pkg.rechalf_reduce_scatter(comm, d))
    import cProfile, pstats, io
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3): pkg.rechalf_reduce_scatter(comm, x)
    pr.disable()
    out = [None] * p
    dist.all_gather_object(out, r)
    if rank == 0:
        for i, o in enumerate(out): print(i, {k: round(v, 3) for k, v in o.items()})
        s_ = io.StringIO(); pstats.Stats(pr, stream=s_).sort_stats("cumulative").print_stats(18); print(s_.getvalue()[:3500])
    dist.destroy_process_group()

if __name__ == "__main__":
    main()
