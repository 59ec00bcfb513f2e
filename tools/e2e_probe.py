"""Break down the end-to-end (host buffers) path: H2D, collective, D2H, and
the pipelined host path against the unpipelined one (torchrun, real mode)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    rank, p = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))); torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import collectives as C, _lib
    L = _lib.lib()
    comm = pkg.init_from_torch(device=dev.index)
    S = 128 << 20
    n = S // 2 // p
    x = torch.empty(n * p, dtype=torch.bfloat16).normal_().pin_memory()
    d = torch.empty(n * p, dtype=torch.bfloat16, device=dev)
    h = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    hbig = torch.empty(n * p, dtype=torch.bfloat16, pin_memory=True)
    st = torch.cuda.current_stream(dev)
    s2 = torch.cuda.Stream(dev)
    def t(f, k=5):
        f(); torch.cuda.synchronize(); dist.barrier()
        t0 = time.perf_counter()
        for _ in range(k): f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / k * 1e3
    r = {}
    r["h2d_128MiB"] = t(lambda: d.copy_(x, non_blocking=True))
    r["d2h_128MiB"] = t(lambda: hbig.copy_(d, non_blocking=True))
    r["d2h_chunk"] = t(lambda: h.copy_(d[:n], non_blocking=True))
    K = 16
    def h2d_2d():
        cs = n // K
        for k in range(K):
            L.pccl_copy2d(d.data_ptr() + k * cs * p * 2, cs * 2, x.data_ptr() + k * cs * 2, n * 2, cs * 2, p, st.cuda_stream)
    r["h2d_2d_16slices"] = t(h2d_2d)
    def h2d_1d():
        cs = n * p // K
        for k in range(K):
            L.pccl_copy2d(d.data_ptr() + k * cs * 2, cs * 2, x.data_ptr() + k * cs * 2, cs * 2, cs * 2, 1, st.cuda_stream)
    r["h2d_1d_16slices"] = t(h2d_1d)
    def both():
        d.copy_(x, non_blocking=True)
        with torch.cuda.stream(s2):
            hbig.copy_(d, non_blocking=True)
        st.wait_stream(s2)
    r["h2d||d2h_128MiB"] = t(both)
    r["api_e2e_piped"] = t(lambda: pkg.rechalf_reduce_scatter(comm, x))
    saved = C.PIPE_MIN_BYTES
    C.PIPE_MIN_BYTES = 1 << 60
    r["api_e2e_unpiped"] = t(lambda: pkg.rechalf_reduce_scatter(comm, x))
    C.PIPE_MIN_BYTES = saved
    for sl in (4 << 20, 16 << 20, 32 << 20):
        C.PIPE_SLICE_BYTES = sl
        r[f"api_e2e_piped_{sl >> 20}MiB"] = t(lambda: pkg.rechalf_reduce_scatter(comm, x))
    C.PIPE_SLICE_BYTES = 8 << 20
    y = comm.world.empty(n, torch.bfloat16); s = comm.world.empty(n * p, torch.bfloat16)
    r["device_only"] = t(lambda: pkg.rechalf_reduce_scatter(comm, s, out=y))
    import cProfile, pstats, io
    pr = cProfile.Profile(); pr.enable()
    for _ in range(3): pkg.rechalf_reduce_scatter(comm, x)
    pr.disable()
    out = [None] * p
    dist.all_gather_object(out, r)
    if rank == 0:
        print(f"p={p}, ms per call")
        for i, o in enumerate(out): print(i, {k: round(v, 3) for k, v in o.items()})
        s_ = io.StringIO(); pstats.Stats(pr, stream=s_).sort_stats("tottime").print_stats(12); print(s_.getvalue()[:3000])
    dist.destroy_process_group()

if __name__ == "__main__":
    main()
