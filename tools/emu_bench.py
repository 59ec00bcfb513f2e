"""Quick emulation-mode timing (p ranks on one GPU, one launch per call)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_18658_b200  # noqa: F401  (loads the library)
from paper_2504_18658_b200 import _lib
from paper_2504_18658_b200.communicator import emulated_world, _emu_group

def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    w = emulated_world(p)
    members = tuple(range(p))
    g, _ = _emu_group(w, members, 0)
    for S_mb in (16, 128):
        S = S_mb << 20
        for coll in ("ag", "rs"):
            for dt in (torch.float32, torch.bfloat16):
                es = 2 if dt == torch.bfloat16 else 4
                if coll == "ag":
                    n = S // es // p
                    segs_in = w.empty(n, dt); segs_out = w.empty(n * p, dt)
                else:
                    n = S // es // p
                    segs_in = w.empty(n * p, dt); segs_out = w.empty(n, dt)
                for t in segs_in: t.normal_()
                w.ensure_staging(int(_lib.lib().pccl_staging_bytes(1, 1, p, n, 1 if es == 2 else 0)) + (S * 2))
                for algo in ("direct", "ring", "recursive"):
                    a = _lib.ALGOS[algo]; code = 1 if es == 2 else 0
                    sp = _lib.ptr_array([t.data_ptr() for t in segs_in]); rp = _lib.ptr_array([t.data_ptr() for t in segs_out])
                    st = torch.cuda.current_stream().cuda_stream
                    def call():
                        if coll == "ag":
                            return _lib.lib().pccl_emu_all_gather(g.handle, a, sp, rp, n, code, st)
                        return _lib.lib().pccl_emu_reduce_scatter(g.handle, a, 0, sp, rp, n, code, st)
                    for _ in range(3): _lib.check(call())
                    torch.cuda.synchronize(); w.check()
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    K = 10
                    e0.record()
                    for _ in range(K): _lib.check(call())
                    e1.record(); torch.cuda.synchronize(); w.check()
                    t = e0.elapsed_time(e1) / K * 1e-3
                    busbw = S * (p - 1) / p / t / 1e9
                    # HBM bytes (all emulated ranks): AG: read (p-1)n+n, write p n per rank; RS similar scale
                    print(f"p={p} {coll} {str(dt)[6:]:9s} S={S_mb:4d}MiB {algo:9s} {t*1e6:9.1f} us  busbw(emu)={busbw:8.1f} GB/s", flush=True)
                for t in segs_in + segs_out: pass

if __name__ == "__main__":
    main()
