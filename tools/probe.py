"""Raw NVLink throughput probe (torchrun, one process per GPU).

Patterns: 'uni' (rank 0 -> rank 1 only), 'bi' (0 <-> 1), 'a2a' (every rank
to every other), 'ring' (r -> r+1), 'one2all' (rank 0 -> all others).
Reports per-GPU egress GB/s (push) / ingress (pull) as max-over-ranks time.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--pats", default="uni,bi,a2a,ring,one2all")
    ap.add_argument("--modes", default="0,1", help="0 push16 1 pull16 2 push32 3 pull32 (bytes per access); "
                    "4 / 5 = TMA bulk push / pull (PROBE_TMA=stages x tile); 9 = copy-engine push (cudaMemcpyAsync into each peer, one stream per peer)")
    ap.add_argument("--ctas", default="8,16,32,64,128")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"])); torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib
    comm = pkg.init_from_torch(device=dev.index, staging_bytes=0)
    w = comm.world
    B = 128 << 20
    seg = w.create_segment(2 * B)
    L = _lib.lib(); st = torch.cuda.current_stream(dev)
    pats = {"uni": lambda r: (1 << 1) if r == 0 else 0, "bi": lambda r: (1 << (1 - r)) if r < 2 else 0,
            "a2a": lambda r: ((1 << p) - 1) & ~(1 << r), "ring": lambda r: 1 << ((r + 1) % p),
            "one2all": lambda r: (((1 << p) - 1) & ~1) if r == 0 else 0}
    names = {0: "push16", 1: "pull16", 2: "push32", 3: "pull32", 4: "tma_push", 5: "tma_pull", 6: "red_f32x4", 7: "red_bf16x8", 9: "ce_push"}
    ap2 = os.environ.get("PROBE_TMA", "")  # "stages x tile", e.g. 4x32768
    if ap2:
        stg, tile = map(int, ap2.split("x"))
        w.set_param("tma_stages", stg)
        w.set_param("tma_tile", tile)
    peer_streams = [torch.cuda.Stream(dev) for _ in range(p)]
    for pat in a.pats.split(","):
        fm = pats[pat]
        for mode in map(int, a.modes.split(",")):
            for ctas in map(int, a.ctas.split(",")):
                mask = fm(rank)
                npeers = bin(mask).count("1")
                per = (B // max(1, npeers)) // 32 * 32
                def f():
                    if mask and mode == 9:
                        src = seg.ptr(rank)
                        for q in range(p):
                            if (mask >> q) & 1:
                                ps = peer_streams[q]
                                ps.wait_stream(st)
                                _lib.check(L.pccl_copy2d(seg.ptr(q) + B + (rank if rank < q else rank - 1) * per, per, src, per, per, 1,
                                                         ps.cuda_stream))
                        for q in range(p):
                            if (mask >> q) & 1:
                                st.wait_stream(peer_streams[q])
                    elif mask:
                        _lib.check(L.pccl_probe(w.handle, seg.id, mode, mask, per, ctas, st.cuda_stream))
                for _ in range(3): f()
                torch.cuda.synchronize(); dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10): f()
                e1.record(); torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 10 * 1e-3
                bw = (per * npeers / t / 1e9) if mask else 0.0
                tt = torch.tensor([bw], device=dev)
                g = [torch.zeros(1, device=dev) for _ in range(p)]
                dist.all_gather(g, tt)
                if rank == 0:
                    vals = [round(float(x), 1) for x in g]
                    print(f"p={p} {pat:8s} {names[mode]} ctas={ctas:4d} per-rank GB/s {vals}", flush=True)
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    main()
