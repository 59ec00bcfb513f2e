"""Per-CTA event timeline of one collective (torchrun, real mode).

For each rank: mean / max over CTAs of the time from kernel start to each
event (wait done W<unit>, signal S<unit>, end E), so the cost of every
handshake and every step is visible. Times are per-GPU %globaltimer.
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coll", default="rs_bf16"); ap.add_argument("--algo", default="recursive")
    ap.add_argument("--variant", type=int, default=-1); ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--size-kib", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0); ap.add_argument("--nsub", type=int, default=1)
    ap.add_argument("--item-kib", type=int, default=-1)
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"])); torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib
    comm = pkg.init_from_torch(device=dev.index); w = comm.world; L = _lib.lib()
    kind, dt = a.coll.split("_"); dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    es = 2 if dt == "bf16" else 4; code = _lib.DTYPES[dt]; S = (a.size_kib << 10) if a.size_kib else (a.size_mib << 20); n = S // es // p
    sin = w.empty(n * p if kind == "rs" else n, dtype); sout = w.empty(n if kind == "rs" else n * p, dtype); sin.normal_()
    alg = _lib.ALGOS[a.algo]
    w.ensure_staging(int(L.pccl_staging_bytes(1 if kind == "rs" else 0, alg, p, n, code)))
    w.set_param("ag_variant" if kind == "ag" else "rs_variant", a.variant)
    if a.ctas: w.set_param("ctas", a.ctas)
    w.set_param("nsub", a.nsub)
    if a.item_kib >= 0: w.set_param("item_kib", a.item_kib)
    st = torch.cuda.current_stream(dev).cuda_stream
    def f():
        if kind == "ag": _lib.check(L.pccl_all_gather(comm.handle, alg, sin.data_ptr(), sout.data_ptr(), n, code, st))
        else: _lib.check(L.pccl_reduce_scatter(comm.handle, alg, 0, sin.data_ptr(), sout.data_ptr(), n, code, st))
    for _ in range(5): f()
    torch.cuda.synchronize(); dist.barrier()
    w.set_param("trace", 1)
    for _ in range(3): f()   # trace keeps the last launch
    torch.cuda.synchronize()
    tr = [[[e for e in ev if e[1] not in (5, 6, 7, 8)] for ev in w.trace()[0]]][0]
    # per CTA: relative times of the k-th event
    import statistics
    nev = min(len(ev) for ev in tr)
    rows = []
    for k in range(nev):
        lab = None; rel = []
        for ev in tr:
            t0 = ev[0][0]; t, kd, u = ev[k]
            lab = {1: "start", 2: f"W{u}", 3: f"S{u}", 4: "end"}[kd]; rel.append((t - t0) / 1e3)
        rows.append((lab, statistics.mean(rel), max(rel), min(rel)))
    starts = [ev[0][0] for ev in tr]; ends = [ev[nev - 1][0] for ev in tr]
    span = (max(ends) - min(starts)) / 1e3
    out = [f"rank {rank}: {len(tr)} CTAs, kernel span {span:.1f} us, CTA start spread {(max(starts)-min(starts))/1e3:.1f} us"]
    for lab, mean, mx, mn in rows:
        out.append(f"   {lab:6s} mean {mean:8.1f}  min {mn:8.1f}  max {mx:8.1f} us")
    outs = [None] * p
    dist.all_gather_object(outs, "\n".join(out))
    if rank == 0:
        print(f"== {a.coll} {a.algo} variant={a.variant} p={p} {S >> 10} KiB ctas={a.ctas or 'auto'} nsub={a.nsub} item_kib={a.item_kib}")
        for o in outs[:2]: print(o)
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    main()
