"""Steady-state timeline of K back-to-back launches of one collective
(torchrun, real mode): per launch, when its CTAs became resident (before the
PDL wait), when they passed it, and when they exited; the gap between
consecutive launches on each GPU and the in-kernel phases.

    torchrun --nproc-per-node 4 tools/trace_seq.py --coll rs_bf16 --algo recursive
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

K = 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--coll", default="rs_bf16")
    ap.add_argument("--algo", default="recursive")
    ap.add_argument("--variant", type=int, default=-1)
    ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--params", default="", help="key=value,... world params")
    ap.add_argument("--backend", default="nccl", help="bootstrap process group (nccl | gloo)")
    ap.add_argument("--poll", type=float, default=0, help="experiment: a host thread queries the stream every POLL ms (0 off)")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    if a.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(a.backend)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    comm = pkg.init_from_torch(device=dev.index)
    w, L = comm.world, _lib.lib()
    kind, dt = a.coll.split("_")
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    es, code = (2 if dt == "bf16" else 4), _lib.DTYPES[dt]
    S = a.size_mib << 20
    n = S // es // p
    sin = w.empty(n * p if kind == "rs" else n, dtype)
    sout = w.empty(n if kind == "rs" else n * p, dtype)
    sin.normal_()
    alg = _lib.ALGOS[a.algo]
    order = _lib.ORDERS["recursive" if a.algo == "recursive" else "ring"]
    w.ensure_staging(int(L.pccl_staging_bytes(1 if kind == "rs" else 0, alg, p, n, code)))
    w.set_param("ag_variant" if kind == "ag" else "rs_variant", a.variant)
    w.set_param("pdl", a.pdl)
    if a.ctas:
        w.set_param("ctas", a.ctas)
    for kv in filter(None, a.params.split(",")):
        k, v = kv.split("=")
        w.set_param(k, int(v))
    st = torch.cuda.current_stream(dev)

    def f():
        if kind == "ag":
            _lib.check(L.pccl_all_gather(comm.handle, alg, sin.data_ptr(), sout.data_ptr(), n, code, st.cuda_stream))
        else:
            _lib.check(L.pccl_reduce_scatter(comm.handle, alg, order, sin.data_ptr(), sout.data_ptr(), n, code,
                                             st.cuda_stream))

    for _ in range(5):
        f()
    torch.cuda.synchronize()
    dist.barrier()
    stop = None
    if a.poll > 0:
        import threading
        import time as _t

        stop = threading.Event()
        qs = torch.cuda.Stream(dev)

        def poller():
            while not stop.is_set():
                qs.query()
                if a.poll >= 0.01:
                    _t.sleep(a.poll / 1e3)

        threading.Thread(target=poller, daemon=True).start()
    w.set_param("trace", K)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f()  # the trace ring is cleared before this launch
    e0.record(st)
    for _ in range(K - 1):
        f()
    e1.record(st)
    torch.cuda.synchronize()
    if stop is not None:
        stop.set()
    per_call = e0.elapsed_time(e1) * 1e3 / (K - 1)
    launches = [w.trace(back)[0] for back in range(K - 1, -1, -1)]  # oldest first
    w.set_param("trace", 0)
    lines = [f"rank {rank}: event-timed {per_call:.1f} us per call"]
    prev_exit = prev_epi = None
    t_base = min(ev[0][0] for ev in launches[0] if ev)
    for i, ctas in enumerate(launches):
        res = [next(t for t, kd, _ in ev if kd == 6) for ev in ctas]
        st0 = [next(t for t, kd, _ in ev if kd == 1) for ev in ctas]
        ex = [next(t for t, kd, _ in ev if kd == 5) for ev in ctas]
        pdl = [next((t for t, kd, _ in ev if kd == 8), None) for ev in ctas]
        epi = [t for ev in ctas for t, kd, _ in ev if kd == 7]
        waits = {}
        for ev in ctas:
            s0 = next(t for t, kd, _ in ev if kd == 1)
            for t, kd, u in ev:
                if kd in (2, 3, 4):
                    waits.setdefault((kd, u), []).append((t - s0) / 1e3)
        phase = " ".join(f"{'WSE'[kd - 2]}{u}={statistics.mean(v):.1f}/{max(v):.1f}" for (kd, u), v in
                         sorted(waits.items(), key=lambda kv: statistics.mean(kv[1])))
        gap = (min(st0) - prev_exit) / 1e3 if prev_exit is not None else float("nan")
        # gap split: last exit -> last epilogue (exit counter atomic) -> PDL release -> start (epoch read)
        split = ""
        if prev_exit is not None and prev_epi and all(pdl):
            split = (f" [exit->epi {(prev_epi - prev_exit) / 1e3:.1f}, epi->pdl {(min(pdl) - prev_epi) / 1e3:.1f},"
                     f" pdl->start {(min(st0) - min(pdl)) / 1e3:.1f}]")
        lines.append(f"  L{i}: resident {(min(res) - t_base) / 1e3:8.1f} start {(min(st0) - t_base) / 1e3:8.1f}"
                     f"..{(max(st0) - t_base) / 1e3:8.1f} exit mean {(statistics.mean(ex) - t_base) / 1e3:8.1f} "
                     f"max {(max(ex) - t_base) / 1e3:8.1f} span {(max(ex) - min(st0)) / 1e3:6.1f} "
                     f"gap {gap:5.1f}{split} | {phase}")
        prev_exit = max(ex)
        prev_epi = max(epi) if epi else None
    outs = [None] * p
    dist.all_gather_object(outs, "\n".join(lines))
    if rank == 0:
        print(f"== {a.coll} {a.algo} variant={a.variant} p={p} {a.size_mib} MiB ctas={a.ctas or 'auto'} pdl={a.pdl}"
              f" {a.params}")
        for o in outs:
            print(o)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
