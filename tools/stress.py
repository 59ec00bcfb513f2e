"""Back-to-back stress of one collective (torchrun, real mode).

    torchrun --nproc-per-node N tools/stress.py --algo recursive --iters 20000 [--smi]

Runs `iters` calls in batches of 20 without host sync in between (like the
bench soak). With --smi an nvidia-smi sampler runs concurrently. On a device
error, prints the per-CTA trace of the last launch (trace param on).
"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="recursive")
    ap.add_argument("--coll", default="rs_bf16")
    ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--iters", type=int, default=10000)
    ap.add_argument("--smi", action="store_true")
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg
    from paper_2504_18658_b200 import _lib

    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    L = _lib.lib()
    kind, dt = a.coll.split("_")
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    es = 2 if dt == "bf16" else 4
    code = _lib.DTYPES[dt]
    n = (a.size_mib << 20) // es // p
    sin = w.empty(n * p if kind == "rs" else n, dtype)
    sout = w.empty(n if kind == "rs" else n * p, dtype)
    sin.normal_()
    alg = _lib.ALGOS[a.algo]
    w.ensure_staging(int(L.pccl_staging_bytes(1 if kind == "rs" else 0, alg, p, n, code)))
    if a.trace:
        w.set_param("trace", 1)
    st = torch.cuda.current_stream(dev).cuda_stream

    def f():
        if kind == "ag":
            return L.pccl_all_gather(comm.handle, alg, sin.data_ptr(), sout.data_ptr(), n, code, st)
        return L.pccl_reduce_scatter(comm.handle, alg, 0, sin.data_ptr(), sout.data_ptr(), n, code, st)

    smi = None
    if a.smi:  # one sampler per rank, the bench's exact query
        smi = subprocess.Popen(["nvidia-smi", "-i", str(dev.index),
                                "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                                "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                                "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                "--format=csv,noheader,nounits", "-lms", "100"],
                               stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    gaps = []
    t0 = time.time()
    err = None
    done = 0
    for it in range(0, a.iters, 20):
        tb = time.time()
        for _ in range(20):
            s = f()
            if s:
                err = f"status {s} ({_lib.error_string(s)}) at call {done}"
                break
            done += 1
        torch.cuda.synchronize()
        gaps.append(time.time() - tb)
        s = L.pccl_world_check(w.handle)
        if s and not err:
            err = f"device {s} ({_lib.error_string(s)}) before call {done}"
        if err:
            break
    dt = time.time() - t0
    if smi:
        smi.terminate()
    msg = (f"[rank {rank}] {a.coll} {a.algo} calls={done} time={dt:.1f}s max-batch={max(gaps) * 1e3:.1f}ms "
           + (f"ERROR {err}" if err else "OK"))
    if err and a.trace:
        tr = w.trace()[0]
        last = {}
        for b, ev in enumerate(tr):
            key = tuple((k, u) for _, k, u in ev[1:])
            last.setdefault(key, []).append(b)
        msg += "\n  last-launch event sequences (kind,unit) -> CTAs: " + "; ".join(
            f"{k}: {len(v)} CTAs (e.g. {v[:4]})" for k, v in sorted(last.items(), key=lambda kv: -len(kv[1]))[:6])
    print(msg, flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
