"""NVLink hardware byte counters around a collective (torchrun, real mode).

ncu cannot replay a kernel that handshakes with peers on other GPUs, so the
NVLink evidence comes from the NVML per-link counters instead: every rank
reads TX/RX (data payload and raw incl. protocol) before and after K calls and
reports bytes per call next to the algorithmic (p-1)/p * S.

    torchrun --nproc-per-node N tools/nvlink_counters.py [--size-mib 128] [--calls 50]

Finding (round 1, gpurun B200 boxes): NVML answers NOT_SUPPORTED (3) for
every NVLink throughput/byte field and `nvidia-smi nvlink -gt d` prints N/A,
so the tool reports n/a there; the timings it prints (device events, max over
ranks, public API) are still valid.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def nvml_handle(dev):
    import pynvml as nv

    nv.nvmlInit()
    props = torch.cuda.get_device_properties(dev)
    bus = f"{props.pci_domain_id:08X}:{props.pci_bus_id:02X}:{props.pci_device_id:02X}.0"
    try:
        return nv, nv.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:  # noqa: BLE001
        return nv, nv.nvmlDeviceGetHandleByIndex(dev.index)


FIELDS = {"data_tx_kib": 138, "data_rx_kib": 139, "raw_tx_kib": 140, "raw_rx_kib": 141, "xmit_bytes": 202,
          "rcv_bytes": 204}


def read_counters(nv, h, links: int = 18) -> dict:
    """Sum over links of each field; None when NVML does not expose it.
    One NVML call per field (all links), scope = link id."""
    out = {}
    for name, fid in FIELDS.items():
        try:
            vals = nv.nvmlDeviceGetFieldValues(h, [(fid, s) for s in range(links)])
        except Exception as exc:  # noqa: BLE001
            out[name] = None
            out[name + "_err"] = repr(exc)[:80]
            continue
        good = [int(v.value.ullVal) for v in vals if v.nvmlReturn == 0]
        out[name] = sum(good) if good else None
        if not good:
            out[name + "_err"] = f"nvmlReturn {vals[0].nvmlReturn}"
    for agg in (0xFFFFFFFF,):
        for name, fid in FIELDS.items():
            if out.get(name) is None:
                try:
                    v = nv.nvmlDeviceGetFieldValues(h, [(fid, agg)])[0]
                    if v.nvmlReturn == 0:
                        out[name] = int(v.value.ullVal)
                        out.pop(name + "_err", None)
                except Exception:  # noqa: BLE001
                    pass
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size-mib", type=int, default=128)
    ap.add_argument("--calls", type=int, default=50)
    ap.add_argument("--cases", default="rs_bf16:recursive,rs_bf16:direct,rs_bf16:ring,ag_f32:direct,ag_f32:ring,"
                                       "ag_f32:recursive,nccl_rs_bf16,nccl_ag_f32")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    import paper_2504_18658_b200 as pkg

    comm = pkg.init_from_torch(device=dev.index)
    w = comm.world
    nv, h = nvml_handle(dev)
    S = a.size_mib << 20
    results = []
    for case in a.cases.split(","):
        nccl = case.startswith("nccl_")
        coll, dt = (case[5:] if nccl else case.split(":")[0]).split("_")
        algo = None if nccl else case.split(":")[1]
        if algo == "recursive" and p & (p - 1):
            continue
        dtype = torch.bfloat16 if dt == "bf16" else torch.float32
        es = 2 if dt == "bf16" else 4
        n_in = S // es if coll == "rs" else S // es // p
        n_out = n_in // p if coll == "rs" else n_in * p
        if nccl:
            x = torch.empty(n_in, dtype=dtype, device=dev).normal_()
            y = torch.empty(n_out, dtype=dtype, device=dev)
            fn = (lambda: dist.reduce_scatter_tensor(y, x)) if coll == "rs" else (
                lambda: dist.all_gather_into_tensor(y, x))
        else:
            x = w.empty(n_in, dtype)
            x.normal_()
            y = w.empty(n_out, dtype)
            op = pkg.reduce_scatter if coll == "rs" else pkg.all_gather
            fn = lambda: op(comm, x, algorithm=algo, out=y)  # noqa: E731
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        c0 = read_counters(nv, h)
        dist.barrier()  # every rank has read its counters before anyone launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.calls):
            fn()
        e1.record()
        torch.cuda.synchronize()
        c1 = read_counters(nv, h)
        dist.barrier()
        if rank == 0 and case == a.cases.split(",")[0]:
            print("counter status:", {k: v for k, v in c1.items() if k.endswith("_err")} or "all available",
                  flush=True)
        tt = torch.tensor([e0.elapsed_time(e1) / 1e3 / a.calls], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt)
        per_call = {}
        for k in FIELDS:
            if c0[k] is None or c1[k] is None:
                per_call[k] = None
            else:
                scale = 1024 if k.endswith("kib") else 1
                per_call[k] = (c1[k] - c0[k]) * scale / a.calls
        algo_bytes = (p - 1) / p * S
        rec = {"case": case, "rank": rank, "p": p, "S": S, "t_us": t * 1e6, "busbw": algo_bytes / t / 1e9,
               "algorithmic_bytes": algo_bytes, **{k + "_per_call": v for k, v in per_call.items()}}
        allr = [None] * p
        dist.all_gather_object(allr, rec)
        if rank == 0:
            results.extend(allr)
            tx = [r["data_tx_kib_per_call"] for r in allr]
            rx = [r["data_rx_kib_per_call"] for r in allr]
            raw = [r["raw_tx_kib_per_call"] for r in allr]
            f = lambda v: "n/a" if v is None else f"{v / algo_bytes:.3f}"  # noqa: E731
            print(f"p={p} {case:22s} {t * 1e6:8.1f} us busbw {algo_bytes / t / 1e9:6.1f} | per call / algorithmic: "
                  f"data tx {[f(v) for v in tx]} rx {[f(v) for v in rx]} raw tx {[f(v) for v in raw]} "
                  f"| xmit {[f(r['xmit_bytes_per_call']) for r in allr]}", flush=True)
    if rank == 0 and a.json:
        with open(a.json, "w") as fh:
            json.dump(results, fh, indent=1)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
