"""Host-link probe for the end-to-end path (torchrun, one rank per GPU): per
GPU H2D / D2H bandwidth with every rank copying at once, pinned buffers
allocated (a) wherever the process happens to run and (b) after binding the
process to the CPUs local to its GPU (so the pinned pages land on the GPU's
NUMA node).

    torchrun --nproc-per-node 4 tools/numa_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def gpu_sysfs(dev: int) -> str:
    pr = torch.cuda.get_device_properties(dev)
    return f"/sys/bus/pci/devices/{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"


def cpulist(s: str) -> set:
    out = set()
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


def main():
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    path = gpu_sysfs(dev)
    try:
        node = open(os.path.join(path, "numa_node")).read().strip()
        local = cpulist(open(os.path.join(path, "local_cpulist")).read())
    except OSError as exc:
        node, local = f"? ({exc})", set()
    n = 64 << 20  # bf16 elements: 128 MiB
    d = torch.empty(n, dtype=torch.bfloat16, device="cuda")

    def measure(tag):
        x = torch.empty(n, dtype=torch.bfloat16).normal_().pin_memory()
        y = torch.empty(n // 4, dtype=torch.bfloat16, pin_memory=True)
        res = {}
        for name, fn in (("h2d_128MiB", lambda: d.copy_(x, non_blocking=True)),
                         ("d2h_32MiB", lambda: y.copy_(d[: n // 4], non_blocking=True))):
            fn()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 10
            nbytes = x.numel() * 2 if name.startswith("h2d") else y.numel() * 2
            res[name] = f"{dt * 1e3:.2f} ms {nbytes / dt / 1e9:.1f} GB/s"
        return {tag: res}

    out = {"gpu": path, "numa": node, "local_cpus": len(local), "affinity_before": len(os.sched_getaffinity(0))}
    out.update(measure("default"))
    if local:
        os.sched_setaffinity(0, local & os.sched_getaffinity(0) or local)
        out.update(measure("numa_local"))
    allr = [None] * p
    dist.all_gather_object(allr, out)
    if rank == 0:
        for i, o in enumerate(allr):
            print(i, o, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
