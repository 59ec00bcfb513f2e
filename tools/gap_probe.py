"""Kernel-to-kernel turnaround per GPU, no communication (torchrun, one rank
per GPU, every rank at once): 2000 one-CTA kernels captured in a CUDA graph
and replayed; the per-kernel time is the GPU's completion -> next-launch gap
plus a trivial body. Used to tell a per-GPU property of the box apart from the
collectives' own exit cost (profiles/r2_overhead_p4.md: 2 vs 5 us gaps).

    torchrun --nproc-per-node 4 tools/gap_probe.py
"""
import os

import torch
import torch.distributed as dist


def main():
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    x = torch.zeros(1, device="cuda")
    s = torch.cuda.Stream()
    K = 2000
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(K):
            x.add_(1)
    res = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        with torch.cuda.stream(s):
            a.record()
            g.replay()
            b.record()
        b.synchronize()
        res.append(a.elapsed_time(b) * 1e3 / K)
    out = [None] * p
    dist.all_gather_object(out, (dev, torch.cuda.get_device_properties(dev).pci_bus_id, [round(v, 3) for v in res]))
    if rank == 0:
        for o in out:
            print(f"GPU {o[0]} (bus {o[1]:#x}): us per graph kernel {o[2]}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
