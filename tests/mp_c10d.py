"""torch.distributed backend worker (torchrun, one process per GPU): a
"pccl" process group (paper_2504_18658_b200.c10d) next to the default NCCL
group; every collective checked against NCCL's result on the same inputs,
then an FSDP1 (FullyShardedDataParallel) forward + backward on the pccl group
against the same model on the NCCL group. Exit code 0 = all checks passed."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> int:
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2504_18658_b200 import c10d  # registers the backend

    g = c10d.new_group()
    failures = []

    def same(name, a, b):
        ia = a.view(torch.int16) if a.dtype in (torch.bfloat16, torch.float16) else a.view(torch.int32)
        ib = b.view(torch.int16) if b.dtype in (torch.bfloat16, torch.float16) else b.view(torch.int32)
        if not torch.equal(ia, ib):
            failures.append(name)

    gen = torch.Generator(device=dev).manual_seed(7 + rank)
    for n, dt in ((4099, torch.float32), (1 << 20, torch.bfloat16), (3 << 20, torch.float32)):
        x = torch.randn(n, generator=gen, device=dev).to(dt)
        a, b = torch.empty(n * p, dtype=dt, device=dev), torch.empty(n * p, dtype=dt, device=dev)
        dist.all_gather_into_tensor(a, x, group=g)
        dist.all_gather_into_tensor(b, x)
        same(f"all_gather_into_tensor {dt} n={n}", a, b)
        outs = [torch.empty(n, dtype=dt, device=dev) for _ in range(p)]
        dist.all_gather(outs, x, group=g)
        same(f"all_gather list {dt} n={n}", torch.cat(outs), b)
        # integer-valued inputs: sums exact in any order, so equal to NCCL's bits
        xi = torch.randint(-30, 31, (n * p,), generator=gen, device=dev).to(dt)
        y, z = torch.empty(n, dtype=dt, device=dev), torch.empty(n, dtype=dt, device=dev)
        dist.reduce_scatter_tensor(y, xi, group=g)
        dist.reduce_scatter_tensor(z, xi)
        same(f"reduce_scatter_tensor {dt} n={n}", y, z)
        dist.reduce_scatter(y, list(xi.chunk(p)), group=g)
        same(f"reduce_scatter list {dt} n={n}", y, z)
        r1, r2 = xi.clone(), xi.clone()
        dist.all_reduce(r1, group=g)
        dist.all_reduce(r2)
        same(f"all_reduce {dt} n={n}", r1, r2)
    dist.barrier(group=g)
    torch.cuda.synchronize()

    # FSDP1 on the pccl group vs the same model on the NCCL group
    from torch.distributed.fsdp import FullyShardedDataParallel as FSDP

    def model():
        torch.manual_seed(0)
        return torch.nn.Sequential(torch.nn.Linear(1024, 4096), torch.nn.GELU(), torch.nn.Linear(4096, 1024)).to(dev)

    xin = torch.randn(64, 1024, generator=gen, device=dev)
    res = []
    for group in (g, None):
        m = FSDP(model(), process_group=group, use_orig_params=True)
        loss = m(xin).float().pow(2).mean()
        loss.backward()
        grads = [q.grad.detach().clone() for q in m.parameters() if q.grad is not None]
        res.append((loss.detach(), grads))
    torch.cuda.synchronize()
    same("fsdp1 loss", res[0][0].reshape(1), res[1][0].reshape(1))
    for i, (ga, gb) in enumerate(zip(res[0][1], res[1][1])):
        if not torch.allclose(ga, gb, rtol=1e-5, atol=1e-6):
            failures.append(f"fsdp1 grad {i}")
    print(f"[rank {rank}] C10D {'OK' if not failures else 'FAIL ' + '; '.join(failures)}", flush=True)
    dist.barrier()
    return 1 if failures else 0


if __name__ == "__main__":
    try:
        code = main()
    except Exception:
        traceback.print_exc()
        code = 2
    sys.stdout.flush()
    os._exit(code)
