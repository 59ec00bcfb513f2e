"""FSDP2 worker (torchrun, one process per GPU): a two-layer model with
GPT-3-style 7B per-layer shapes (12h^2 + 13h parameters, h = 4096), bf16
mixed precision, one forward + backward with PyTorch's default NCCL
collectives and one with the B200 collectives installed through
``paper_2504_18658_b200.fsdp.install`` (same init, same data). Checks:

* unsharded parameters (the all-gather outputs) bit-identical to NCCL's;
* the forward loss bit-identical;
* sharded gradients (the reduce-scatter outputs) within the bf16 bound of
  NCCL's (different reduction order / rounding points);
* zero bytes staged by the B200 worlds (every FSDP buffer came from the
  symmetric heaps);
and prints the step times of both. Exit code 0 = all checks passed."""
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.nn as nn  # noqa: E402

H = int(os.environ.get("PCCL_FSDP_H", "4096"))
REPS = int(os.environ.get("PCCL_FSDP_REPS", "5"))


class Block(nn.Module):
    """12h^2 + 13h parameters: QKV (3h^2+3h), attention out (h^2+h), MLP
    (4h^2+4h, 4h^2+h), two LayerNorms (4h)."""

    def __init__(self, h):
        super().__init__()
        self.ln1, self.ln2 = nn.LayerNorm(h), nn.LayerNorm(h)
        self.qkv, self.proj = nn.Linear(h, 3 * h), nn.Linear(h, h)
        self.fc1, self.fc2 = nn.Linear(h, 4 * h), nn.Linear(4 * h, h)

    def forward(self, x):
        q, k, v = self.qkv(self.ln1(x)).chunk(3, dim=-1)
        x = x + self.proj(torch.tanh(q) * k + v)
        return x + self.fc2(torch.nn.functional.gelu(self.fc1(self.ln2(x))))


def build(dev):
    from torch.distributed.fsdp import MixedPrecisionPolicy, fully_shard

    torch.manual_seed(0)
    model = nn.Sequential(Block(H), Block(H)).to(dev)
    mp = MixedPrecisionPolicy(param_dtype=torch.bfloat16, reduce_dtype=torch.bfloat16)
    for blk in model:
        fully_shard(blk, mp_policy=mp)
    fully_shard(model, mp_policy=mp)
    return model


def step(model, x, reps=1):
    """Forward + backward; returns the last loss and the mean step time."""
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        model.zero_grad(set_to_none=True)
        loss = model(x).float().pow(2).mean()
        loss.backward()
    torch.cuda.synchronize()
    return loss.detach(), (time.perf_counter() - t0) / reps


def full_params(model):
    """The all-gather outputs: every FSDP unit unsharded (bf16 params)."""
    out = []
    for blk in model:
        blk.unshard()
        out += [p.detach().clone() for p in blk.parameters()]
        blk.reshard()
    return out


def grads(model):
    return [p.grad.to_local().detach().clone() for p in model.parameters()]


def main() -> int:
    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    from paper_2504_18658_b200 import fsdp

    g = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn(4, 256, H, device=dev, generator=g, dtype=torch.bfloat16)
    failures = []

    ref = build(dev)
    step(ref, x, 2)  # warm-up (allocator, cuBLAS handles)
    _, t_ref = step(ref, x, REPS)
    loss_ref, _ = step(ref, x)
    g_ref = grads(ref)
    w_ref = full_params(ref)
    del ref
    torch.cuda.empty_cache()

    ours = build(dev)
    ag, rs = fsdp.install(ours, heap_bytes=3 << 30, algorithm=os.environ.get("PCCL_FSDP_ALGO", "auto"),
                          ag_ctas=int(os.environ.get("PCCL_FSDP_AG_CTAS", fsdp.AG_CTAS)),
                          rs_ctas=int(os.environ.get("PCCL_FSDP_RS_CTAS", fsdp.RS_CTAS)))
    step(ours, x, 2)
    _, t = step(ours, x, REPS)
    ag.world.set_param("staged_bytes", 0)
    rs.world.set_param("staged_bytes", 0)
    calls0 = (ag.calls, rs.calls)
    loss, _ = step(ours, x)
    calls = (ag.calls - calls0[0], rs.calls - calls0[1])
    g_ours = grads(ours)
    w_ours = full_params(ours)
    ag.world.check()
    rs.world.check()
    staged = ag.world.get_param("staged_bytes") + rs.world.get_param("staged_bytes")

    if not all(torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                           b.view(torch.int16) if b.dtype == torch.bfloat16 else b) for a, b in zip(w_ref, w_ours)):
        failures.append("all-gathered params differ from NCCL's")
    if not torch.equal(loss.view(torch.int32), loss_ref.view(torch.int32)):
        failures.append(f"loss {loss.item()} != NCCL's {loss_ref.item()}")
    worst = 0.0
    for a, b in zip(g_ours, g_ref):
        a32, b32 = a.float(), b.float()
        # both are p-way bf16 sums of the same local gradients, rounded at
        # different points: |a - b| <= 2 * p * 2^-8 * max|g| elementwise bound
        bound = 2 * p * 2.0 ** -8 * b32.abs().max().clamp_min(1e-30)
        err = (a32 - b32).abs().max()
        worst = max(worst, float(err / bound))
        if bool(err > bound):
            failures.append("reduce-scattered grads outside the bf16 bound")
            break
    if staged:
        failures.append(f"{staged} bytes went through staging")
    if calls[0] < 2 or calls[1] != 2:  # >= one AG per layer (forward; again in backward after resharding), one RS
        failures.append(f"B200 collectives issued per step (AG, RS) = {calls}")
    diff = sum(int((a.view(torch.int16) != b.view(torch.int16)).sum()) for a, b in zip(g_ours, g_ref))
    n_params = sum(w.numel() for w in w_ours)
    msg = (f"[rank {rank}] params {n_params} (2 x 12h^2+13h, h={H}) step NCCL {t_ref * 1e3:.1f} ms, "
           f"B200 {t * 1e3:.1f} ms, B200 collectives per step {calls}, staged {staged} B, grad err/bound {worst:.3f} "
           f"({diff} elements differ from NCCL's)")
    print(msg + (" OK" if not failures else " FAIL " + "; ".join(failures)), flush=True)
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
