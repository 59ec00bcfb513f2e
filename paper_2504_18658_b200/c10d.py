"""A ``torch.distributed`` backend on the B200 collectives.

    from paper_2504_18658_b200 import c10d            # registers backend "pccl" for CUDA tensors
    g = c10d.new_group()                              # collective, like any process group
    torch.distributed.all_gather_into_tensor(out, x, group=g)
    torch.distributed.reduce_scatter_tensor(y, grads, group=g)

Any ``torch.distributed`` user — FSDP1 (``process_group=g``), DeepSpeed-style
ZeRO-3 code, custom training loops — then runs its all-gathers and
reduce-scatters through the sm_100a kernels without code changes. The group's
World is bootstrapped through the process group's own c10d store (the IPC
handles travel as store keys), so it needs nothing besides the store.

Supported: ``all_gather_into_tensor`` / ``all_gather`` (list form),
``reduce_scatter_tensor`` / ``reduce_scatter`` (list form) with SUM / AVG,
``all_reduce`` (SUM / AVG, as reduce-scatter + all-gather), ``barrier``.
Collectives are stream-ordered on the caller's current stream, like NCCL's;
the returned Work is complete on return (its ``wait()`` has nothing left to
order). Everything else raises ``Unsupported``: run it on a NCCL group.
"""
from __future__ import annotations

import torch
import torch.distributed as dist
from torch._C._distributed_c10d import (
    AllgatherOptions,
    AllreduceOptions,
    BarrierOptions,
    ReduceScatterOptions,
    _create_work_from_future,
)

from .collectives import all_gather_into_tensor, reduce_scatter_tensor
from .communicator import Communicator
from .errors import Unsupported
from .world import World

BACKEND = "pccl"


def _done(result=None):
    fut = torch.futures.Future()
    fut.set_result(result)
    return _create_work_from_future(fut)


def _avg(op) -> bool:
    if op == dist.ReduceOp.SUM:
        return False
    if op == dist.ReduceOp.AVG:
        return True
    raise Unsupported(f"reduce op {op}: the B200 path reduces with SUM (and AVG = SUM / p)")


class PcclProcessGroup(dist.ProcessGroup):
    """Process group whose collectives are the B200 kernels."""

    def __init__(self, store, rank: int, size: int, timeout=None):
        super().__init__(rank, size)
        self._seq = 0

        def exchange(blob: bytes) -> list:
            k = self._seq
            self._seq += 1
            store.set(f"pccl/{k}/{rank}", blob)
            return [store.get(f"pccl/{k}/{q}") for q in range(size)]

        self.world = World.create(size, rank, torch.cuda.current_device(), exchange)
        self.world.ensure_staging(64 << 20)
        self.comm = Communicator(self.world, range(size), 0)

    def getBackendName(self) -> str:
        return BACKEND

    # ---- all-gather ---------------------------------------------------------
    def _allgather_base(self, output_tensor, input_tensor, opts=AllgatherOptions()):
        all_gather_into_tensor(output_tensor.view(-1), input_tensor.reshape(-1), self.comm)
        return _done(output_tensor)

    def allgather(self, output_tensors, input_tensor, opts=AllgatherOptions()):
        outs, inp = output_tensors[0], input_tensor[0]
        flat = torch.empty(inp.numel() * self.size(), dtype=inp.dtype, device=inp.device)
        all_gather_into_tensor(flat, inp.reshape(-1), self.comm)
        n = inp.numel()
        for q, o in enumerate(outs):
            o.copy_(flat[q * n:(q + 1) * n].view_as(o))
        return _done(output_tensors)

    def allgather_into_tensor_coalesced(self, outputs, inputs, opts=AllgatherOptions()):
        for o, i in zip(outputs, inputs):
            all_gather_into_tensor(o.view(-1), i.reshape(-1), self.comm)
        return _done(outputs)

    # ---- reduce-scatter -----------------------------------------------------
    def _reduce_scatter_base(self, output_tensor, input_tensor, opts=ReduceScatterOptions()):
        avg = _avg(opts.reduceOp)
        reduce_scatter_tensor(output_tensor.view(-1), input_tensor.reshape(-1), self.comm)
        if avg:
            output_tensor.div_(self.size())
        return _done(output_tensor)

    def reduce_scatter(self, output_tensors, input_tensors, opts=ReduceScatterOptions()):
        out = output_tensors[0]
        flat = torch.cat([x.reshape(-1) for x in input_tensors[0]])
        return self._reduce_scatter_base(out, flat, opts)

    def reduce_scatter_tensor_coalesced(self, outputs, inputs, opts=ReduceScatterOptions()):
        for o, i in zip(outputs, inputs):
            self._reduce_scatter_base(o, i, opts)
        return _done(outputs)

    # ---- all-reduce = reduce-scatter + all-gather ------------------------------
    def allreduce(self, tensors, opts=AllreduceOptions()):
        avg = _avg(opts.reduceOp)
        p = self.size()
        for t in tensors:
            flat = t.reshape(-1)
            n = (flat.numel() + p - 1) // p
            buf = torch.zeros(n * p, dtype=t.dtype, device=t.device)
            buf[: flat.numel()].copy_(flat)
            part = torch.empty(n, dtype=t.dtype, device=t.device)
            reduce_scatter_tensor(part, buf, self.comm)
            if avg:
                part.div_(p)
            all_gather_into_tensor(buf, part, self.comm)
            t.copy_(buf[: flat.numel()].view_as(t))
        return _done(tensors)

    def barrier(self, opts=BarrierOptions()):
        self.comm.barrier()
        return _done()

    def broadcast(self, *args, **kwargs):
        raise Unsupported("broadcast is not on the B200 collective path; use a NCCL group")


def _create(store, rank, size, timeout):
    return PcclProcessGroup(store, rank, size, timeout)


def new_group(ranks=None, **kwargs):
    """``torch.distributed.new_group(ranks, backend="pccl")``. A Python-defined
    process group cannot be eagerly bound to a device, which torch attempts
    when the default group was initialised with ``device_id``; the binding is
    suspended for the creation (plain ``dist.new_group(backend="pccl")`` works
    whenever the default group is not device-bound)."""
    default = dist.distributed_c10d._get_default_group()
    bound = default.bound_device_id
    default.bound_device_id = None
    try:
        return dist.new_group(ranks, backend=BACKEND, **kwargs)
    finally:
        default.bound_device_id = bound


if BACKEND not in dist.Backend.backend_list:
    dist.Backend.register_backend(BACKEND, _create, devices=["cuda"])
