"""FSDP2 / ZeRO-3 integration.

PyTorch's FSDP2 (``torch.distributed.fsdp.fully_shard``) exposes its two
collectives as pluggable objects (``FSDPModule.set_custom_all_gather`` /
``set_custom_reduce_scatter``, interfaces ``AllGather`` / ``ReduceScatter`` in
``torch/distributed/fsdp/_fully_shard/_fsdp_api.py``): an ``allocate()`` hook
for the communication buffers and a ``__call__`` that runs the collective on
the current stream. This module implements both with the B200 kernels:

* ``allocate()`` hands out tensors from a :class:`~.world.SymmetricHeap`
  (one symmetric arena, deterministic first-fit allocator): FSDP allocates the
  same sequence of buffers on every rank, so every all-gather output and
  reduce-scatter input sits at the same offset everywhere and the collectives
  run zero-copy — no staging copies (checked by the ``staged_bytes``
  statistic in ``tests/mp_fsdp.py``);
* ``__call__`` runs ``all_gather_into_tensor`` / ``reduce_scatter_tensor``
  (algorithm picked by the measured selector; the all-gather input is FSDP's
  slice of the output, which the kernels treat as in place);
* FSDP2 issues all-gathers and reduce-scatters on two different streams that
  overlap in the backward pass, and all collectives of one World must be
  stream-ordered, so the all-gather and the reduce-scatter each own a World
  (their own flag arena, staging and heap).

``ReduceOp.AVG`` (FSDP2's default for bf16 / fp32 gradients) is the SUM
reduce-scatter followed by a division by the group size on the same stream.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist
from torch.distributed.fsdp._fully_shard._fsdp_api import AllGather, ReduceScatter

from .collectives import all_gather_into_tensor, reduce_scatter_tensor
from .communicator import init_from_torch
from .errors import Unsupported

DEFAULT_HEAP_BYTES = 4 << 30
AG_CTAS = 32  # CTAs per collective inside FSDP (profiles/r2_fsdp2_p4.txt: 128 -> 32/64 cuts the step 6.8 -> 5.9 ms)
RS_CTAS = 64


class _SymmetricComm:
    def __init__(self, group=None, heap_bytes: int = DEFAULT_HEAP_BYTES, algorithm: str = "auto",
                 staging_bytes: int = 64 << 20, ctas: int = 0):
        self.comm = init_from_torch(group, staging_bytes=staging_bytes)  # collective over the group
        self.heap = self.comm.world.heap(heap_bytes)                      # collective
        self.algorithm = algorithm
        if ctas:  # CTAs per collective: FSDP overlaps the collectives with GEMMs competing for the SMs
            self.comm.world.set_param("ctas", ctas)
        self.calls = 0  # collectives issued through this object
        self.bytes = 0  # all-gather output / reduce-scatter input bytes moved

    def allocate(self, size, *, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
        numel = math.prod(int(s) for s in size)
        if device.type != "cuda" or (device.index is not None and device.index != self.comm.world.device):
            raise Unsupported(f"symmetric heap lives on cuda:{self.comm.world.device}, asked for {device}")
        return self.heap.empty(numel, dtype).view(*[int(s) for s in size])

    @property
    def world(self):
        return self.comm.world

    def close(self) -> None:
        self.comm.world.close()


class PcclAllGather(_SymmetricComm, AllGather):
    """FSDP2 all-gather on the B200 kernels (zero-copy on heap buffers)."""

    def __call__(self, output_tensor: torch.Tensor, input_tensor: torch.Tensor, group: dist.ProcessGroup,
                 async_op: bool = False):
        all_gather_into_tensor(output_tensor.view(-1), input_tensor.view(-1), self.comm, algorithm=self.algorithm)
        self.calls += 1
        self.bytes += output_tensor.numel() * output_tensor.element_size()
        return None  # stream-ordered: FSDP records its event after this call


class PcclReduceScatter(_SymmetricComm, ReduceScatter):
    """FSDP2 reduce-scatter on the B200 kernels (SUM; AVG = SUM / p)."""

    def __call__(self, output_tensor: torch.Tensor, input_tensor: torch.Tensor, group: dist.ProcessGroup,
                 op=dist.ReduceOp.SUM, async_op: bool = False):
        if op == dist.ReduceOp.SUM:
            avg = False
        elif op == dist.ReduceOp.AVG:
            avg = True
        else:
            raise Unsupported(f"reduce-scatter op {op} (SUM / AVG only; FSDPModule."
                              "set_force_sum_reduction_for_comms(True) selects SUM)")
        reduce_scatter_tensor(output_tensor.view(-1), input_tensor.view(-1), self.comm, algorithm=self.algorithm)
        self.calls += 1
        self.bytes += input_tensor.numel() * input_tensor.element_size()
        if avg:
            output_tensor.div_(self.comm.size)
        return None


def install(module, group=None, *, heap_bytes: int = DEFAULT_HEAP_BYTES, algorithm: str = "auto",
            ag_ctas: int = AG_CTAS, rs_ctas: int = RS_CTAS):
    """Route every FSDP2 module under ``module`` through the B200 collectives.
    Collective over ``group`` (default: the world). ``ag_ctas`` / ``rs_ctas``:
    CTAs per all-gather / reduce-scatter launch (0 = the library's automatic
    choice, tuned for a collective running alone; FSDP overlaps them with the
    GEMMs, which want the SMs). Returns the (all_gather, reduce_scatter) comm
    objects (their worlds' ``staged_bytes`` statistic shows whether any
    buffer had to be staged)."""
    from torch.distributed.fsdp import FSDPModule

    ag = PcclAllGather(group, heap_bytes=heap_bytes, algorithm=algorithm, ctas=ag_ctas)
    rs = PcclReduceScatter(group, heap_bytes=heap_bytes, algorithm=algorithm, ctas=rs_ctas)
    n = 0
    for m in module.modules():
        if isinstance(m, FSDPModule):
            m.set_custom_all_gather(ag)
            m.set_custom_reduce_scatter(rs)
            n += 1
    if n == 0:
        raise ValueError("install: no FSDPModule found (call fully_shard first)")
    return ag, rs
