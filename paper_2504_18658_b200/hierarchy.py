"""Two-level (virtual-node) all-gather / reduce-scatter, drop-in for
``collkit/hierarchy.py``.

The paper's hierarchy (inter-node phase on the stride-M groups, intra-node
ring, device-local shuffle; reduce-scatter mirrored) is mapped onto one
NVSwitch box as N virtual nodes of M GPUs. Both phases are sm_100a kernels
over NVLink peer memory; the device-local block transpose is *fused into the
addressing* — the inter phase writes every gathered block straight to its
global position and the intra phase moves strided block sets — so no separate
shuffle pass touches HBM (``shuffle_*`` remain available as standalone GPU
kernels for callers that need them). Reduction order equals the reference's:
outer {ring | butterfly over nodes} of an inner ring over local ranks.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr_array
from .collectives import (
    _In,
    _align,
    _ensure_io,
    _download,
    _finish,
    _stream,
    as_elements,
    is_power_of_two,
)
from .errors import LengthMismatch, NonPowerOfTwo, NotDivisible
from .selector import CalibrationTable, CostParams, choose_inter_algorithm
from .topology import Topology
from .world import TORCH_DTYPES

INTER_ALGORITHMS = ("ring", "recursive", "auto")


def inter_comm_id(topo: Topology, local_rank: int) -> int:
    """hierarchy.py:31-34: world 0, inter-node group j is 1 + j."""
    return 1 + local_rank


def intra_comm_id(topo: Topology, node: int) -> int:
    """hierarchy.py:37-38: intra-node group n is 1 + M + n."""
    return 1 + topo.gpus_per_node + node


@dataclass(frozen=True)
class BlockLayout:
    block_count: int
    block_len: int
    ordering: str

    def __post_init__(self) -> None:
        if self.ordering not in ("global_rank_major", "local_major"):
            raise ValueError(f"unknown ordering {self.ordering!r}")

    @property
    def total_elems(self) -> int:
        return self.block_count * self.block_len


@dataclass(frozen=True)
class HierPlan:
    """Configuration of one hierarchical collective (hierarchy.py:60-100)."""

    topo: Topology
    inter_alg: str = "auto"
    collective: str | None = None
    params: CostParams = field(default_factory=CostParams)
    selector_mode: str = "analytic"
    table: CalibrationTable | None = None

    def __post_init__(self) -> None:
        if self.inter_alg not in INTER_ALGORITHMS:
            raise ValueError(f"inter_alg must be one of {INTER_ALGORITHMS}")
        if self.collective not in (None, "all_gather", "reduce_scatter"):
            raise ValueError(f"unknown collective {self.collective!r}")
        if self.inter_alg == "recursive" and not is_power_of_two(self.topo.num_nodes):
            raise NonPowerOfTwo(f"recursive inter-node algorithm requires a power-of-two node count, "
                                f"got {self.topo.num_nodes}")

    def resolve_inter(self, sub_m_bytes: int) -> str:
        if self.inter_alg != "auto":
            return self.inter_alg
        if self.topo.num_nodes < 2:
            return "ring"
        return choose_inter_algorithm(self.topo.num_nodes, sub_m_bytes, self.params,
                                      mode=self.selector_mode, table=self.table)


# ---------------------------------------------------------------------------
# standalone shuffles (GPU block transpose)
# ---------------------------------------------------------------------------
def _shuffle(direction: int, buf, num_nodes: int, gpus_per_node: int, block_len: int):
    is_tensor = isinstance(buf, torch.Tensor)
    expected = num_nodes * gpus_per_node * block_len
    numel = buf.numel() if is_tensor else as_elements(buf).size
    if numel != expected:
        raise LengthMismatch(f"buffer has {numel} elements, expected {expected}")
    dev = buf.device if is_tensor and buf.is_cuda else torch.device("cuda", torch.cuda.current_device())
    if is_tensor:
        src = buf.reshape(-1).contiguous().to(dev)
    else:
        src = torch.from_numpy(as_elements(buf)).to(dev)
    out = torch.empty_like(src)
    code = _lib.DTYPES.get(TORCH_DTYPES.get(src.dtype, "u8"))
    n_blk = block_len
    if src.dtype not in TORCH_DTYPES:
        src, out = src.view(torch.uint8), out.view(torch.uint8)
        n_blk = block_len * buf.element_size()
        code = _lib.DTYPES["u8"]
    if expected:
        check(lib().pccl_shuffle(direction, src.data_ptr(), out.data_ptr(), num_nodes, gpus_per_node, n_blk, code,
                                 _stream(dev)), "shuffle")
    if is_tensor:
        return out.view(buf.dtype) if buf.is_cuda else out.view(buf.dtype).cpu()
    return out.cpu().numpy()


def shuffle_local_major_to_global(buf, num_nodes: int, gpus_per_node: int, block_len: int):
    """Out-of-place M x N -> N x M block transpose (hierarchy.py:103-114)."""
    return _shuffle(0, buf, num_nodes, gpus_per_node, block_len)


def shuffle_global_to_local_major(buf, num_nodes: int, gpus_per_node: int, block_len: int):
    """Exact inverse (hierarchy.py:117-126)."""
    return _shuffle(1, buf, num_nodes, gpus_per_node, block_len)


# ---------------------------------------------------------------------------
# hierarchical collectives
# ---------------------------------------------------------------------------
def _check_world(plan: HierPlan, comm):
    """hierarchy.py:129-134: the communicator's size must match the topology
    (any communicator: topology rank g is its member g)."""
    topo = plan.topo
    if comm.size != topo.world_size:
        raise LengthMismatch(f"communicator size {comm.size} != topology world {topo.world_size}")


def _hier(plan: HierPlan, comm, buf, reduce: bool, out=None):
    topo = plan.topo
    N, M = topo.num_nodes, topo.gpus_per_node
    arg = _In(buf, reduce, comm.device, out)
    p = topo.world_size
    es = arg.t.element_size()
    if reduce:
        if arg.t.numel() % p:
            raise NotDivisible(f"input of {arg.t.numel()} elements not divisible by p={p}")
        n = arg.t.numel() // p
        out_numel = n
        alg = plan.resolve_inter(N * n * es)
    else:
        n = arg.t.numel()
        out_numel = n * p
        alg = plan.resolve_inter(N * n * es)
    inter = _lib.ALGOS[alg]
    dtype = _lib.DTYPES[TORCH_DTYPES.get(arg.t.dtype, "u8")]

    def execute(args: list):
        emu = comm.emulated
        ranks = list(comm.members) if emu else [comm.world_rank]
        sizes = [a.t.numel() for a in args]
        if len(set(sizes)) > 1:
            raise LengthMismatch(f"buffer sizes differ across ranks: {sizes}")
        world = comm.world
        need = int(lib().pccl_staging_bytes(_lib.REDUCE_SCATTER if reduce else _lib.ALL_GATHER, 3, p, n, dtype))
        if world.staging is None or world.staging.nbytes < need:
            world.ensure_staging(need)
        if all(a.host for a in args):
            in_bytes = args[0].nbytes
            io = _ensure_io(comm, _align(in_bytes) + _align(out_numel * es))
            sends, recvs = [], []
            for a, r in zip(args, ranks):
                dst = io.tensor(r, 0, a.nbytes)
                if a.nbytes:
                    src = a.t.view(torch.uint8).reshape(-1)
                    dst.copy_(src, non_blocking=src.is_pinned())
                sends.append(dst.view(a.t.dtype))
                recvs.append(io.tensor(r, _align(in_bytes), out_numel * es).view(a.t.dtype))
        else:
            sends = [a.t.to(comm.device) for a in args]
            recvs = [a.out.reshape(-1) if a.out is not None else
                     torch.empty(out_numel, dtype=sends[0].dtype, device=comm.device) for a in args]
        stream = _stream(comm.device)
        if emu:
            fn = lib().pccl_emu_hier_reduce_scatter_comm if reduce else lib().pccl_emu_hier_all_gather_comm
            st = fn(comm.handle, N, M, inter, ptr_array([t.data_ptr() for t in sends]),
                    ptr_array([t.data_ptr() for t in recvs]), n, dtype, stream)
        else:
            fn = lib().pccl_hier_reduce_scatter_comm if reduce else lib().pccl_hier_all_gather_comm
            st = fn(comm.handle, N, M, inter, sends[0].data_ptr(), recvs[0].data_ptr(), n, dtype, stream)
        check(st, "hier_reduce_scatter" if reduce else "hier_all_gather")
        host = _download([rv for a, rv in zip(args, recvs) if a.host])
        if emu and not host:
            torch.cuda.current_stream(comm.device).synchronize()
        if emu or host:
            world.check()
        res, hi = [], 0
        for a, rv in zip(args, recvs):
            if a.host:
                res.append(_finish(a, host[hi]))
                hi += 1
            else:
                res.append(rv if a.out is None else a.out)
        return res

    if comm.emulated:
        return comm._rendezvous(arg, execute)
    comm.next_base_tag()
    return execute([arg])[0]


def hier_all_gather(plan: HierPlan, comm_world, buf, *, out=None):
    """Hierarchical all-gather (hierarchy.py:158-173); output identical to a
    flat all-gather on the world communicator."""
    if plan.collective == "reduce_scatter":
        raise ValueError("plan is configured for reduce_scatter")
    _check_world(plan, comm_world)
    return _hier(plan, comm_world, buf, False, out)


def hier_reduce_scatter(plan: HierPlan, comm_world, buf, *, out=None):
    """Hierarchical reduce-scatter (hierarchy.py:176-195)."""
    if plan.collective == "all_gather":
        raise ValueError("plan is configured for all_gather")
    _check_world(plan, comm_world)
    return _hier(plan, comm_world, buf, True, out)
