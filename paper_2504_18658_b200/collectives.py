"""Flat all-gather / reduce-scatter, drop-in for ``collkit/collectives.py``.

Same names, arguments and semantics as the reference:

* ``ring_all_gather(comm, buf)`` (collectives.py:55-76), ``recdbl_all_gather``
  (:107-129), ``ring_reduce_scatter`` (:79-104), ``rechalf_reduce_scatter``
  (:132-165); plus the one-shot ``direct_all_gather`` /
  ``direct_reduce_scatter`` and the dispatching
  ``all_gather`` / ``reduce_scatter``;
* SPMD, blocking for host inputs, output is a fresh array the caller owns, the
  input is never modified; numpy input is cast to contiguous 1-D float32
  exactly like ``as_elements`` (collectives.py:26-29);
* errors: ``NotDivisible``, ``NonPowerOfTwo``, ``LengthMismatch`` (also across
  ranks), ``Timeout``.

What differs is underneath: buffers live in HBM, peers' symmetric buffers are
read over NVLink by the sm_100a kernels in ``csrc/kernels.cuh``, and the
reduction is fused into the peer-load loop. CUDA tensors (fp32 / bf16 / fp16)
are accepted natively and stay on the device (stream-ordered, no host sync);
pass ``out=`` a tensor from ``comm.world.empty`` to skip every staging copy.
"""
from __future__ import annotations

import enum
import math
import os

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, ptr_array
from .errors import LengthMismatch, NonPowerOfTwo, NotDivisible, OutOfMemory, Unsupported
from .world import TORCH_DTYPES


class ReduceOp(enum.Enum):
    SUM = "sum"


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def as_elements(buf) -> np.ndarray:
    """Contiguous 1-D float32 view/copy (collectives.py:26-29)."""
    return np.ascontiguousarray(buf, dtype=np.float32).reshape(-1)


ALL_GATHER_ALGOS = ("direct", "ring", "recursive")
REDUCE_SCATTER_ALGOS = ("direct", "ring", "recursive")


def _align(n: int) -> int:
    return (n + 255) & ~255


try:  # raw handle of the current stream without building a Stream object
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover
    _raw_stream = None


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _stream_of(t: torch.Tensor) -> int:
    if _raw_stream is not None:
        return _raw_stream(t.get_device())
    return torch.cuda.current_stream(t.device).cuda_stream


# ---------------------------------------------------------------------------
# input normalisation
# ---------------------------------------------------------------------------
class _In:
    """One rank's argument: a flat CUDA tensor to run on, plus how to return."""

    __slots__ = ("t", "host", "numpy", "out")

    def __init__(self, buf, reduce: bool, device: torch.device, out=None):
        self.out = out
        if isinstance(buf, torch.Tensor):
            t = buf.reshape(-1)
            if not t.is_contiguous():
                t = t.contiguous()
            if reduce and t.dtype not in (torch.float32, torch.bfloat16, torch.float16):
                t = t.to(torch.float32)
            if not reduce and t.dtype not in TORCH_DTYPES:
                raise Unsupported(f"dtype {t.dtype} not supported")
            self.host = not t.is_cuda
            self.numpy = False
            self.t = t
        else:
            arr = as_elements(buf)
            self.host = True
            self.numpy = True
            self.t = torch.from_numpy(arr)

    @property
    def dtype_code(self) -> int:
        return _lib.DTYPES[TORCH_DTYPES[self.t.dtype]]

    @property
    def nbytes(self) -> int:
        return self.t.numel() * self.t.element_size()


def _download(results: list) -> list:
    """Device results -> fresh pinned host tensors, one sync for all."""
    outs = []
    for r in results:
        h = torch.empty(r.shape, dtype=r.dtype, pin_memory=True)
        h.copy_(r, non_blocking=True)
        outs.append(h)
    if results:
        torch.cuda.current_stream(results[0].device).synchronize()
    return outs


def _finish(arg: _In, host: torch.Tensor):
    """Return in the caller's type: numpy for numpy input, host tensor for a
    host tensor (fresh, caller-owned)."""
    return host.numpy() if arg.numpy else host


def _check_world_size_growth(comm, need: int, what: str):
    """Segments grow collectively: only a world-sized call (every rank
    present) may grow them in real mode; emulated worlds grow locally."""
    world = comm.world
    if comm.size == world.nranks or world.emulated:
        return True
    seg = world.staging if what == "staging" else world.io
    if seg is None or seg.nbytes < need:
        raise OutOfMemory(
            f"sub-communicator call needs {need} B of {what}; grow it collectively first "
            f"(world.ensure_{what}({need}) on every rank)"
        )
    return False


def _ensure_staging(comm, collective: int, algo: int, count: int, dtype_code: int):
    need = int(lib().pccl_staging_bytes(collective, algo, comm.size, count, dtype_code))
    world = comm.world
    if world.staging is not None and world.staging.nbytes >= need:
        return
    if _check_world_size_growth(comm, need, "staging"):
        world.ensure_staging(need)


def _ensure_io(comm, need: int):
    world = comm.world
    if world.io is not None and world.io.nbytes >= need:
        return world.io
    if _check_world_size_growth(comm, need, "io"):
        return world.ensure_io(need)
    return world.io


# ---------------------------------------------------------------------------
# device execution (shared by real and emulated mode)
# ---------------------------------------------------------------------------
def _all_gather_device(comm, algo: str, sends: list, recvs: list, emu: bool) -> None:
    """sends/recvs: one CUDA tensor per executed rank (real: [mine])."""
    a = _lib.ALGOS[algo]
    s0 = sends[0]
    dtype = _lib.DTYPES[TORCH_DTYPES.get(s0.dtype, "u8")]
    count = s0.numel() if s0.dtype in TORCH_DTYPES else s0.numel() * s0.element_size()
    _ensure_staging(comm, _lib.ALL_GATHER, a, count, dtype)
    stream = _stream(comm.device)
    if emu:
        st = lib().pccl_emu_all_gather(comm.handle, a, ptr_array([t.data_ptr() for t in sends]),
                                       ptr_array([t.data_ptr() for t in recvs]), count, dtype, stream)
    else:
        st = lib().pccl_all_gather(comm.handle, a, sends[0].data_ptr(), recvs[0].data_ptr(), count, dtype, stream)
    check(st, f"all_gather[{algo}]")


def _reduce_scatter_device(comm, algo: str, order: str, sends: list, recvs: list, emu: bool) -> None:
    a = _lib.ALGOS[algo]
    o = _lib.ORDERS[order]
    s0 = sends[0]
    dtype = _lib.DTYPES[TORCH_DTYPES[s0.dtype]]
    n = s0.numel() // comm.size
    _ensure_staging(comm, _lib.REDUCE_SCATTER, a, n, dtype)
    stream = _stream(comm.device)
    if emu:
        st = lib().pccl_emu_reduce_scatter(comm.handle, a, o, ptr_array([t.data_ptr() for t in sends]),
                                           ptr_array([t.data_ptr() for t in recvs]), n, dtype, stream)
    else:
        st = lib().pccl_reduce_scatter(comm.handle, a, o, sends[0].data_ptr(), recvs[0].data_ptr(), n, dtype, stream)
    check(st, f"reduce_scatter[{algo}]")


def _upload(comm, args: list, ranks: list, out_bytes: int):
    """Host inputs -> each rank's io segment (input, then output region)."""
    in_bytes = max(a.nbytes for a in args)
    io = _ensure_io(comm, _align(in_bytes) + _align(out_bytes))
    sends, recvs = [], []
    for a, r in zip(args, ranks):
        dst = io.tensor(r, 0, a.nbytes)
        if a.nbytes:
            src = a.t.view(torch.uint8).reshape(-1)
            dst.copy_(src, non_blocking=src.is_pinned())
        sends.append(dst.view(a.t.dtype))
        recvs.append(io.tensor(r, _align(in_bytes), out_bytes).view(a.t.dtype))
    return sends, recvs


# Pipelined host path: host buffers of at least PIPE_MIN_BYTES per rank
# are moved in slices (one slice of every chunk / block per collective call),
# so the H2D copy of slice k+1 and the D2H copy of slice k-1 run on the copy
# engines while the collective of slice k runs. Elementwise the slices
# compute exactly what the whole call computes (same algorithm, same order).
PIPE_MIN_BYTES = int(os.environ.get("PCCL_PIPE_MIN_BYTES", 8 << 20))
PIPE_SLICE_BYTES = int(os.environ.get("PCCL_PIPE_SLICE_BYTES", 8 << 20))
PIPE_MAX_SLICES = 16
_PIPE_BUFS = 3
_side_streams: dict = {}


def _pipe_streams(device: torch.device):
    key = device.index
    if key not in _side_streams:
        _side_streams[key] = (torch.cuda.Stream(device), torch.cuda.Stream(device))
    return _side_streams[key]


def _pipeline_slices(row_len: int, es: int, in_bytes: int):
    """[(offset, length)] in elements over one row (chunk or block), or None
    when the call is too small to gain from pipelining."""
    if in_bytes < PIPE_MIN_BYTES or row_len == 0:
        return None
    k = max(2, min(PIPE_MAX_SLICES, in_bytes // PIPE_SLICE_BYTES))
    grain = max(1, 256 // es)  # slices start 256-byte aligned (vector path)
    cs = -(-row_len // k)
    cs = -(-cs // grain) * grain
    out = [(off, min(cs, row_len - off)) for off in range(0, row_len, cs)]
    return out if len(out) >= 2 else None


def _host_pipeline(comm, args: list, ranks: list, reduce: bool, algo: str, order: str, out_numel: int, emu: bool):
    """Host inputs -> fresh pinned host outputs through the io segment in slices.

    RS: rank r's input is p chunks of L elements; slice (off, ln) uploads
    column range [off, off+ln) of every chunk (one strided copy) into a
    contiguous p x ln send buffer, reduce-scatters it (count ln) and downloads
    the ln results to out[off:off+ln]. AG mirrors it: ln input elements
    up, a p x ln gathered slice down into column range [off, off+ln) of the
    p blocks. Buffer reuse is event-ordered: slice k's upload waits for the
    collective of slice k-3 (pull kernels exit only after every peer finished
    reading the send buffer), and slice k's collective waits for the download
    of slice k-3 (its peers may write into the receive buffer as soon as it
    starts). The decision depends only on sizes, so it is SPMD-uniform (pageable
inputs are correct too; their uploads are just not asynchronous). Returns
None when the call is too small to gain."""
    t0 = args[0].t
    es = t0.element_size()
    p = comm.size
    row_len = t0.numel() // p if reduce else t0.numel()
    slices = _pipeline_slices(row_len, es, t0.numel() * es)
    if slices is None:
        return None
    cs = slices[0][1]
    in_sl = (p * cs if reduce else cs) * es
    out_sl = (cs if reduce else p * cs) * es
    per_buf = _align(in_sl) + _align(out_sl)
    io = _ensure_io(comm, _PIPE_BUFS * per_buf)
    if io is None or io.nbytes < _PIPE_BUFS * per_buf:
        return None
    dev = comm.device
    cur = torch.cuda.current_stream(dev)
    up, down = _pipe_streams(dev)
    outs = [torch.empty(out_numel, dtype=t0.dtype, pin_memory=True) for _ in args]
    bases = {r: io.tensor(r, 0, _PIPE_BUFS * per_buf) for r in ranks}
    L = lib()
    ev_comp, ev_down = [], []
    up.wait_stream(cur)
    down.wait_stream(cur)
    for k, (off, ln) in enumerate(slices):
        b = k % _PIPE_BUFS
        sends, recvs = [], []
        for r in ranks:
            base = bases[r]
            sends.append(base[b * per_buf: b * per_buf + (p * ln if reduce else ln) * es].view(t0.dtype))
            ob = b * per_buf + _align(in_sl)
            recvs.append(base[ob: ob + (ln if reduce else p * ln) * es].view(t0.dtype))
        with torch.cuda.stream(up):
            if k >= _PIPE_BUFS:
                up.wait_event(ev_comp[k - _PIPE_BUFS])
            for a, snd in zip(args, sends):
                src = a.t.data_ptr() + off * es
                if reduce:  # column range of every chunk -> p x ln
                    st = L.pccl_copy2d(snd.data_ptr(), ln * es, src, row_len * es, ln * es, p, up.cuda_stream)
                else:
                    st = L.pccl_copy2d(snd.data_ptr(), ln * es, src, ln * es, ln * es, 1, up.cuda_stream)
                check(st, "copy2d (upload)")
            ev_up = torch.cuda.Event()
            ev_up.record(up)
        cur.wait_event(ev_up)
        if k >= _PIPE_BUFS:
            cur.wait_event(ev_down[k - _PIPE_BUFS])
        if reduce:
            _reduce_scatter_device(comm, algo, order, sends, recvs, emu)
        else:
            _all_gather_device(comm, algo, sends, recvs, emu)
        ev = torch.cuda.Event()
        ev.record(cur)
        ev_comp.append(ev)
        with torch.cuda.stream(down):
            down.wait_event(ev)
            for o, rcv in zip(outs, recvs):
                dst = o.data_ptr() + off * es
                if reduce:
                    st = L.pccl_copy2d(dst, ln * es, rcv.data_ptr(), ln * es, ln * es, 1, down.cuda_stream)
                else:  # p x ln gathered slice -> column range of every block
                    st = L.pccl_copy2d(dst, row_len * es, rcv.data_ptr(), ln * es, ln * es, p, down.cuda_stream)
                check(st, "copy2d (download)")
            evd = torch.cuda.Event()
            evd.record(down)
            ev_down.append(evd)
    cur.wait_stream(down)
    cur.wait_stream(up)
    cur.synchronize()
    return outs


_REDUCE_DTYPES = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}


def _fast_device(comm, buf, reduce: bool, algo: str, order: str, out):
    """Real mode with contiguous CUDA tensors: validate and go straight to the
    C ABI (stream-ordered, no host sync, ~7 us of host time per call instead
    of ~20). Returns None when the general path must handle the call."""
    if comm.emulated or type(buf) is not torch.Tensor or not buf.is_cuda or not buf.is_contiguous():
        return None
    if reduce:
        code = _REDUCE_DTYPES.get(buf.dtype)
    else:
        name = TORCH_DTYPES.get(buf.dtype)
        code = None if name is None else _lib.DTYPES[name]
    if code is None or (out is not None and (type(out) is not torch.Tensor or not out.is_cuda
                                             or not out.is_contiguous() or out.dtype != buf.dtype)):
        return None
    p = comm.size
    n = buf.numel()
    pow2 = p & (p - 1) == 0
    if reduce:
        if n % p:
            raise NotDivisible(f"input of {n} elements not divisible by p={p}")
        if (algo == "recursive" or (algo == "direct" and order.startswith("recursive"))) and not pow2:
            raise NonPowerOfTwo(f"recursive algorithms require power-of-two ranks, got {p}")
        cnt = n // p
        out_numel = cnt
    else:
        if algo == "recursive" and not pow2:
            raise NonPowerOfTwo(f"recursive doubling requires power-of-two ranks, got {p}")
        cnt = n
        out_numel = n * p
    if out is None:
        out = torch.empty(out_numel, dtype=buf.dtype, device=buf.device)
    elif out.numel() != out_numel:
        raise LengthMismatch(f"output has {out.numel()} elements, expected {out_numel}")
    a = _lib.ALGOS[algo]
    comm.next_base_tag()
    key = (reduce, a, cnt, code)
    need = comm._stage_need.get(key)
    if need is None:
        need = int(lib().pccl_staging_bytes(1 if reduce else 0, a, p, cnt, code))
        comm._stage_need[key] = need
    st = comm.world.staging
    if (st is None or st.nbytes < need) and _check_world_size_growth(comm, need, "staging"):
        comm.world.ensure_staging(need)
    stream = _stream_of(buf)
    L = lib()
    if reduce:
        status = L.pccl_reduce_scatter(comm.handle, a, _lib.ORDERS[order], buf.data_ptr(), out.data_ptr(), cnt, code,
                                       stream)
    else:
        status = L.pccl_all_gather(comm.handle, a, buf.data_ptr(), out.data_ptr(), cnt, code, stream)
    if status:
        check(status, f"{'reduce_scatter' if reduce else 'all_gather'}[{algo}]")
    return out


def _run(comm, buf, reduce: bool, algo: str, order: str, out=None):
    """One rank's call (real) or rendezvous into one launch (emulated)."""
    fast = _fast_device(comm, buf, reduce, algo, order, out)
    if fast is not None:
        return fast
    arg = _In(buf, reduce, comm.device, out)
    p = comm.size
    if reduce:
        if arg.t.numel() % p:
            raise NotDivisible(f"input of {arg.t.numel()} elements not divisible by p={p}")
        if algo == "recursive" and not is_power_of_two(p):
            raise NonPowerOfTwo(f"recursive halving requires power-of-two ranks, got {p}")
        if algo == "direct" and order.startswith("recursive") and not is_power_of_two(p):
            raise NonPowerOfTwo(f"recursive order requires power-of-two ranks, got {p}")
    elif algo == "recursive" and not is_power_of_two(p):
        raise NonPowerOfTwo(f"recursive doubling requires power-of-two ranks, got {p}")
    out_numel = arg.t.numel() // p if reduce else arg.t.numel() * p

    def execute(args: list):
        emu = comm.emulated
        ranks = list(comm.members) if emu else [comm.world_rank]
        sizes = [a.t.numel() for a in args]
        if len(set(sizes)) > 1 or len({a.t.dtype for a in args}) > 1:
            raise LengthMismatch(f"buffer sizes/dtypes differ across ranks: {sizes}")
        if all(a.host for a in args):
            piped = _host_pipeline(comm, args, ranks, reduce, algo, order, out_numel, emu)
            if piped is not None:
                comm.world.check()
                return [_finish(a, h) for a, h in zip(args, piped)]
        if all(a.host for a in args):
            es = args[0].t.element_size()
            sends, recvs = _upload(comm, args, ranks, out_numel * es)
        else:
            sends = [a.t if not a.host else a.t.to(comm.device) for a in args]
            recvs = [a.out.reshape(-1) if a.out is not None else
                     torch.empty(out_numel, dtype=sends[0].dtype, device=comm.device) for a in args]
        if reduce:
            _reduce_scatter_device(comm, algo, order, sends, recvs, emu)
        else:
            _all_gather_device(comm, algo, sends, recvs, emu)
        host = _download([rv for a, rv in zip(args, recvs) if a.host])
        if emu and not host:
            torch.cuda.current_stream(comm.device).synchronize()
        if emu or host:
            comm.world.check()
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


# ---------------------------------------------------------------------------
# public API (reference names)
# ---------------------------------------------------------------------------
def ring_all_gather(comm, buf, *, out=None):
    """Ring all-gather: p-1 neighbour steps (collectives.py:55-76)."""
    return _run(comm, buf, False, "ring", "ring", out)


def recdbl_all_gather(comm, buf, *, out=None):
    """Recursive-doubling all-gather: log2 p partner steps (collectives.py:107-129)."""
    return _run(comm, buf, False, "recursive", "ring", out)


def direct_all_gather(comm, buf, *, out=None):
    """One-shot all-gather: every rank pulls every peer's block in one step."""
    return _run(comm, buf, False, "direct", "ring", out)


def ring_reduce_scatter(comm, buf, *, out=None):
    """Ring reduce-scatter with the add fused into the peer load (collectives.py:79-104)."""
    return _run(comm, buf, True, "ring", "ring", out)


def rechalf_reduce_scatter(comm, buf, *, out=None):
    """Recursive-halving reduce-scatter, fused add (collectives.py:132-165)."""
    return _run(comm, buf, True, "recursive", "ring", out)


def direct_reduce_scatter(comm, buf, *, order: str = "ring", out=None):
    """One-shot reduce-scatter: chunk r pulled from every peer and folded in
    fp32 in ``order`` ("ring" | "recursive" | "rank"), which makes fp32 results
    bit-identical to the named step-wise algorithm; bf16 / fp16 are rounded
    once. "ring/wire" / "recursive/wire" also round after every add, where the
    step-wise algorithm stores its partials: bit-identical to it for every
    dtype (what ``reduce_scatter(algorithm="auto")`` uses)."""
    if order not in _lib.ORDERS:
        raise ValueError(f"unknown order {order!r}")
    return _run(comm, buf, True, "direct", order, out)


def _resolve_auto(comm, collective: str, m_bytes: int, order: str | None = None) -> str:
    """``auto``: the measured winner for (collective, p, size). Real mode
    first calibrates the live world when the table has nothing within 8x of
    this size at this GPU count (``tuning.autotune``, SPMD-uniform: the table
    and the call are the same on every rank, so every rank measures the same
    candidates and agrees on the result). Emulated ranks (no NVLink to
    measure) and calls under CUDA-graph capture use the table as it is, with
    the one-shot ``direct`` when it has nothing for this p."""
    from . import selector, tuning

    p = comm.size
    if p > 1 and not comm.emulated and not torch.cuda.is_current_stream_capturing():
        t = selector.flat_table()
        have = [e.m_bytes for e in (t.entries if t else []) if e.collective == collective and e.p == p]
        # calibration size: this size's power-of-two bucket, clamped to 1-256 MiB
        m = 1 << max(20, min(28, (max(m_bytes, 1) - 1).bit_length()))
        m = max(16 * p * 4, m // (16 * p * 4) * (16 * p * 4))  # whole 16-byte units per rank, any dtype
        if not have or min(abs(math.log2(m / h)) for h in have) > 3:
            tuning.autotune(comm, collective, m, dtype=torch.float32 if collective == "all_gather" else torch.bfloat16)
    return selector.choose_algorithm(collective, p, m_bytes, order)


def all_gather(comm, buf, *, algorithm: str = "auto", out=None):
    """Dispatching all-gather; ``auto`` picks from the measured selector."""
    if algorithm == "auto":
        algorithm = _resolve_auto(comm, "all_gather", _nbytes(buf) * comm.size)
    if algorithm not in ALL_GATHER_ALGOS:
        raise Unsupported(f"unknown all-gather algorithm {algorithm!r}")
    return _run(comm, buf, False, algorithm, "ring", out)


def reduce_scatter(comm, buf, *, algorithm: str = "auto", order: str = "ring", out=None):
    """Dispatching reduce-scatter; ``auto`` picks from the measured selector."""
    if algorithm == "auto":  # the data movement is measured; the add order is pinned by `order`
        algorithm = _resolve_auto(comm, "reduce_scatter", _nbytes(buf), order)
        if algorithm == "direct" and order in ("ring", "recursive"):
            # and so are the rounding points: the one-step kernel rounds where
            # the step-wise algorithm would, so auto's result never depends on
            # which data movement won (bit-identical for every dtype)
            order = order + "/wire"
    if algorithm not in REDUCE_SCATTER_ALGOS:
        raise Unsupported(f"unknown reduce-scatter algorithm {algorithm!r}")
    return _run(comm, buf, True, algorithm, order, out)


def _nbytes(buf) -> int:
    if isinstance(buf, torch.Tensor):
        return buf.numel() * buf.element_size()
    return as_elements(buf).nbytes


def reduce_inplace(acc, other, op: ReduceOp = ReduceOp.SUM):
    """``acc[i] <- acc[i] + other[i]`` on the GPU (collectives.py:45-52);
    returns ``acc`` (updated in place for numpy and tensors alike)."""
    if op is not ReduceOp.SUM:
        raise ValueError(f"unsupported reduce op {op}")
    shape_a = tuple(acc.shape)
    shape_b = tuple(other.shape)
    if shape_a != shape_b:
        raise LengthMismatch(f"length mismatch: {shape_a} vs {shape_b}")
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(acc, torch.Tensor) and acc.is_cuda:
        a = acc
        b = other if isinstance(other, torch.Tensor) else torch.as_tensor(np.asarray(other))
        b = b.to(device=a.device, dtype=a.dtype).contiguous()
    else:
        a = torch.as_tensor(np.ascontiguousarray(acc)).to(dev)
        b = torch.as_tensor(np.ascontiguousarray(other, dtype=np.asarray(acc).dtype)).to(dev)
    if a.dtype not in (torch.float32, torch.bfloat16, torch.float16):
        raise Unsupported(f"reduce_inplace does not support {a.dtype}")
    if not a.is_contiguous():
        raise ValueError("acc must be contiguous")
    code = _lib.DTYPES[TORCH_DTYPES[a.dtype]]
    check(lib().pccl_reduce_inplace(a.data_ptr(), b.data_ptr(), a.numel(), code, _stream(a.device)), "reduce_inplace")
    if isinstance(acc, torch.Tensor) and acc.is_cuda:
        return acc
    res = a.cpu().numpy()
    if isinstance(acc, torch.Tensor):
        acc.copy_(torch.from_numpy(res))
    else:
        np.copyto(acc, res.reshape(acc.shape))
    return acc


# ---------------------------------------------------------------------------
# torch.distributed-shaped wrappers for FSDP / ZeRO-3
# ---------------------------------------------------------------------------
def all_gather_into_tensor(output: torch.Tensor, input: torch.Tensor, comm, *, algorithm: str = "auto"):
    """``output[g*n:(g+1)*n] = input of rank g`` (same contract as
    ``torch.distributed.all_gather_into_tensor``). Zero-copy when both tensors
    come from ``comm.world.empty`` (parameters kept in symmetric memory);
    in-place when ``input`` is this rank's slice of ``output``."""
    if output.numel() != input.numel() * comm.size:
        raise LengthMismatch(f"output has {output.numel()} elements, expected {input.numel() * comm.size}")
    all_gather(comm, input, algorithm=algorithm, out=output)
    return output


def reduce_scatter_tensor(output: torch.Tensor, input: torch.Tensor, comm, *, algorithm: str = "auto",
                          order: str = "ring"):
    """``output = chunk(rank) of the sum of every rank's input`` (same contract
    as ``torch.distributed.reduce_scatter_tensor`` with SUM)."""
    if input.numel() != output.numel() * comm.size:
        raise LengthMismatch(f"input has {input.numel()} elements, expected {output.numel() * comm.size}")
    reduce_scatter(comm, input, algorithm=algorithm, order=order, out=output)
    return output
