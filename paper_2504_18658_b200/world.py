"""Symmetric device memory of one NVSwitch box (host side).

A :class:`World` is the B200 replacement of the reference's transport state
(``collkit/transport/inprocess.py:14-51``, ``transport/base.py:76-102``): instead
of queues of byte payloads it owns *segments* of device memory that every rank
maps (CUDA IPC over NVLink 5 / NVSwitch):

* segment 0 — flag arena (cross-GPU signals, see ``csrc/device.cuh``);
* staging — where the C layer copies device buffers that peers must read but
  that the caller did not allocate symmetrically;
* io — where host (numpy) inputs are uploaded and outputs downloaded, so the
  drop-in numpy path never pays a device-to-device staging copy;
* user segments — :meth:`World.empty` returns tensors peers can read
  zero-copy (the FSDP path keeps parameters / gradients there).

Real mode: one process per GPU; segment handles are exchanged through the
caller's bootstrap (``exchange(bytes) -> list[bytes]``, normally
``torch.distributed.all_gather_object``). Emulation mode: ``nranks`` ranks in one
process on one GPU, every "peer" pointer local; the same kernels run all ranks
in one cooperative launch.
"""
from __future__ import annotations

import ctypes
import threading
from typing import Callable

import torch

from . import _lib
from ._lib import check, lib, ptr_array
from .errors import OutOfMemory

TORCH_DTYPES = {
    torch.float32: "f32",
    torch.bfloat16: "bf16",
    torch.float16: "f16",
    torch.uint8: "u8",
    torch.int32: "i32",
    torch.int64: "i64",
    torch.float64: "f64",
}


class _CudaArray:
    """Minimal ``__cuda_array_interface__`` view of a raw device pointer."""

    def __init__(self, ptr: int, nbytes: int, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": (nbytes,),
            "typestr": "|u1",
            "data": (ptr, False),
            "version": 3,
            "strides": None,
        }


class _Lease:
    """Lifetime of memory handed out as tensors (World.empty / SymmetricHeap):
    the tensors' storages keep it alive; when the last one dies the release
    callback is queued on the world and run at the next allocation outside
    CUDA-graph capture (it synchronises the device)."""

    def __init__(self, world: "World", release: Callable[[], None]):
        self._world = world
        self._release = release

    def __del__(self):  # pragma: no cover - GC timing
        w = self._world
        if w is not None and not w._closed:
            w._pending.append(self._release)


class Segment:
    def __init__(self, world: "World", seg_id: int, nbytes: int):
        self.world = world
        self.id = seg_id
        self.nbytes = nbytes

    def ptr(self, rank: int) -> int:
        p = ctypes.c_void_p()
        check(lib().pccl_segment_ptr(self.world.handle, self.id, rank, ctypes.byref(p), None), "segment_ptr")
        return p.value or 0

    def tensor(self, rank: int, offset: int = 0, nbytes: int | None = None, owner=None) -> torch.Tensor:
        """uint8 tensor over [offset, offset + nbytes) of rank's copy (this
        process must own it: its own rank in real mode, any rank in emulation).
        ``owner`` is kept alive by the tensor's storage."""
        nbytes = self.nbytes - offset if nbytes is None else nbytes
        base = torch.as_tensor(_CudaArray(self.ptr(rank) + offset, nbytes, owner or self),
                               device=f"cuda:{self.world.device}")
        return base


class Registration:
    """Caller-owned tensors registered collectively as a segment (zero-copy
    for collectives whose buffers lie inside it). Keeps the tensors alive
    until ``close()``."""

    def __init__(self, world: "World", seg: Segment, tensors):
        self.world, self.segment, self._tensors = world, seg, tensors

    def close(self) -> None:
        if self.segment is not None and not self.world._closed:
            self.world.destroy_segment(self.segment)
        self.segment, self._tensors = None, None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class SymmetricHeap:
    """A symmetric arena (one collective segment) with a deterministic
    first-fit allocator: as long as every rank performs the same sequence of
    ``empty`` calls and tensor releases (SPMD code, e.g. FSDP), a block lands
    at the same offset on every rank, so collectives on heap tensors are
    zero-copy. A divergence is not silent: the offset enters every call's
    signature and mismatched ranks raise LengthMismatch. Freed blocks are
    reused in address order; reuse is stream-ordered like the caching
    allocator's (a block freed while another stream still uses it needs the
    usual event / record_stream discipline)."""

    ALIGN = 256

    def __init__(self, world: "World", nbytes: int):
        self.world = world
        self.segment = world.create_segment(nbytes)
        self.nbytes = self.segment.nbytes
        self._free = [(0, self.nbytes)]  # sorted (offset, size)
        self._lock = threading.Lock()

    def _alloc(self, size: int) -> int:
        size = max(self.ALIGN, (size + self.ALIGN - 1) // self.ALIGN * self.ALIGN)
        with self._lock:
            for i, (off, sz) in enumerate(self._free):
                if sz >= size:
                    if sz == size:
                        self._free.pop(i)
                    else:
                        self._free[i] = (off + size, sz - size)
                    return off, size
        raise OutOfMemory(f"symmetric heap: no free block of {size} bytes ({self.nbytes} total)")

    def _release(self, off: int, size: int) -> None:
        with self._lock:
            self._free.append((off, size))
            self._free.sort()
            merged = []
            for o, z in self._free:
                if merged and merged[-1][0] + merged[-1][1] == o:
                    merged[-1] = (merged[-1][0], merged[-1][1] + z)
                else:
                    merged.append((o, z))
            self._free = merged

    def empty(self, numel: int, dtype=torch.float32):
        """This rank's tensor (real mode) or one per rank (emulation)."""
        self.world._run_pending()
        es = torch.empty(0, dtype=dtype).element_size()
        off, size = self._alloc(numel * es)
        heap = self
        lease = _Lease(self.world, lambda: heap._release(off, size))
        if self.world.emulated:
            return [self.segment.tensor(r, off, numel * es, lease).view(dtype) for r in range(self.world.nranks)]
        return self.segment.tensor(self.world.rank, off, numel * es, lease).view(dtype)

    def bytes_free(self) -> int:
        with self._lock:
            return sum(z for _, z in self._free)


class World:
    """Symmetric memory + flag arena shared by all communicators of a box."""

    def __init__(self, handle: int, nranks: int, rank: int, device: int, emulated: bool,
                 exchange: Callable[[bytes], list] | None):
        self.handle = ctypes.c_void_p(handle)
        self.nranks = nranks
        self.rank = rank
        self.device = device
        self.emulated = emulated
        self._exchange = exchange
        self._segments: dict[int, Segment] = {}
        self._pending: list = []  # releases queued by dead leases (run outside graph capture)
        self.staging: Segment | None = None
        self.io: Segment | None = None
        self.lock = threading.RLock()
        self._closed = False
        self._share(0, 0)  # flag arena

    # ---- construction -------------------------------------------------
    @classmethod
    def create(cls, nranks: int, rank: int, device: int, exchange: Callable[[bytes], list]) -> "World":
        h = ctypes.c_void_p()
        check(lib().pccl_world_create(nranks, rank, device, ctypes.byref(h)), "world_create")
        return cls(h.value, nranks, rank, device, False, exchange)

    @classmethod
    def emulated_world(cls, nranks: int, device: int = 0) -> "World":
        h = ctypes.c_void_p()
        check(lib().pccl_emu_world_create(nranks, device, ctypes.byref(h)), "emu_world_create")
        return cls(h.value, nranks, -1, device, True, None)

    # ---- segments -------------------------------------------------------
    def _share(self, seg_id: int, nbytes: int) -> Segment:
        """Export/exchange/import segment seg_id (collective in real mode)."""
        if not self.emulated:
            buf = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
            check(lib().pccl_segment_export(self.handle, seg_id, buf), "segment_export")
            handles = self._exchange(bytes(buf))
            if len(handles) != self.nranks:
                raise RuntimeError("bootstrap exchange returned the wrong number of handles")
            allh = (ctypes.c_char * (_lib.IPC_HANDLE_BYTES * self.nranks))()
            for q, hb in enumerate(handles):
                ctypes.memmove(ctypes.addressof(allh) + q * _lib.IPC_HANDLE_BYTES, hb, _lib.IPC_HANDLE_BYTES)
            check(lib().pccl_segment_import(self.handle, seg_id, allh), "segment_import")
        seg = Segment(self, seg_id, nbytes)
        self._segments[seg_id] = seg
        return seg

    def _run_pending(self) -> None:
        if not self._pending or torch.cuda.is_current_stream_capturing():
            return
        todo, self._pending = self._pending, []
        for release in todo:
            release()

    def create_segment(self, nbytes: int) -> Segment:
        """Collective (real mode): allocate nbytes on every rank and map them."""
        self._run_pending()
        sid = ctypes.c_int(-1)
        check(lib().pccl_segment_create(self.handle, nbytes, ctypes.byref(sid)), "segment_create")
        return self._share(sid.value, nbytes)

    def destroy_segment(self, seg: Segment) -> None:
        torch.cuda.synchronize(self.device)
        check(lib().pccl_segment_destroy(self.handle, seg.id), "segment_destroy")
        self._segments.pop(seg.id, None)

    @staticmethod
    def _grow(need: int) -> int:
        size = 1 << 20
        while size < need:
            size <<= 1
        return size

    def ensure_staging(self, nbytes: int) -> None:
        """Collective over the world when it grows (all ranks ask for the same size)."""
        with self.lock:
            if self.staging is not None and self.staging.nbytes >= nbytes:
                return
            if self.staging is not None:
                self.destroy_segment(self.staging)
            self.staging = self.create_segment(self._grow(nbytes))
            check(lib().pccl_world_set_staging(self.handle, self.staging.id), "set_staging")

    def ensure_io(self, nbytes: int) -> Segment:
        with self.lock:
            if self.io is None or self.io.nbytes < nbytes:
                if self.io is not None:
                    self.destroy_segment(self.io)
                self.io = self.create_segment(self._grow(nbytes))
            return self.io

    def empty(self, numel: int, dtype=torch.float32, rank: int | None = None):
        """Symmetric tensor(s) peers can read zero-copy. Collective in real
        mode (returns this rank's tensor); in emulation returns one tensor per
        rank. The segment is released (collectively: every rank drops its
        tensors in the same program order) once its tensors are gone."""
        es = torch.empty(0, dtype=dtype).element_size()
        seg = self.create_segment(max(256, numel * es))
        lease = _Lease(self, lambda: self.destroy_segment(seg) if seg.id in self._segments else None)
        if self.emulated:
            return [seg.tensor(r, 0, numel * es, lease).view(dtype) for r in range(self.nranks)]
        return seg.tensor(self.rank, 0, numel * es, lease).view(dtype)

    def heap(self, nbytes: int) -> SymmetricHeap:
        """A symmetric arena with a deterministic allocator (collective)."""
        return SymmetricHeap(self, nbytes)

    def register(self, tensor) -> Registration:
        """Register caller-owned CUDA tensor(s) for zero-copy collectives.
        Collective in real mode: every rank passes its own tensor of the same
        byte size (the peers map the cudaMalloc allocation that contains it;
        torch's caching allocator qualifies, expandable segments do not ->
        Unsupported). Emulation: a list with one tensor per rank."""
        self._run_pending()
        ts = list(tensor) if self.emulated else [tensor]
        if self.emulated and len(ts) != self.nranks:
            raise ValueError(f"emulation: register one tensor per rank ({self.nranks})")
        for t in ts:
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
                raise ValueError("register: contiguous CUDA tensors only")
        nbytes = ts[0].numel() * ts[0].element_size()
        sid = ctypes.c_int(-1)
        if self.emulated:
            check(lib().pccl_emu_segment_register(self.handle, ptr_array([t.data_ptr() for t in ts]), nbytes,
                                                  ctypes.byref(sid)), "segment_register")
        else:
            check(lib().pccl_segment_register(self.handle, ts[0].data_ptr(), nbytes, ctypes.byref(sid)),
                  "segment_register")
            try:
                buf = (ctypes.c_char * _lib.REG_HANDLE_BYTES)()
                st = lib().pccl_segment_register_export(self.handle, sid.value, buf)
                blobs = self._exchange(bytes([st & 0xff]) + bytes(buf))
                bad = [b[0] for b in blobs if b[0]]
                if bad:  # every rank fails the same way (no one imports)
                    check(bad[0], "segment_register_export")
                allh = (ctypes.c_char * (_lib.REG_HANDLE_BYTES * self.nranks))()
                for q, hb in enumerate(blobs):
                    ctypes.memmove(ctypes.addressof(allh) + q * _lib.REG_HANDLE_BYTES, hb[1:], _lib.REG_HANDLE_BYTES)
                check(lib().pccl_segment_register_import(self.handle, sid.value, allh), "segment_register_import")
            except Exception:
                lib().pccl_segment_destroy(self.handle, sid.value)
                raise
        seg = Segment(self, sid.value, nbytes)
        self._segments[sid.value] = seg
        return Registration(self, seg, ts)

    # ---- status --------------------------------------------------------
    def check(self) -> None:
        """Raise a device-reported error (Timeout, LengthMismatch, ...)."""
        check(lib().pccl_world_check(self.handle), "device")

    def reset_flags(self) -> None:
        check(lib().pccl_world_reset_flags(self.handle), "reset_flags")

    def set_tuning(self, ctas: int = 0, nsub: int = 0) -> None:
        check(lib().pccl_world_set_tuning(self.handle, ctas, nsub, 0), "set_tuning")

    def set_param(self, key: str, value: int) -> None:
        """Tuning knob (ctas, nsub, ag_variant, rs_variant, tma_stages, tma_tile, timeout_ms)."""
        check(lib().pccl_world_set_param(self.handle, key.encode(), int(value)), f"set_param({key})")

    def get_param(self, key: str) -> int:
        v = ctypes.c_int64()
        check(lib().pccl_world_get_param(self.handle, key.encode(), ctypes.byref(v)), f"get_param({key})")
        return v.value

    def trace(self, back: int = 0):
        """Events of a traced launch (param "trace" = K keeps the last K;
        back = 0 is the latest): list over rows of lists over CTAs of
        (t_ns, kind, unit) tuples; kinds: 1 start, 2 wait done, 3 signal,
        4 exit barrier done, 5 CTA exit."""
        cap = 16 * 320 * 128
        buf = (ctypes.c_uint64 * cap)()
        rows, ctas = ctypes.c_int(), ctypes.c_int()
        check(lib().pccl_world_trace_at(self.handle, back, buf, cap, ctypes.byref(rows), ctypes.byref(ctas)),
              "trace")
        out = []
        for y in range(rows.value):
            row = []
            for b in range(ctas.value):
                base = (y * ctas.value + b) * 128
                ev = [(int(v) >> 16, (int(v) >> 12) & 0xF, int(v) & 0xFFF) for v in buf[base:base + 128] if v]
                row.append(ev)
            out.append(row)
        return out

    def set_timeout_ms(self, ms: int) -> None:
        check(lib().pccl_world_set_timeout_ms(self.handle, ms), "set_timeout")

    def close(self) -> None:
        if not self._closed and self.handle:
            self._closed = True
            lib().pccl_world_destroy(self.handle)

    def __del__(self):  # pragma: no cover - interpreter teardown order varies
        try:
            self.close()
        except Exception:
            pass
