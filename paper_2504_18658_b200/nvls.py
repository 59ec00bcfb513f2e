"""NVLS (NVLink SHARP) multicast segments and collectives (real mode).

A multicast segment is one NVSwitch multicast object spanning every GPU of the
world; each rank's physical memory is bound to it and mapped twice — unicast
(its own copy, ordinary tensors) and multicast (``multimem`` ops, executed by
the switch). On it:

* :func:`nvls_all_gather` — every rank ``multimem.st``-s its block once and
  the switch writes it into every rank's copy of the output;
* :func:`nvls_reduce_scatter` — every rank's input sits in its copy of the
  segment and chunk r is read by rank r as the switch's sum over all copies
  (``multimem.ld_reduce``, fp32 accumulation for bf16 / fp16).

SURVEY.md §8(f) row 3. The switch's summation order is not any of the
reference's (collectives.py:79-165), so this path is for bf16 / fp16 training
traffic, never for fp32 order parity. Measured against the unicast kernels in
DESIGN.md §5 (``bench.py`` extras ``nvls_*``).

Setup is collective: rank 0 creates the object and hands its POSIX file
descriptor to the other ranks over a Unix socket (SCM_RIGHTS); every rank
adds its device, and after a barrier binds its memory.
"""
from __future__ import annotations

import ctypes
import json
import os
import socket
import tempfile
import time

import torch

from . import _lib
from ._lib import check, lib
from .errors import LengthMismatch, Unsupported
from .world import TORCH_DTYPES, _CudaArray

_counter = [0]


class NvlsSegment:
    """This rank's unicast view of a multicast segment."""

    def __init__(self, world, nvls_id: int, nbytes: int):
        self.world = world
        self.id = nvls_id
        self.nbytes = nbytes
        uc, mc, sz = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_size_t()
        check(lib().pccl_nvls_ptr(world.handle, nvls_id, ctypes.byref(uc), ctypes.byref(mc), ctypes.byref(sz)),
              "nvls_ptr")
        self.ptr = uc.value
        self._base = torch.as_tensor(_CudaArray(self.ptr, sz.value, self), device=f"cuda:{world.device}")

    def tensor(self, offset: int, numel: int, dtype=torch.uint8) -> torch.Tensor:
        es = torch.empty(0, dtype=dtype).element_size()
        if offset % 16 or offset + numel * es > self.nbytes:
            raise ValueError(f"view [{offset}, +{numel * es}) outside the {self.nbytes}-byte segment or unaligned")
        return self._base[offset: offset + numel * es].view(dtype)

    def offset_of(self, t: torch.Tensor) -> int:
        off = t.data_ptr() - self.ptr
        if not (0 <= off and off + t.numel() * t.element_size() <= self.nbytes) or not t.is_contiguous():
            raise ValueError("tensor is not a contiguous view of this NVLS segment")
        return off

    def close(self) -> None:
        """Collective: every rank's collectives on the segment are finished
        before any rank unbinds its memory from the multicast object."""
        if self.id >= 0:
            torch.cuda.synchronize(self.world.device)
            self.world._exchange(b"nvls-close")
            lib().pccl_nvls_destroy(self.world.handle, self.id)
            self.id = -1


def nvls_supported(world) -> bool:
    """True on every rank iff every rank's GPU supports switch multicast."""
    if world.emulated:
        return False
    mine = bool(lib().pccl_nvls_supported(world.handle))
    return all(json.loads(b.decode())["ok"] for b in world._exchange(json.dumps({"ok": mine}).encode()))


def create_nvls_segment(world, nbytes: int) -> NvlsSegment:
    """Collective over the world: a multicast segment of >= nbytes per rank."""
    if world.emulated:
        raise Unsupported("NVLS needs one process per GPU (real mode)")
    L = lib()
    me = {"ok": False}
    srv = None
    fd = ctypes.c_int(-1)
    nid = ctypes.c_int(-1)
    alloc = ctypes.c_size_t(0)
    if world.rank == 0:
        st = L.pccl_nvls_create(world.handle, nbytes, ctypes.byref(alloc), ctypes.byref(fd), ctypes.byref(nid))
        if st == 0:
            _counter[0] += 1
            path = os.path.join(tempfile.gettempdir(), f"pccl-nvls-{os.getpid()}-{_counter[0]}.sock")
            if os.path.exists(path):
                os.unlink(path)
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(path)
            srv.listen(world.nranks)
            srv.settimeout(120.0)  # a rank that never connects fails the setup instead of hanging it
            me = {"ok": True, "path": path, "alloc": alloc.value}
        else:
            me = {"ok": False, "why": _lib.error_string(st)}
    info = json.loads(world._exchange(json.dumps(me).encode())[0].decode())
    if not info["ok"]:
        raise Unsupported(f"NVLS multicast object: {info.get('why')}")
    try:
        if world.rank == 0:
            for _ in range(world.nranks - 1):
                conn, _addr = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"f"], [fd.value])
        else:
            cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            cli.settimeout(120.0)
            for _ in range(200):  # the server is listening before the exchange returned
                try:
                    cli.connect(info["path"])
                    break
                except OSError:
                    time.sleep(0.01)
            with cli:
                _msg, fds, _flags, _addr = socket.recv_fds(cli, 16, 1)
            if not fds:
                raise RuntimeError("no file descriptor received for the NVLS segment")
            st = L.pccl_nvls_import(world.handle, fds[0], info["alloc"], ctypes.byref(nid))
            os.close(fds[0])
            check(st, "nvls_import")
    finally:
        if srv is not None:
            srv.close()
            os.unlink(info["path"])
            os.close(fd.value)
    check(L.pccl_nvls_add_device(world.handle, nid.value), "nvls_add_device")
    world._exchange(b"added")  # every device is in the team before anyone binds
    check(L.pccl_nvls_bind(world.handle, nid.value), "nvls_bind")
    world._exchange(b"bound")
    return NvlsSegment(world, nid.value, info["alloc"])


def _code(t: torch.Tensor) -> int:
    name = TORCH_DTYPES.get(t.dtype)
    if name is None:
        raise Unsupported(f"dtype {t.dtype} not supported")
    return _lib.DTYPES[name]


def nvls_all_gather(comm, seg: NvlsSegment, x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out (a view of ``seg``, p * x.numel() elements) <- concat of every rank's x."""
    if out.numel() != x.numel() * comm.size or out.dtype != x.dtype:
        raise LengthMismatch(f"output has {out.numel()} elements, expected {x.numel() * comm.size}")
    st = lib().pccl_nvls_all_gather(comm.handle, seg.id, x.data_ptr(), seg.offset_of(out), x.numel(), _code(x),
                                    torch.cuda.current_stream(x.device).cuda_stream)
    check(st, "nvls_all_gather")
    return out


def nvls_reduce_scatter(comm, seg: NvlsSegment, x: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out <- chunk comm.rank of the sum over ranks of x (a view of ``seg``)."""
    if x.numel() != out.numel() * comm.size or out.dtype != x.dtype:
        raise LengthMismatch(f"input has {x.numel()} elements, expected {out.numel() * comm.size}")
    st = lib().pccl_nvls_reduce_scatter(comm.handle, seg.id, seg.offset_of(x), out.data_ptr(), out.numel(), _code(x),
                                        torch.cuda.current_stream(x.device).cuda_stream)
    check(st, "nvls_reduce_scatter")
    return out
