"""Communicators over a :class:`~.world.World` (mirrors
``collkit/transport/base.py:105-174`` and ``transport/inprocess.py:74-113``).

A :class:`Communicator` is an ordered group of world ranks used by exactly one
rank (one thread). It exposes the reference's attributes (``rank``, ``size``,
``members``, ``comm_id``, ``next_base_tag()``, ``barrier()``, ``subgroup()``)
and carries the C-ABI group handle the collectives run on. Point-to-point
``send``/``recv`` are not part of this path: the collectives move data with
device loads over NVLink, not with messages.

Two modes:

* **real** — one process per GPU; build the world communicator with
  :func:`init_from_torch` after ``torch.distributed.init_process_group``
  (the process group is only the bootstrap that exchanges IPC handles);
* **emulated** — :func:`run_ranks` runs ``fn(comm)`` on one thread per rank,
  like the reference, but every collective is a rendezvous: the last rank to
  arrive issues ONE cooperative launch that executes all ranks' work on
  ``cuda:0`` with the same kernels as the real path.
"""
from __future__ import annotations

import ctypes
import threading
import time

import torch

from . import _lib
from ._lib import check, lib
from .errors import IndexOutOfRange, LengthMismatch, SelfSend, Timeout, Unsupported
from .world import World

STEP_TAGS_PER_COLLECTIVE = 1 << 13
COLLECTIVE_TAGS_PER_COMM = 1 << 26
MAX_COMM_ID = (1 << 32) // COLLECTIVE_TAGS_PER_COMM - 1


class _GroupHandle:
    """C pccl_comm for one member set (shared by the members' Communicators in
    emulation; one per process in real mode)."""

    def __init__(self, world: World, members: tuple, comm_id: int):
        arr = (ctypes.c_int * len(members))(*members)
        h = ctypes.c_void_p()
        check(lib().pccl_comm_create(world.handle, arr, len(members), comm_id, ctypes.byref(h)), "comm_create")
        self.handle = h
        self.members = members

    def __del__(self):  # pragma: no cover
        try:
            lib().pccl_comm_destroy(self.handle)
        except Exception:
            pass


class Rendezvous:
    """Collects one call per member of an emulated group and runs it once."""

    def __init__(self, timeout: float = 120.0):
        self._cond = threading.Condition()
        self._pending: dict = {}
        self._timeout = timeout

    def arrive(self, key, size: int, rank_in_group: int, payload, execute):
        with self._cond:
            # a fast rank may reach the next call with the same key before the
            # slow ranks have collected the previous result
            while key in self._pending and self._pending[key]["done"]:
                self._cond.wait(1.0)
            entry = self._pending.setdefault(key, {"payloads": {}, "done": False, "result": None, "error": None})
            entry["payloads"][rank_in_group] = payload
            if len(entry["payloads"]) == size:
                try:
                    entry["result"] = execute([entry["payloads"][i] for i in range(size)])
                except BaseException as exc:  # noqa: BLE001 - delivered to every member
                    entry["error"] = exc
                entry["done"] = True
                entry["left"] = size
                self._cond.notify_all()
            else:
                deadline = time.monotonic() + self._timeout
                while not entry["done"]:
                    left = deadline - time.monotonic()
                    if left <= 0:
                        raise Timeout(f"rank {rank_in_group} waited {self._timeout}s for its peers at {key}")
                    self._cond.wait(left)
            entry["left"] -= 1
            if entry["left"] == 0:
                del self._pending[key]
                self._cond.notify_all()
            if entry["error"] is not None:
                raise entry["error"]
            return entry["result"][rank_in_group]


class Communicator:
    """An ordered group of ranks sharing a World (one object per rank)."""

    def __init__(self, world: World, members, comm_id: int = 0, *, rank: int | None = None,
                 _group: _GroupHandle | None = None, _rdv: Rendezvous | None = None):
        self.world = world
        self.members = tuple(int(m) for m in members)
        if not 0 <= comm_id <= MAX_COMM_ID:
            raise ValueError(f"comm_id {comm_id} out of range")
        self.comm_id = comm_id
        self.world_rank = world.rank if not world.emulated else rank
        if self.world_rank is None:
            raise ValueError("emulated communicators need their world rank")
        try:
            self.rank = self.members.index(self.world_rank)
        except ValueError:
            raise IndexError(f"rank {self.world_rank} is not a member of {self.members}") from None
        for m in self.members:
            if not 0 <= m < world.nranks:
                raise IndexOutOfRange(f"member {m} not in [0, {world.nranks})")
        self._group = _group or _GroupHandle(world, self.members, comm_id)
        self._rdv = _rdv
        self._next_seq = 0
        self._stage_need: dict = {}  # (reduce, algo, count, dtype) -> staging bytes

    @property
    def size(self) -> int:
        return len(self.members)

    @property
    def emulated(self) -> bool:
        return self.world.emulated

    @property
    def handle(self):
        return self._group.handle

    @property
    def device(self) -> torch.device:
        return torch.device("cuda", self.world.device)

    def epoch(self) -> int:
        """Completed collectives on this member set (device counter; equal on
        every member between calls — the SPMD invariant)."""
        e = ctypes.c_uint64()
        check(lib().pccl_comm_epoch(self.handle, self.rank, ctypes.byref(e)), "comm_epoch")
        return e.value

    def next_base_tag(self) -> int:
        """Same numbering as the reference (transport/base.py:131-138); the
        device epoch of the group advances in lockstep with it."""
        seq = self._next_seq
        self._next_seq += 1
        seq %= COLLECTIVE_TAGS_PER_COMM // STEP_TAGS_PER_COLLECTIVE
        return self.comm_id * COLLECTIVE_TAGS_PER_COMM + seq * STEP_TAGS_PER_COLLECTIVE

    # -- emulation plumbing ------------------------------------------------
    def _rendezvous(self, payload, execute):
        key = (self.members, self.comm_id, self.next_base_tag())

        def locked(payloads):
            # emulated sub-groups share the world's staging segment and one
            # device: their host-side staging copies + launch must not interleave
            with self.world.lock:
                return execute(payloads)

        return self._rdv.arrive(key, self.size, self.rank, payload, locked)

    def barrier(self) -> None:
        """Device-side barrier: a zero-byte all-gather (entry + exit handshake
        with every member), then a stream sync."""
        from .collectives import _all_gather_device

        if self.size == 1:
            return
        if self.emulated:
            def execute(_payloads):
                empty = [torch.empty(0, device=self.device) for _ in range(self.size)]
                _all_gather_device(self, "direct", empty, empty, emu=True)
                torch.cuda.synchronize(self.device)
                self.world.check()
                return [None] * self.size

            self._rendezvous(None, execute)
            return
        self.next_base_tag()
        e = torch.empty(0, device=self.device)
        _all_gather_device(self, "direct", [e], [e], emu=False)
        torch.cuda.synchronize(self.device)
        self.world.check()

    def subgroup(self, members, comm_id: int) -> "Communicator | None":
        members = tuple(members)
        if self.world_rank not in members:
            return None
        if self.emulated:
            group, rdv = _emu_group(self.world, members, comm_id)
            return Communicator(self.world, members, comm_id, rank=self.world_rank, _group=group, _rdv=rdv)
        return Communicator(self.world, members, comm_id)

    # -- point-to-point (transport/base.py:140-152) ---------------------------
    # Tagged messages over per-pair mailbox rings in the flag arena (C ABI
    # pccl_send / pccl_recv): exact (source, tag) FIFO matching; send never
    # waits for a matching recv. Payloads: bytes-like (host) or CUDA tensors.
    def send(self, dst: int, tag: int, payload) -> None:
        if not 0 <= dst < self.size:
            raise IndexOutOfRange(f"destination {dst} not in [0, {self.size})")
        if dst == self.rank:  # transport contract (inprocess.py, tests/test_transport_inprocess.py)
            raise SelfSend(f"rank {self.rank} cannot send to itself")
        if tag < 0:
            raise ValueError(f"tag must be >= 0, got {tag}")
        keep = None
        if isinstance(payload, torch.Tensor) and payload.is_cuda:
            t = payload.contiguous()
            ptr, nbytes, host, keep = t.data_ptr(), t.numel() * t.element_size(), 0, t
        else:
            if isinstance(payload, torch.Tensor):
                payload = payload.contiguous().numpy()
            mv = memoryview(payload).cast("B")
            nbytes = mv.nbytes
            if nbytes % 4:  # payloads are whole fp32 elements (transport/base.py:46)
                raise LengthMismatch(f"payload of {nbytes} bytes is not a whole number of 4-byte elements")
            keep = (ctypes.c_char * max(nbytes, 1)).from_buffer_copy(mv) if nbytes else None
            ptr, host = (ctypes.addressof(keep) if keep is not None else None), 1
        check(lib().pccl_send(self.handle, self.rank, dst, int(tag), ptr, nbytes, host), "send")
        del keep

    def recv(self, src: int, tag: int) -> bytes:
        if not 0 <= src < self.size:
            raise IndexOutOfRange(f"source {src} not in [0, {self.size})")
        n = ctypes.c_size_t(0)
        check(lib().pccl_recv(self.handle, self.rank, src, int(tag), None, 0, 1, ctypes.byref(n)), "recv")
        buf = (ctypes.c_char * max(n.value, 1))()
        check(lib().pccl_recv(self.handle, self.rank, src, int(tag), buf, n.value, 1, ctypes.byref(n)), "recv")
        return bytes(buf[: n.value])

    def recv_into(self, src: int, tag: int, out: torch.Tensor) -> torch.Tensor:
        """Receive straight into a CUDA tensor (its byte size must hold the message)."""
        if not (out.is_cuda and out.is_contiguous()):
            raise ValueError("recv_into: contiguous CUDA tensor required")
        n = ctypes.c_size_t(0)
        check(lib().pccl_recv(self.handle, self.rank, src, int(tag), out.data_ptr(), out.numel() * out.element_size(),
                              0, ctypes.byref(n)), "recv")
        return out

    def sendrecv(self, peer: int, tag: int, payload) -> bytes:
        """Exchange with one peer; no deadlock whatever the peer's ordering
        (sends never wait for the receiver, base.py:143-149)."""
        if peer == self.rank:
            raise SelfSend(f"rank {self.rank} cannot exchange with itself")
        self.send(peer, tag, payload)
        return self.recv(peer, tag)


# ---------------------------------------------------------------------------
# emulated worlds (cached per rank count) and run_ranks
# ---------------------------------------------------------------------------
_emu_lock = threading.Lock()
_emu_worlds: dict = {}
_emu_groups: dict = {}


def emulated_world(nranks: int, device: int = 0) -> World:
    with _emu_lock:
        w = _emu_worlds.get((nranks, device))
        if w is None:
            w = World.emulated_world(nranks, device)
            _emu_worlds[(nranks, device)] = w
        return w


def _emu_group(world: World, members: tuple, comm_id: int):
    with _emu_lock:
        key = (id(world), members, comm_id)
        g = _emu_groups.get(key)
        if g is None:
            g = (_GroupHandle(world, members, comm_id), Rendezvous())
            _emu_groups[key] = g
        return g


def emulated_communicators(nranks: int, device: int = 0) -> list:
    """One world Communicator per emulated rank (use from separate threads)."""
    world = emulated_world(nranks, device)
    members = tuple(range(nranks))
    group, rdv = _emu_group(world, members, 0)
    # fresh Rendezvous/sequence per set of communicators
    rdv = Rendezvous()
    return [Communicator(world, members, 0, rank=r, _group=group, _rdv=rdv) for r in range(nranks)]


def run_ranks(num_ranks: int, fn, *, transport=None, device: int = 0) -> list:
    """Run ``fn(comm)`` once per rank on concurrent threads over an emulated
    world on one GPU and return the per-rank results in rank order (drop-in
    for ``collkit.transport.inprocess.run_ranks``). The lowest-rank error is
    re-raised (inprocess.py:110-112)."""
    if num_ranks < 1:
        raise ValueError("num_ranks must be >= 1")
    comms = emulated_communicators(num_ranks, device)
    world = comms[0].world
    results: list = [None] * num_ranks
    errors: list = []

    def runner(r: int) -> None:
        try:
            torch.cuda.set_device(device)
            results[r] = fn(comms[r])
        except BaseException as exc:  # noqa: BLE001
            errors.append((r, exc))

    threads = [threading.Thread(target=runner, args=(r,), daemon=True) for r in range(num_ranks)]
    for t in threads:
        t.start()
    deadline = time.monotonic() + 300.0
    for t in threads:
        t.join(max(0.0, deadline - time.monotonic()))
    if any(t.is_alive() for t in threads):
        raise RuntimeError("ranks did not finish (possible deadlock)")
    if errors:
        torch.cuda.synchronize(device)
        world.reset_flags()  # a failed emulated collective may leave ABORT flags
        errors.sort(key=lambda e: e[0])
        raise errors[0][1]
    return results


# ---------------------------------------------------------------------------
# real mode bootstrap
# ---------------------------------------------------------------------------
def init_from_torch(group=None, device: int | None = None, staging_bytes: int = 64 << 20) -> Communicator:
    """World communicator over the current torch.distributed job (one process
    per GPU). The process group only carries the IPC handles at init and on
    segment growth; collectives never touch it."""
    import torch.distributed as dist

    rank, size = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()

    def exchange(blob: bytes) -> list:
        out = [None] * size
        dist.all_gather_object(out, blob, group=group)
        return out

    world = World.create(size, rank, device, exchange)
    if staging_bytes:
        world.ensure_staging(staging_bytes)
    return Communicator(world, range(size), 0)


def check_uniform(values, what: str) -> None:
    if len(set(values)) > 1:
        raise LengthMismatch(f"{what} differs across ranks: {values}")
