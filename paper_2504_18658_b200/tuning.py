"""Online calibration of the flat selector on the running box.

``algorithm="auto"`` picks from :class:`~.selector.FlatTable` — measured bus
bandwidth per (collective, p, size). The shipped table covers the GPU counts
it was measured on; :func:`autotune` measures the candidates for another
(collective, p, size) on the live world, agrees on the result across ranks
(max over ranks of each candidate's device time, exchanged with this
package's own all-gather) and adds the entries to the in-process table, so
every rank resolves ``auto`` identically afterwards. This is the B200
counterpart of the reference's ``calibrate_selector`` (bench/sweep.py:370-404),
which fills its table from simulation instead of measurement.
"""
from __future__ import annotations

import torch

from . import collectives as C
from .errors import Unsupported
from .selector import FlatEntry, FlatTable, _is_pow2
from . import selector as _sel


def _table() -> FlatTable:
    t = _sel.flat_table()
    if t is None:
        t = FlatTable()
        _sel._flat_table = t
    return t


def has_entries(collective: str, p: int) -> bool:
    t = _sel.flat_table()
    return t is not None and any(e.collective == collective and e.p == p for e in t.entries)


def autotune(comm, collective: str, m_bytes: int, *, dtype=torch.bfloat16, algorithms=None, iters: int = 10,
             warmup: int = 3) -> dict:
    """Time every candidate algorithm on symmetric buffers of ``m_bytes``
    (the all-gather output / reduce-scatter input) and record the results.
    Collective over the world: every rank must call it with the same
    arguments. Returns {algorithm: busbw GB/s} (max-over-ranks times)."""
    if comm.emulated:
        raise Unsupported("autotune measures NVLink: real mode (one process per GPU) only")
    if collective not in ("all_gather", "reduce_scatter"):
        raise Unsupported(f"unknown collective {collective!r}")
    p = comm.size
    algos = list(algorithms or [a for a in ("direct", "ring", "recursive") if a != "recursive" or _is_pow2(p)])
    es = torch.empty(0, dtype=dtype).element_size()
    if m_bytes % (es * p):
        raise ValueError(f"{m_bytes} bytes do not split into whole {dtype} elements over p={p}")
    total = m_bytes // es
    n_in, n_out = (total // p, total) if collective == "all_gather" else (total, total // p)
    world = comm.world
    off = (n_in * es + 255) // 256 * 256
    seg = world.create_segment(off + n_out * es)
    try:
        x = seg.tensor(world.rank, 0, n_in * es).view(dtype)
        y = seg.tensor(world.rank, off, n_out * es).view(dtype)
        x.zero_()
        op = C.all_gather if collective == "all_gather" else C.reduce_scatter
        times = []
        for a in algos:
            for _ in range(warmup):
                op(comm, x, algorithm=a, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                op(comm, x, algorithm=a, out=y)
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3 / iters)
        world.check()
        mine = torch.tensor(times, dtype=torch.float64, device=comm.device)
        every = C.all_gather(comm, mine, algorithm="direct").view(p, len(algos))
        tmax = every.max(dim=0).values.tolist()
    finally:
        world.destroy_segment(seg)
    t = _table()
    _sel._choice_cache.clear()
    t.entries = [e for e in t.entries if not (e.collective == collective and e.p == p and e.m_bytes == m_bytes)]
    result = {}
    for a, s in zip(algos, tmax):
        bw = m_bytes * (p - 1) / p / s / 1e9
        t.add(FlatEntry(collective, p, m_bytes, a, bw))
        result[a] = bw
    return result
