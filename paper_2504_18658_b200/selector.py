"""Algorithm selection (mirrors ``collkit/costmodel.py:24-196``).

Two layers:

* the reference's inter-node selector, same contract: ``choose_inter_algorithm``
  (analytic mode compares the alpha-beta formulas, ring on ties and for
  non-power-of-two N; table mode looks up a :class:`CalibrationTable`), used
  by ``HierPlan.resolve_inter``;
* a flat selector for ``all_gather(..., algorithm="auto")`` /
  ``reduce_scatter``: a :class:`FlatTable` of *measured* B200 bus bandwidth per
  (collective, p, message size) — measured on the GPU box by ``tools/sweep.py``
  / ``tuning.autotune`` into ``data/flat_calibration.csv`` — with the nearest
  log-size bucket winning, as in ``CalibrationTable.lookup``
  (costmodel.py:127-139). A GPU count the table does not cover is calibrated
  on the live world the first time ``auto`` meets it (``tuning.autotune``,
  SPMD: every rank measures the same candidates and agrees on the result).

``CostParams()`` keeps the reference's desk-scale defaults
(costmodel.py:35-41), so reference code that evaluates ``t_ring(...,
CostParams())`` gets the reference's numbers; ``B200_NVLINK`` is the preset
for NVLink 5 on B200 (flag round trip a few microseconds; 770 GB/s measured
peer copy per direction). The analytic selector's decisions are the same
under both: with equal per-step bandwidth the recursive variant wins exactly
when it has fewer steps (pow2 N >= 4), and N = 2 ties go to ring.
"""
from __future__ import annotations

import csv
import math
import os
from dataclasses import dataclass, field

from .errors import EmptyTable, NonPowerOfTwo

DATA_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
FLAT_TABLE_PATH = os.path.join(DATA_DIR, "flat_calibration.csv")


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class CostParams:
    """alpha: seconds per message, beta: seconds per byte, gamma: seconds per
    reduced byte (costmodel.py:24-41; same defaults)."""

    alpha_inter: float = 10e-6
    beta_inter: float = 0.04e-9
    alpha_intra: float = 3e-6
    beta_intra: float = 0.01e-9
    gamma_reduce_fast: float = 0.002e-9
    gamma_reduce_slow: float = 0.4e-9
    packet_bytes: int = 2048

    def __post_init__(self) -> None:
        for name in ("alpha_inter", "beta_inter", "alpha_intra", "beta_intra", "gamma_reduce_fast",
                     "gamma_reduce_slow"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if self.packet_bytes < 1:
            raise ValueError("packet_bytes must be >= 1")

    def alpha_beta(self, level: str):
        if level == "inter":
            return self.alpha_inter, self.beta_inter
        if level == "intra":
            return self.alpha_intra, self.beta_intra
        raise ValueError(f"unknown level {level!r}")

    def gamma(self, profile: str) -> float:
        if profile == "fast":
            return self.gamma_reduce_fast
        if profile == "slow":
            return self.gamma_reduce_slow
        raise ValueError(f"unknown reduce profile {profile!r}")


# NVLink 5 / NVSwitch on B200: ~3 us per flag handshake, 770 GB/s measured peer
# copy per direction (B200_PROFILING.md), 6.5 TB/s HBM for the fused adds
B200_NVLINK = CostParams(alpha_inter=3e-6, beta_inter=1.0 / 770e9, alpha_intra=3e-6, beta_intra=1.0 / 770e9,
                         gamma_reduce_fast=1.0 / 6.5e12, gamma_reduce_slow=0.4e-9)


def t_ring(p: int, m_bytes: float, params: CostParams, level: str = "inter") -> float:
    if p < 1:
        raise ValueError(f"p must be >= 1, got {p}")
    a, b = params.alpha_beta(level)
    return a * (p - 1) + b * m_bytes * (p - 1) / p


def t_rec(p: int, m_bytes: float, params: CostParams, level: str = "inter") -> float:
    if not _is_pow2(p):
        raise NonPowerOfTwo(f"recursive algorithms require power-of-two p, got {p}")
    a, b = params.alpha_beta(level)
    return a * math.log2(p) + b * m_bytes * (p - 1) / p


def t_direct(p: int, m_bytes: float, params: CostParams, level: str = "intra") -> float:
    """One step: every peer's share moves concurrently over the switch."""
    a, b = params.alpha_beta(level)
    return (a if p > 1 else 0.0) + b * m_bytes * (p - 1) / p


def t_hierarchical(topo, m_bytes: float, inter_alg: str, params: CostParams) -> float:
    """Two-level model (costmodel.py:88-105): the inter phase moves the
    per-local-rank share m / M across the N nodes, the intra ring moves the
    whole buffer inside each node; the transpose is free."""
    n, m_gpus = topo.num_nodes, topo.gpus_per_node
    sub_m = m_bytes / m_gpus
    if inter_alg == "auto":
        inter_alg = choose_inter_algorithm(n, sub_m, params) if n >= 2 else "ring"
    if inter_alg == "ring":
        inter = t_ring(n, sub_m, params, level="inter")
    elif inter_alg == "recursive":
        inter = t_rec(n, sub_m, params, level="inter")
    else:
        raise ValueError(f"unknown inter_alg {inter_alg!r}")
    return inter + t_ring(m_gpus, m_bytes, params, level="intra")


@dataclass(frozen=True)
class CalibrationEntry:
    n_nodes: int
    m_bytes: int
    ring_seconds: float
    recursive_seconds: float
    winner: str


@dataclass
class CalibrationTable:
    entries: list = field(default_factory=list)

    def add(self, entry: CalibrationEntry) -> None:
        self.entries.append(entry)

    def lookup(self, n_nodes: int, m_bytes: float) -> str:
        cands = [e for e in self.entries if e.n_nodes == n_nodes]
        if not cands:
            raise EmptyTable(f"no calibration entries for N={n_nodes} ({len(self.entries)} entries total)")
        x = math.log(max(m_bytes, 1.0))
        return min(cands, key=lambda e: abs(x - math.log(e.m_bytes))).winner

    def save_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["N", "m_bytes", "ring_seconds", "recursive_seconds", "winner"])
            for e in self.entries:
                w.writerow([e.n_nodes, e.m_bytes, repr(e.ring_seconds), repr(e.recursive_seconds), e.winner])

    @classmethod
    def load_csv(cls, path) -> "CalibrationTable":
        t = cls()
        with open(path, newline="") as fh:
            for row in csv.DictReader(fh):
                t.add(CalibrationEntry(int(row["N"]), int(row["m_bytes"]), float(row["ring_seconds"]),
                                       float(row["recursive_seconds"]), row["winner"]))
        return t


def choose_inter_algorithm(n_nodes: int, m_bytes: float, params: CostParams | None = None,
                           mode: str = "analytic", table: CalibrationTable | None = None) -> str:
    """Same contract as costmodel.choose_inter_algorithm (costmodel.py:169-196)."""
    if n_nodes < 2:
        raise ValueError(f"selection needs at least 2 nodes, got {n_nodes}")
    if mode == "table":
        if table is None or not table.entries:
            raise EmptyTable("table mode requires a calibration table")
        return table.lookup(n_nodes, m_bytes)
    if mode != "analytic":
        raise ValueError(f"unknown selection mode {mode!r}")
    if not _is_pow2(n_nodes):
        return "ring"
    params = params or CostParams()
    return "ring" if t_ring(n_nodes, m_bytes, params) <= t_rec(n_nodes, m_bytes, params) else "recursive"


# ---------------------------------------------------------------------------
# flat selector from measured bus bandwidth
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class FlatEntry:
    collective: str
    p: int
    m_bytes: int
    algorithm: str
    busbw_gbs: float


@dataclass
class FlatTable:
    entries: list = field(default_factory=list)

    def add(self, e: FlatEntry) -> None:
        self.entries.append(e)
        _choice_cache.clear()

    def best(self, collective: str, p: int, m_bytes: float, allowed=None) -> str:
        cands = [e for e in self.entries if e.collective == collective and e.p == p
                 and (allowed is None or e.algorithm in allowed)]
        if not cands:
            raise EmptyTable(f"no measurements for {collective} at p={p}")
        x = math.log(max(m_bytes, 1.0))
        size = min({e.m_bytes for e in cands}, key=lambda m: abs(x - math.log(m)))
        return max((e for e in cands if e.m_bytes == size), key=lambda e: e.busbw_gbs).algorithm

    def save_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["collective", "p", "m_bytes", "algorithm", "busbw_gbs"])
            for e in self.entries:
                w.writerow([e.collective, e.p, e.m_bytes, e.algorithm, f"{e.busbw_gbs:.3f}"])

    @classmethod
    def load_csv(cls, path) -> "FlatTable":
        t = cls()
        with open(path, newline="") as fh:
            for row in csv.DictReader(fh):
                t.add(FlatEntry(row["collective"], int(row["p"]), int(row["m_bytes"]), row["algorithm"],
                                float(row["busbw_gbs"])))
        return t


_flat_table: FlatTable | None = None


def flat_table() -> FlatTable | None:
    global _flat_table
    if _flat_table is None and os.path.exists(FLAT_TABLE_PATH):
        _flat_table = FlatTable.load_csv(FLAT_TABLE_PATH)
    return _flat_table


_choice_cache: dict = {}


def order_preserving(order: str) -> tuple:
    """Reduce-scatter algorithms that add in ``order``: the one-shot direct
    kernel folds in any order; ring adds in ring order and recursive halving
    in butterfly order only. ``auto`` picks among these, so an fp32 result
    never changes bits with the message size or the table."""
    return {"ring": ("direct", "ring"), "recursive": ("direct", "recursive"), "rank": ("direct",)}[order]


def choose_algorithm(collective: str, p: int, m_bytes: float, order: str | None = None) -> str:
    """Measured winner for (collective, p, size) — for a reduce-scatter only
    among the algorithms that reduce in ``order`` (default ring); one-shot
    ``direct`` (the fewest steps over a full-bandwidth switch) when nothing
    was measured. Memoised per (collective, p, size, order); table edits
    clear the memo."""
    if collective == "reduce_scatter" and order is None:
        order = "ring"
    key = (collective, p, m_bytes, order)
    hit = _choice_cache.get(key)
    if hit is None:
        hit = _choice_cache[key] = _choose(collective, p, m_bytes, order)
    return hit


def _choose(collective: str, p: int, m_bytes: float, order: str | None) -> str:
    t = flat_table()
    allowed = order_preserving(order) if collective == "reduce_scatter" else None
    if t is not None:
        try:
            return t.best(collective, p, m_bytes, allowed)
        except EmptyTable:
            pass
    return "direct"
