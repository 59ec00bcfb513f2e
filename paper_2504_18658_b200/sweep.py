"""Measurement harness in the reference's vocabulary (``collkit/bench/sweep.py``).

Same records, same deterministic per-cell inputs and the same protocol as the
reference's ``run_sweep`` / ``summarize`` (sweep.py:36-338): every (grid cell x
size) runs ``trials`` independent timed trials (plus a leading warm-up trial
when ``warmup``), inputs are integer-valued float32 in [-1024, 1024] drawn from
``sha256(f"{seed}:{cell_id}")`` (sweep.py:124-136), so they are the very bytes
the reference's CPU path would see. Differences, B200-side: a trial is timed on
the device with CUDA events between two device barriers and the max over
ranks is kept (the reference keeps rank 0's wall clock); ``verify`` checks
outputs on the device against the exact sums (integer inputs make every fold
order exact).

Run under torchrun (one process per GPU)::

    torchrun --nproc-per-node 8 -m paper_2504_18658_b200.sweep \
        --collective all_gather --algorithm ring --sizes 64MiB,128MiB --verify --warmup
"""
from __future__ import annotations

import argparse
import csv
import hashlib
import os
import statistics
from dataclasses import dataclass

import numpy as np
import torch

from .errors import EmptyCell, GridMismatch, NotDivisible, Unsupported, VerificationFailed

DEFAULT_SIZES = tuple(2**i * 2**20 for i in range(4, 11))  # 16 MiB .. 1 GiB (sweep.py:37)
ALGORITHMS = ("ring", "recursive", "direct", "hierarchical", "auto")


@dataclass(frozen=True)
class RunRecord:
    backend: str
    collective: str
    algorithm: str
    inter: str
    p: int
    n_nodes: int
    m_gpus: int
    m_bytes: int
    trial: int
    seconds: float
    verified: bool

    CSV_FIELDS = ("backend", "collective", "algorithm", "inter", "p", "N", "M", "m_bytes", "trial", "seconds",
                  "verified")

    def cell_key(self) -> tuple:
        return (self.backend, self.collective, self.algorithm, self.inter, self.n_nodes, self.m_gpus, self.m_bytes)

    def row(self) -> list:
        return [self.backend, self.collective, self.algorithm, self.inter, self.p, self.n_nodes, self.m_gpus,
                self.m_bytes, self.trial, repr(self.seconds), int(self.verified)]


@dataclass(frozen=True)
class SweepConfig:
    collective: str = "all_gather"
    algorithm: str = "ring"
    inter: str = "ring"
    sizes: tuple = DEFAULT_SIZES
    grid: tuple = ()           # (N, M) cells; () = flat over the world
    trials: int = 10
    seed: int = 0
    verify: bool = False
    warmup: bool = False

    def cells(self, world: int | None = None) -> tuple:
        return self.grid or ((1, world or 8),)

    def validate(self, world: int | None = None) -> None:
        """sweep.py:98-111; ``world`` (real backends) pins every cell's N*M."""
        if self.collective not in ("all_gather", "reduce_scatter"):
            raise Unsupported(f"unknown collective {self.collective!r}")
        if self.algorithm not in ALGORITHMS:
            raise Unsupported(f"unknown algorithm {self.algorithm!r}")
        if self.trials < 1:
            raise ValueError("trials must be >= 1")
        for (n_nodes, m_gpus) in self.cells(world):
            p = n_nodes * m_gpus
            if world is not None and p != world:
                raise Unsupported(f"grid cell {n_nodes}x{m_gpus} does not match the world of {world} ranks")
            if self.algorithm == "recursive" and p & (p - 1):
                raise Unsupported(f"recursive algorithm needs power-of-two p, got {p}")
            for m in self.sizes:
                if m % (4 * p):
                    raise NotDivisible(f"size {m} not divisible into whole elements over p={p}")


def cell_seed(global_seed: int, cell_id: str) -> int:
    """sweep.py:124-126."""
    return int.from_bytes(hashlib.sha256(f"{global_seed}:{cell_id}".encode()).digest()[:8], "little")


def make_inputs(config: SweepConfig, cell_id: str, p: int, m_bytes: int, collective: str) -> list:
    """Per-rank integer-valued float32 inputs, identical to the reference's
    make_inputs (sweep.py:129-136)."""
    rng = np.random.default_rng(cell_seed(config.seed, cell_id))
    per_rank = m_bytes // 4 if collective == "reduce_scatter" else m_bytes // (4 * p)
    return [rng.integers(-1024, 1025, size=per_rank).astype(np.float32) for _ in range(p)]


BACKENDS = ("b200", "emulated", "nccl")


def _flat_op(collective: str, algorithm: str):
    from . import collectives as C

    if collective == "all_gather":
        return lambda comm, x, out: C.all_gather(comm, x, algorithm=algorithm, out=out)
    return lambda comm, x, out: C.reduce_scatter(comm, x, algorithm=algorithm, out=out)


def _expected(collective: str, ins: list, rank: int) -> np.ndarray:
    """Exact result (integer-valued inputs: any fold order is exact)."""
    if collective == "all_gather":
        return np.concatenate(ins)
    n = ins[0].size // len(ins)
    return np.sum([x[rank * n:(rank + 1) * n].astype(np.float64) for x in ins], axis=0).astype(np.float32)


def _cell_call(config: SweepConfig, n_nodes: int, m_gpus: int):
    """fn(comm, x, out) running the configured collective on device tensors."""
    if config.algorithm != "hierarchical":
        return _flat_op(config.collective, config.algorithm)
    from .hierarchy import HierPlan, hier_all_gather, hier_reduce_scatter
    from .topology import Topology

    plan = HierPlan(topo=Topology(n_nodes, m_gpus), inter_alg=config.inter)
    op = hier_all_gather if config.collective == "all_gather" else hier_reduce_scatter
    return lambda comm, x, out: op(plan, comm, x, out=out)


def run_sweep(config: SweepConfig, backend: str = "b200", *, comm=None) -> list:
    """Execute every (grid cell x size) ``trials`` times (+1 leading warm-up
    trial, recorded, when ``warmup``) — sweep.py:203-302.

    * ``b200``: this process is one rank of a real world; pass the world
      communicator (:func:`init_from_torch`). The grid is one cell matching it.
      Trials are device-timed (CUDA events between device barriers), max over
      ranks; every rank returns the same records.
    * ``nccl``: same, timing ``torch.distributed`` all_gather_into_tensor /
      reduce_scatter_tensor on the same inputs (the comparison baseline).
    * ``emulated``: every cell's ranks run on this GPU through :func:`run_ranks`
      (the reference's in-process backend); rank 0's wall clock between
      barriers, like the reference.
    """
    if backend not in BACKENDS:
        raise Unsupported(f"unknown backend {backend!r}")
    if backend == "emulated":
        return _run_emulated(config)
    if comm is None:
        raise Unsupported(f"{backend} sweeps need the world communicator (init_from_torch)")
    import torch.distributed as dist

    p = comm.size
    config.validate(p)
    if backend == "nccl" and config.algorithm not in ("auto", "ring"):
        raise Unsupported("the nccl backend picks its own algorithm; use --algorithm auto")
    dev = comm.device
    records = []
    for (n_nodes, m_gpus) in config.cells(p):
        for m_bytes in config.sizes:
            cell_id = f"{config.collective}:{config.algorithm}:{config.inter}:{n_nodes}x{m_gpus}:{m_bytes}"
            ins = make_inputs(config, cell_id, p, m_bytes, config.collective)
            out_n = ins[0].size // p if config.collective == "reduce_scatter" else ins[0].size * p
            if backend == "b200":
                x = comm.world.empty(ins[comm.rank].size, torch.float32)
                out = comm.world.empty(out_n, torch.float32)
                op = _cell_call(config, n_nodes, m_gpus)
                call = lambda: op(comm, x, out)  # noqa: E731
                barrier = comm.barrier
            else:
                x = torch.empty(ins[comm.rank].size, dtype=torch.float32, device=dev)
                out = torch.empty(out_n, dtype=torch.float32, device=dev)
                if config.collective == "all_gather":
                    call = lambda: dist.all_gather_into_tensor(out, x)  # noqa: E731
                else:
                    call = lambda: dist.reduce_scatter_tensor(out, x)  # noqa: E731
                barrier = lambda: dist.barrier(device_ids=[dev.index])  # noqa: E731
            x.copy_(torch.from_numpy(ins[comm.rank]))
            verified = False
            if config.verify:
                call()
                ok = torch.equal(out, torch.from_numpy(_expected(config.collective, ins, comm.rank)).to(dev))
                flag = torch.tensor([int(ok)], device=dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                if not int(flag):
                    raise VerificationFailed(f"{config.collective} output wrong in cell {cell_id}")
                verified = True
            for trial in range(config.trials + (1 if config.warmup else 0)):
                barrier()
                torch.cuda.synchronize(dev)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                call()
                e1.record()
                torch.cuda.synchronize(dev)
                t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                records.append(RunRecord(backend, config.collective, config.algorithm, config.inter, p, n_nodes,
                                         m_gpus, m_bytes, trial, float(t), verified))
            if backend == "b200":
                comm.world.check()
    return records


def _run_emulated(config: SweepConfig) -> list:
    import time

    from .communicator import run_ranks

    config.validate()
    records = []
    for (n_nodes, m_gpus) in config.cells():
        p = n_nodes * m_gpus
        op = _cell_call(config, n_nodes, m_gpus)
        for m_bytes in config.sizes:
            cell_id = f"{config.collective}:{config.algorithm}:{config.inter}:{n_nodes}x{m_gpus}:{m_bytes}"
            ins = make_inputs(config, cell_id, p, m_bytes, config.collective)
            out_n = ins[0].size // p if config.collective == "reduce_scatter" else ins[0].size * p
            xs = [torch.from_numpy(a).cuda() for a in ins]
            outs = [torch.empty(out_n, dtype=torch.float32, device="cuda") for _ in range(p)]
            verified = False
            if config.verify:
                run_ranks(p, lambda c: op(c, xs[c.rank], outs[c.rank]))
                for r in range(p):
                    if not torch.equal(outs[r].cpu(), torch.from_numpy(_expected(config.collective, ins, r))):
                        raise VerificationFailed(f"{config.collective} output wrong at rank {r} in {cell_id}")
                verified = True
            for trial in range(config.trials + (1 if config.warmup else 0)):
                secs = [0.0] * p

                def timed(c):
                    c.barrier()
                    t0 = time.perf_counter()
                    op(c, xs[c.rank], outs[c.rank])
                    c.barrier()
                    secs[c.rank] = time.perf_counter() - t0

                run_ranks(p, timed)
                records.append(RunRecord("emulated", config.collective, config.algorithm, config.inter, p, n_nodes,
                                         m_gpus, m_bytes, trial, secs[0], verified))
            del xs, outs
    return records


@dataclass(frozen=True)
class CellSummary:
    cell: tuple
    count: int
    mean: float
    std: float
    min: float


def summarize(records, *, drop_first_trial: bool = False) -> list:
    """Per-cell mean, (n-1)-std and min; trial 0 dropped on request
    (sweep.py:313-338)."""
    cells: dict = {}
    for rec in records:
        cells.setdefault(rec.cell_key(), []).append(rec)
    if not cells:
        raise EmptyCell("no records to summarize")
    out = []
    for key in sorted(cells):
        rows = cells[key]
        if drop_first_trial and len(rows) > 1:
            rows = [r for r in rows if r.trial != 0]
        if not rows:
            raise EmptyCell(f"cell {key} has no records")
        v = [r.seconds for r in rows]
        out.append(CellSummary(key, len(v), statistics.fmean(v), statistics.stdev(v) if len(v) > 1 else 0.0, min(v)))
    return out


def busbw_gbs(m_bytes: int, p: int, seconds: float) -> float:
    return m_bytes * (p - 1) / p / seconds / 1e9


def emit_heatmap_data(records_a, records_b) -> list:
    """(p, m_bytes, speedup of A over baseline B = mean_B / mean_A) per cell;
    both record sets must cover the same (p, size) grid (sweep.py:341-360)."""
    def means(records):
        acc: dict = {}
        for r in records:
            acc.setdefault((r.p, r.m_bytes), []).append(r.seconds)
        return {k: statistics.fmean(v) for k, v in acc.items()}

    a, b = means(records_a), means(records_b)
    if not a or set(a) != set(b):
        raise GridMismatch(f"grids differ: {sorted(set(a) ^ set(b))}" if a else "empty record sets")
    return [(p, m, b[(p, m)] / a[(p, m)]) for (p, m) in sorted(a)]


def write_heatmap_csv(rows, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(("p", "m_bytes", "speedup"))
        w.writerows((p, m, repr(s)) for p, m, s in rows)


def write_records_csv(records, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(RunRecord.CSV_FIELDS)
        w.writerows(r.row() for r in records)


def read_records_csv(path) -> list:
    with open(path, newline="") as fh:
        return [RunRecord(d["backend"], d["collective"], d["algorithm"], d["inter"], int(d["p"]), int(d["N"]),
                          int(d["M"]), int(d["m_bytes"]), int(d["trial"]), float(d["seconds"]),
                          bool(int(d["verified"]))) for d in csv.DictReader(fh)]


def _parse_size(s: str) -> int:
    s = s.strip().upper()
    for suf, mul in (("GIB", 1 << 30), ("MIB", 1 << 20), ("KIB", 1 << 10), ("G", 1 << 30), ("M", 1 << 20)):
        if s.endswith(suf):
            return int(float(s[: -len(suf)]) * mul)
    return int(s)


def _print_summary(recs, drop_first: bool, verified: bool) -> None:
    for c in summarize(recs, drop_first_trial=drop_first):
        be, col, alg, inter, N, M, m = c.cell
        print(f"{be:8s} {col:14s} {alg:12s} inter={inter:9s} {N}x{M} {m / 2**20:8.1f} MiB  mean {c.mean * 1e6:9.1f} us "
              f"+- {c.std * 1e6:6.1f}  min {c.min * 1e6:9.1f}  busbw {busbw_gbs(m, N * M, c.mean):7.1f} GB/s "
              f"({c.count} trials{', verified' if verified else ''})", flush=True)


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--backend", choices=list(BACKENDS), default="b200",
                    help="b200/nccl: one process per GPU under torchrun; emulated: all ranks on this GPU")
    ap.add_argument("--collective", choices=["all_gather", "reduce_scatter", "ag", "rs"], default="all_gather")
    ap.add_argument("--algorithm", "--algo", choices=list(ALGORITHMS), default="ring")
    ap.add_argument("--inter", choices=["ring", "recursive", "auto"], default="ring")
    ap.add_argument("--sizes", default="64MiB,128MiB,256MiB")
    ap.add_argument("--grid", default="", help="N x M cells, e.g. 2x4,4x2 (hierarchical)")
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--verify", action="store_true")
    ap.add_argument("--warmup", action="store_true")
    ap.add_argument("--csv", default="")
    ap.add_argument("--compare", default="", help="records CSV of a baseline run: print speedup per cell")
    a = ap.parse_args(argv)
    coll = {"ag": "all_gather", "rs": "reduce_scatter"}.get(a.collective, a.collective)
    grid = tuple(tuple(int(x) for x in c.split("x")) for c in a.grid.split(",") if c)
    cfg = SweepConfig(coll, a.algorithm, a.inter, tuple(_parse_size(s) for s in a.sizes.split(",")), grid, a.trials,
                      a.seed, a.verify, a.warmup)
    rank0 = True
    if a.backend == "emulated":
        recs = run_sweep(cfg, "emulated")
    else:
        import torch.distributed as dist

        from .communicator import init_from_torch

        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = init_from_torch(device=local)
        rank0 = comm.rank == 0
        recs = run_sweep(cfg, a.backend, comm=comm)
    if rank0:
        _print_summary(recs, a.warmup, cfg.verify)
        if a.csv:
            write_records_csv(recs, a.csv)
        if a.compare:
            for p, m, sp in emit_heatmap_data(recs, read_records_csv(a.compare)):
                print(f"speedup p={p} {m / 2**20:8.1f} MiB: {sp:.3f}x", flush=True)
    if a.backend != "emulated":
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
