"""Measurement harness (paper_2504_18658_b200.sweep) vs the reference's
collkit.bench.sweep, pinned by tests/golden/sweep.json (made by
tests/golden/make_sweep_golden.py from the real reference)."""
import dataclasses
import hashlib
import json
import os

import pytest

from paper_2504_18658_b200 import sweep as S
from paper_2504_18658_b200.errors import EmptyCell, GridMismatch, NotDivisible, Unsupported

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sweep.json")))


@pytest.mark.parametrize("cell", GOLD["cells"], ids=lambda c: c["cell_id"])
def test_cell_inputs_match_reference(cell):
    cfg = S.SweepConfig(cell["collective"], cell["algorithm"], cell["inter"], (cell["m_bytes"],),
                        ((cell["N"], cell["M"]),), seed=cell["seed"])
    assert S.cell_seed(cfg.seed, cell["cell_id"]) == cell["cell_seed"]
    ins = S.make_inputs(cfg, cell["cell_id"], cell["N"] * cell["M"], cell["m_bytes"], cell["collective"])
    assert ins[0].size == cell["per_rank"]
    assert [float(v) for v in ins[0][:8]] == cell["head"]
    assert hashlib.sha256(b"".join(x.tobytes() for x in ins)).hexdigest() == cell["inputs_sha256"]


def _records():
    return [S.RunRecord("emulated", "all_gather", "ring", "ring", 4, 1, 4, m, t, s, False)
            for m, t, s in GOLD["records"]]


def test_summarize_matches_reference():
    recs = _records()
    got = []
    for drop in (False, True):
        for c in S.summarize(recs, drop_first_trial=drop):
            got.append((drop, c.cell[-1], c.count, c.mean, c.std, c.min))
    want = [(d["drop"], d["m_bytes"], d["count"], d["mean"], d["std"], d["min"]) for d in GOLD["summaries"]]
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g[:3] == w[:3]
        assert g[3:] == pytest.approx(w[3:], rel=1e-15, abs=0)


def test_heatmap_matches_reference():
    recs = _records()
    slow = [dataclasses.replace(r, seconds=r.seconds * (2 + r.trial)) for r in recs]
    got = S.emit_heatmap_data(recs, slow)
    assert [tuple(x[:2]) for x in got] == [tuple(x[:2]) for x in GOLD["heatmap_vs_slow"]]
    assert [x[2] for x in got] == pytest.approx([x[2] for x in GOLD["heatmap_vs_slow"]], rel=1e-15)
    with pytest.raises(GridMismatch):
        S.emit_heatmap_data(recs, recs[:4])
    with pytest.raises(EmptyCell):
        S.summarize([])


def test_records_csv_roundtrip(tmp_path):
    recs = _records()
    path = tmp_path / "r.csv"
    S.write_records_csv(recs, path)
    assert open(path).readline().strip().split(",") == list(S.RunRecord.CSV_FIELDS)
    assert S.read_records_csv(path) == recs
    rows = S.emit_heatmap_data(recs, recs)
    S.write_heatmap_csv(rows, tmp_path / "h.csv")
    assert open(tmp_path / "h.csv").read().splitlines()[0] == "p,m_bytes,speedup"


def test_config_validation():
    S.SweepConfig(sizes=(1 << 20,)).validate(8)
    with pytest.raises(Unsupported):
        S.SweepConfig(collective="all_reduce").validate()
    with pytest.raises(Unsupported):
        S.SweepConfig(algorithm="tree").validate()
    with pytest.raises(NotDivisible):
        S.SweepConfig(sizes=(100,), grid=((1, 8),)).validate()
    with pytest.raises(Unsupported):
        S.SweepConfig(algorithm="recursive", sizes=(96,), grid=((1, 6),)).validate()
    with pytest.raises(Unsupported):  # real backends: cells must match the world
        S.SweepConfig(grid=((2, 2),), sizes=(1024,)).validate(8)
    with pytest.raises(ValueError):
        S.SweepConfig(trials=0).validate()
    with pytest.raises(Unsupported):
        S.run_sweep(S.SweepConfig(), "socket")
    with pytest.raises(Unsupported):
        S.run_sweep(S.SweepConfig(), "b200")  # needs the world communicator


def test_size_parser():
    assert S._parse_size("64MiB") == 64 << 20
    assert S._parse_size("1GiB") == 1 << 30
    assert S._parse_size("4096") == 4096
    assert S.busbw_gbs(1 << 30, 8, 1.0) == pytest.approx((1 << 30) * 7 / 8 / 1e9)


@pytest.mark.gpu
@pytest.mark.parametrize("coll,algo,grid", [("all_gather", "ring", ((1, 8),)),
                                            ("reduce_scatter", "recursive", ((1, 4),)),
                                            ("reduce_scatter", "direct", ((1, 8),)),
                                            ("all_gather", "hierarchical", ((2, 4), (4, 2))),
                                            ("reduce_scatter", "hierarchical", ((2, 4),))])
def test_emulated_sweep_verifies(coll, algo, grid):
    cfg = S.SweepConfig(coll, algo, "recursive", (1 << 16, 1 << 20), grid, trials=2, verify=True, warmup=True)
    recs = S.run_sweep(cfg, "emulated")
    assert len(recs) == len(grid) * 2 * 3
    assert all(r.verified and r.seconds > 0 for r in recs)
    summ = S.summarize(recs, drop_first_trial=True)
    assert len(summ) == len(grid) * 2 and all(c.count == 2 for c in summ)
