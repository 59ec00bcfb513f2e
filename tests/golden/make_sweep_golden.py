"""Golden vectors for the measurement harness, produced by the REAL reference
(``collkit.bench.sweep``) in this container:

    python tests/golden/make_sweep_golden.py

Writes ``tests/golden/sweep.json``: per-cell seeds and a digest of the
per-rank inputs the reference's ``make_inputs`` draws for sweep cells, plus
``summarize`` output over a fixed record list. Nothing on the GPU box reads
/root/reference; the JSON is committed.
"""
from __future__ import annotations

import dataclasses
import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from collkit.bench import sweep as S

    cells = []
    for coll, algo, inter, N, M, m in [("all_gather", "ring", "ring", 1, 8, 4096),
                                       ("reduce_scatter", "recursive", "ring", 1, 4, 1024),
                                       ("all_gather", "hierarchical", "recursive", 2, 4, 8192),
                                       ("reduce_scatter", "hierarchical", "ring", 4, 2, 2048)]:
        cfg = S.SweepConfig(collective=coll, algorithm=algo, inter=inter, sizes=(m,), grid=((N, M),), seed=3)
        cell_id = f"{coll}:{algo}:{inter}:{N}x{M}:{m}"
        ins = S.make_inputs(cfg, cell_id, N * M, m, coll)
        digest = hashlib.sha256(b"".join(x.tobytes() for x in ins)).hexdigest()
        cells.append(dict(collective=coll, algorithm=algo, inter=inter, N=N, M=M, m_bytes=m, seed=3,
                          cell_id=cell_id, cell_seed=S.cell_seed(3, cell_id), inputs_sha256=digest,
                          per_rank=int(ins[0].size), head=[float(v) for v in ins[0][:8]]))
    recs = []
    for m, secs in [(1024, [0.5, 0.1, 0.2, 0.3]), (2048, [0.9, 0.4])]:
        for t, s in enumerate(secs):
            recs.append(S.RunRecord("inprocess", "all_gather", "ring", "ring", 4, 1, 4, m, t, s, False))
    summ = []
    for drop in (False, True):
        for c in S.summarize(recs, drop_first_trial=drop):
            summ.append(dict(drop=drop, m_bytes=c.cell[-1], count=c.count, mean=c.mean, std=c.std, min=c.min))
    slow = [dataclasses.replace(r, seconds=r.seconds * (2 + r.trial)) for r in recs]
    heat = S.emit_heatmap_data(recs, slow)
    with open(os.path.join(HERE, "sweep.json"), "w") as f:
        json.dump(dict(cells=cells, records=[[r.m_bytes, r.trial, r.seconds] for r in recs], summaries=summ,
                       heatmap_vs_slow=heat), f, indent=1)
    print(f"{len(cells)} cells, {len(summ)} summaries")


if __name__ == "__main__":
    main()
