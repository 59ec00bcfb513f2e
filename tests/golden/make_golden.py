"""Generate golden vectors by running the REAL reference (collkit) in this
container. Run from the repo root:

    python tests/golden/make_golden.py

It imports ``collkit`` from ``/root/reference/pkg/src`` (read-only; never copied),
executes every hot-path algorithm through the reference's own
``transport.inprocess.run_ranks`` on seeded standard-normal fp32 inputs (which
pin the floating-point reduction order) and integer-valued inputs (the
reference's own test domain), and writes:

* ``tests/golden/collectives.npz`` — inputs and per-rank outputs per case;
* ``tests/golden/schedules.json`` — ``simnet.build_schedule`` step multisets.

The fixtures are committed; nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from collkit import collectives as C
    from collkit import hierarchy as H
    from collkit.costmodel import CostParams
    from collkit.simnet import SimConfig, build_schedule
    from collkit.topology import Topology
    from collkit.transport.inprocess import run_ranks

    def topo_for(n, m):
        return Topology(n, m, max(1, m // 2) if m % 2 == 0 else 1)

    arrays: dict[str, np.ndarray] = {}
    cases = []

    def inputs_for(kind, p, size, seed):
        rng = np.random.default_rng(seed)
        if kind == "normal":
            return [rng.standard_normal(size).astype(np.float32) for _ in range(p)]
        return [rng.integers(-1024, 1025, size=size).astype(np.float32) for _ in range(p)]

    def record(name, inputs, outs, meta):
        arrays[name + "/in"] = np.stack(inputs)
        arrays[name + "/out"] = np.stack(outs)
        cases.append(dict(name=name, **meta))

    seed = 1000
    for kind in ("normal", "int"):
        for p in (1, 2, 3, 4, 5, 8, 16):
            for n in (1, 37, 64):
                seed += 1
                ins = inputs_for(kind, p, n, seed)
                outs = run_ranks(p, lambda c: C.ring_all_gather(c, ins[c.rank]))
                record(f"ag_ring_{kind}_p{p}_n{n}", ins, outs, dict(op="ag", algo="ring", p=p, n=n))
                if p & (p - 1) == 0:
                    outs = run_ranks(p, lambda c: C.recdbl_all_gather(c, ins[c.rank]))
                    record(f"ag_recursive_{kind}_p{p}_n{n}", ins, outs, dict(op="ag", algo="recursive", p=p, n=n))
                seed += 1
                ins = inputs_for(kind, p, n * p, seed)
                outs = run_ranks(p, lambda c: C.ring_reduce_scatter(c, ins[c.rank]))
                record(f"rs_ring_{kind}_p{p}_n{n}", ins, outs, dict(op="rs", algo="ring", p=p, n=n))
                if p & (p - 1) == 0:
                    outs = run_ranks(p, lambda c: C.rechalf_reduce_scatter(c, ins[c.rank]))
                    record(f"rs_recursive_{kind}_p{p}_n{n}", ins, outs, dict(op="rs", algo="recursive", p=p, n=n))

    grid = [(1, 1), (1, 2), (1, 8), (2, 1), (2, 2), (2, 4), (4, 2), (4, 4), (2, 8), (8, 1), (3, 2)]
    for kind in ("normal", "int"):
        for (N, M) in grid:
            for inter in ("ring", "recursive"):
                if inter == "recursive" and N & (N - 1):
                    continue
                p = N * M
                n = 24
                topo = topo_for(N, M)
                plan = H.HierPlan(topo=topo, inter_alg=inter)
                seed += 1
                ins = inputs_for(kind, p, n, seed)
                outs = run_ranks(p, lambda c: H.hier_all_gather(plan, c, ins[c.rank]))
                record(f"ag_hier_{kind}_{N}x{M}_{inter}", ins, outs,
                       dict(op="ag", algo="hierarchical", N=N, M=M, inter=inter, p=p, n=n))
                seed += 1
                ins = inputs_for(kind, p, n * p, seed)
                outs = run_ranks(p, lambda c: H.hier_reduce_scatter(plan, c, ins[c.rank]))
                record(f"rs_hier_{kind}_{N}x{M}_{inter}", ins, outs,
                       dict(op="rs", algo="hierarchical", N=N, M=M, inter=inter, p=p, n=n))

    # Shuffles (known-answer + random).
    rng = np.random.default_rng(7)
    for (N, M, blk) in [(2, 2, 1), (2, 3, 4), (4, 2, 5), (2, 4, 3), (1, 4, 3), (4, 1, 3)]:
        buf = rng.standard_normal(N * M * blk).astype(np.float32)
        arrays[f"shuffle_{N}x{M}_b{blk}/in"] = buf
        arrays[f"shuffle_{N}x{M}_b{blk}/l2g"] = H.shuffle_local_major_to_global(buf, N, M, blk)
        arrays[f"shuffle_{N}x{M}_b{blk}/g2l"] = H.shuffle_global_to_local_major(buf, N, M, blk)

    np.savez_compressed(os.path.join(HERE, "collectives.npz"), **arrays)

    sched = []
    cells = [
        ("all_gather", "ring", "ring", 1, 4, 64),
        ("all_gather", "ring", "ring", 1, 8, 64 * 8),
        ("reduce_scatter", "ring", "ring", 1, 6, 48),
        ("reduce_scatter", "ring", "ring", 1, 8, 64 * 8),
        ("all_gather", "recursive", "ring", 1, 8, 32),
        ("reduce_scatter", "recursive", "ring", 1, 16, 64),
        ("reduce_scatter", "recursive", "ring", 1, 8, 64 * 8),
        ("all_gather", "hierarchical", "recursive", 4, 4, 128),
        ("all_gather", "hierarchical", "ring", 2, 4, 256),
        ("all_gather", "hierarchical", "recursive", 4, 2, 256),
        ("reduce_scatter", "hierarchical", "ring", 2, 8, 256),
        ("reduce_scatter", "hierarchical", "ring", 2, 4, 256),
        ("reduce_scatter", "hierarchical", "recursive", 4, 2, 256),
    ]
    for coll, algo, inter, N, M, m_bytes in cells:
        topo = topo_for(N, M)
        steps = build_schedule(SimConfig(topo=topo, params=CostParams()), coll, algo, m_bytes, inter)
        sched.append(dict(collective=coll, algorithm=algo, inter=inter, N=N, M=M, m_bytes=m_bytes,
                          steps=[sorted(list(m) for m in msgs) for msgs, _ in steps]))
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(sched, f)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"{len(cases)} collective cases, {len(sched)} schedules")


if __name__ == "__main__":
    main()
