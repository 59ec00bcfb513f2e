"""CPU: bench.py's own checker and launcher logic.

``bench.expected_rs`` is the torch restatement the bench uses to verify every
timed call on the device; here it is pinned against the oracle (itself pinned
against collkit's golden vectors) for every algorithm, order, dtype and the
hierarchical groupings, so a ``"verified": true`` on a bench line means
"bit-identical to the reference's reduction order"."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import bench
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _inputs(p, n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(n * p, generator=g).to(dtype) for _ in range(p)]


def _np(x: torch.Tensor):
    if x.dtype == torch.bfloat16:
        return x.view(torch.int16).numpy().view(np.uint16)
    return x.numpy()


def _expected_all(xs, algo, order="ring", grid=None, inter="ring"):
    p = len(xs)
    n = xs[0].numel() // p
    return [bench.expected_rs([x[c * n : (c + 1) * n] for x in xs], c, algo, order, grid, inter) for c in range(p)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_expected_rs_matches_oracle_flat(p, dtype):
    xs = _inputs(p, 257, dtype, 7 * p)
    dn = "f32" if dtype == torch.float32 else "bf16"
    nx = [_np(x) for x in xs]
    cases = [
        ("ring", "ring", oracle.ring_reduce_scatter(nx, dn)),
        ("recursive", "recursive", oracle.rechalf_reduce_scatter(nx, dn)),
        ("direct", "ring", oracle.direct_reduce_scatter(nx, dn, order="ring")),
        ("direct", "recursive", oracle.direct_reduce_scatter(nx, dn, order="recursive")),
        ("direct", "rank", oracle.direct_reduce_scatter(nx, dn, order="rank")),
    ]
    for algo, order, want in cases:
        got = _expected_all(xs, algo, order)
        for c in range(p):
            assert np.array_equal(_np(got[c]).view(np.uint8), np.asarray(want[c]).view(np.uint8)), (algo, order, c)


@pytest.mark.parametrize("grid,inter", [((2, 4), "ring"), ((4, 2), "recursive"), ((2, 2), "ring"),
                                        ((4, 2), "ring")])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_expected_rs_matches_oracle_hierarchical(grid, inter, dtype):
    p = grid[0] * grid[1]
    xs = _inputs(p, 129, dtype, 11)
    dn = "f32" if dtype == torch.float32 else "bf16"
    want = oracle.hier_reduce_scatter([_np(x) for x in xs], grid[0], grid[1], inter, dn)
    got = _expected_all(xs, "hierarchical", grid=grid, inter=inter)
    for c in range(p):
        assert np.array_equal(_np(got[c]).view(np.uint8), np.asarray(want[c]).view(np.uint8)), c


def test_expected_rs_differs_between_orders():
    # the check has teeth: on random fp32 the orders disagree somewhere
    xs = _inputs(8, 4096, torch.float32, 3)
    a = _expected_all(xs, "ring")
    b = _expected_all(xs, "recursive")
    assert any(not torch.equal(x, y) for x, y in zip(a, b))


def test_seeded_fill_is_reproducible():
    a, b = torch.empty(1000, dtype=torch.bfloat16), torch.empty(1000, dtype=torch.bfloat16)
    bench.seeded_fill(a, 5)
    bench.seeded_fill(b, 5)
    assert bench._bits_equal(a, b)
    bench.seeded_fill(b, 6)
    assert not bench._bits_equal(a, b)


def test_bench_refuses_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "WORLD_SIZE=2" in line["error"]


def test_bench_refuses_more_ranks_than_gpus():
    # no GPU here: --gpus 2 must refuse instead of time-sharing a device
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "visible GPU" in line["error"] and line["n_gpus"] == 2


def test_reference_arm_config_matches_ours():
    class A:
        dtype, size_mib, algo = "bf16", 128, "recursive"

    assert bench.config_for(A, 8, False) == bench.config_for(A, 8, False)
    assert bench.config_for(A, 4, True)["parallelism"] == "dp4"
