"""CPU: the oracle (numpy restatement of collkit) is pinned against golden
vectors produced by running the real reference, and against the reference's
own known-answer tests (pkg/tests/test_collectives.py, test_hierarchy.py)."""
import numpy as np
import pytest

import oracle
from tests.golden import fixtures

CASES = fixtures.cases()
Z = fixtures.arrays()


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8)


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_oracle_matches_reference_golden(case):
    ins = list(Z[case["name"] + "/in"])
    want = Z[case["name"] + "/out"]
    if case["algo"] == "hierarchical":
        fn = oracle.hier_all_gather if case["op"] == "ag" else oracle.hier_reduce_scatter
        got = fn(ins, case["N"], case["M"], case["inter"])
    else:
        fn = {
            ("ag", "ring"): oracle.ring_all_gather,
            ("ag", "recursive"): oracle.recdbl_all_gather,
            ("rs", "ring"): oracle.ring_reduce_scatter,
            ("rs", "recursive"): oracle.rechalf_reduce_scatter,
        }[(case["op"], case["algo"])]
        got = fn(ins)
    assert np.array_equal(_bits(np.stack(got)), _bits(want))


@pytest.mark.parametrize("case", [c for c in CASES if c["op"] == "rs"], ids=lambda c: c["name"])
def test_direct_fold_orders_equal_stepwise_algorithms(case):
    """The one-shot fold in the named order is bit-identical (fp32) to the
    step-wise reference algorithm — the property the direct kernels rely on."""
    ins = list(Z[case["name"] + "/in"])
    want = Z[case["name"] + "/out"]
    got = oracle.direct_reduce_scatter(ins, "f32", case["algo"], case.get("N"), case.get("M"), case.get("inter", "ring"))
    assert np.array_equal(_bits(np.stack(got)), _bits(want))


def test_rank_order_comparator_differs_for_random_floats():
    """collkit's bench oracle folds in rank order; for random floats the ring
    order differs on many elements, so parity must use the
    algorithm's own order."""
    rng = np.random.default_rng(0)
    p = 8
    ins = [rng.standard_normal(4096 * p).astype(np.float32) for _ in range(p)]
    ring = np.stack(oracle.ring_reduce_scatter(ins))
    rank = np.stack(oracle.expected_reduce_scatter(ins))
    assert (ring != rank).sum() > 1000
    assert np.array_equal(np.stack(oracle.direct_reduce_scatter(ins, "f32", "rank")), rank)


def test_reference_known_answers():
    # collectives (pkg/tests/test_collectives.py:102-111, 85-90, 154-158)
    assert [list(x) for x in oracle.ring_reduce_scatter([np.array([1, 2], np.float32), np.array([3, 4], np.float32)])] == [[4], [6]]
    outs = oracle.ring_reduce_scatter([np.full(4, r, np.float32) for r in range(4)])
    assert all(list(o) == [6.0] for o in outs)
    outs = oracle.ring_all_gather([np.array([r], np.float32) for r in range(4)])
    assert all(list(o) == [0, 1, 2, 3] for o in outs)
    outs = oracle.rechalf_reduce_scatter([np.array([1, 2], np.float32), np.array([3, 4], np.float32)])
    assert [list(o) for o in outs] == [[4], [6]]
    # shuffles (pkg/tests/test_hierarchy.py:45-62)
    lm = np.array([0.0, 2.0, 1.0, 3.0], np.float32)
    assert list(oracle.shuffle_local_major_to_global(lm, 2, 2, 1)) == [0, 1, 2, 3]
    assert list(oracle.shuffle_global_to_local_major(np.arange(4, dtype=np.float32), 2, 2, 1)) == list(lm)
    # hierarchical all-ones 2x2 (test_hierarchy.py:181-187)
    outs = oracle.hier_reduce_scatter([np.ones(4, np.float32) for _ in range(4)], 2, 2)
    assert all(list(o) == [4.0] for o in outs)


def test_shuffle_golden():
    for key in [k[: -len("/in")] for k in Z.files if k.startswith("shuffle_") and k.endswith("/in")]:
        dims, b = key[len("shuffle_"):].split("_b")
        N, M = map(int, dims.split("x"))
        buf = Z[key + "/in"]
        assert np.array_equal(oracle.shuffle_local_major_to_global(buf, N, M, int(b)), Z[key + "/l2g"])
        assert np.array_equal(oracle.shuffle_global_to_local_major(buf, N, M, int(b)), Z[key + "/g2l"])


# --- bf16 helpers --------------------------------------------------------------
def test_bf16_rounding_is_rne():
    import torch

    rng = np.random.default_rng(1)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32),
                        np.array([0.0, -0.0, 1e-40, -1e-40, 3.4e38, np.inf, -np.inf], np.float32)])
    ours = oracle.f32_to_bf16(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    assert np.array_equal(oracle.bf16_to_f32(ours), torch.from_numpy(ref.view(np.int16)).view(torch.bfloat16).float().numpy())


def test_bf16_wire_semantics_within_tolerance():
    """Step-wise bf16 (a rounding per hop) stays within p * 2^-8 * sum|x| of
    the exact sum — the bound the GPU tests assert."""
    rng = np.random.default_rng(2)
    p, n = 8, 2048
    ins = [oracle.f32_to_bf16(rng.standard_normal(n * p).astype(np.float32)) for _ in range(p)]
    f = [oracle.bf16_to_f32(x).astype(np.float64) for x in ins]
    for fn in (oracle.ring_reduce_scatter, oracle.rechalf_reduce_scatter):
        outs = fn(ins, "bf16")
        for r in range(p):
            exact = sum(x[r * n:(r + 1) * n] for x in f)
            mag = sum(np.abs(x[r * n:(r + 1) * n]) for x in f)
            err = np.abs(oracle.bf16_to_f32(outs[r]).astype(np.float64) - exact)
            assert np.all(err <= p * 2.0 ** -8 * mag + 1e-30)


def test_schedule_restatement_matches_golden():
    for c in fixtures.schedules():
        got = oracle.build_schedule(c["collective"], c["algorithm"], c["m_bytes"], c["N"], c["M"], c["inter"])
        want = [sorted(tuple(m) for m in s) for s in c["steps"]]
        assert [sorted(tuple(m) for m in s) for s in got] == want
