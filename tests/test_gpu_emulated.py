"""GPU parity tests, emulation mode: p ranks of one process on cuda:0, every
collective ONE cooperative launch of the same kernels the multi-GPU path runs
(peer pointers are local). Called through the reference-shaped public API
(``run_ranks`` + ``ring_all_gather(comm, buf)`` ...), checked bit-for-bit
against golden vectors produced by the real reference (collkit) and against
the oracle."""
import numpy as np
import pytest
import torch

import oracle
from tests.golden import fixtures

pytestmark = pytest.mark.gpu

P = None  # imported lazily so collection works without the library


def _pkg():
    global P
    if P is None:
        import paper_2504_18658_b200 as pkg

        P = pkg
    return P


CASES = fixtures.cases()
Z = fixtures.arrays()


def _flat_fn(op, algo):
    pkg = _pkg()
    return {
        ("ag", "ring"): pkg.ring_all_gather,
        ("ag", "recursive"): pkg.recdbl_all_gather,
        ("rs", "ring"): pkg.ring_reduce_scatter,
        ("rs", "recursive"): pkg.rechalf_reduce_scatter,
    }[(op, algo)]


def _bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("case", [c for c in CASES if c["algo"] != "hierarchical"], ids=lambda c: c["name"])
def test_flat_matches_reference_golden(case):
    pkg = _pkg()
    ins = Z[case["name"] + "/in"]
    want = Z[case["name"] + "/out"]
    p = case["p"]
    fn = _flat_fn(case["op"], case["algo"])
    outs = pkg.run_ranks(p, lambda c: fn(c, ins[c.rank]))
    for r in range(p):
        assert outs[r].dtype == np.float32
        assert _bits_equal(outs[r], want[r]), (case["name"], r)


@pytest.mark.parametrize("case", [c for c in CASES if c["algo"] != "hierarchical"], ids=lambda c: c["name"])
def test_direct_matches_reference_golden(case):
    """One-shot kernels: AG identical; RS folded in the named algorithm's
    order is bit-identical to that algorithm's reference output."""
    pkg = _pkg()
    ins = Z[case["name"] + "/in"]
    want = Z[case["name"] + "/out"]
    p = case["p"]
    if case["op"] == "ag":
        outs = pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, ins[c.rank]))
    else:
        outs = pkg.run_ranks(p, lambda c: pkg.direct_reduce_scatter(c, ins[c.rank], order=case["algo"]))
    for r in range(p):
        assert _bits_equal(outs[r], want[r]), (case["name"], r)


@pytest.mark.parametrize("case", [c for c in CASES if c["algo"] == "hierarchical"], ids=lambda c: c["name"])
def test_hierarchical_matches_reference_golden(case):
    pkg = _pkg()
    ins = Z[case["name"] + "/in"]
    want = Z[case["name"] + "/out"]
    N, M = case["N"], case["M"]
    plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=case["inter"])
    fn = pkg.hier_all_gather if case["op"] == "ag" else pkg.hier_reduce_scatter
    outs = pkg.run_ranks(N * M, lambda c: fn(plan, c, ins[c.rank]))
    for r in range(N * M):
        assert _bits_equal(outs[r], want[r]), (case["name"], r)


# ---------------------------------------------------------------------------
# low precision: bit-exact against the oracle's wire semantics, and within the
# stated tolerance of the exact sum
# ---------------------------------------------------------------------------
def _bf16_inputs(p, n, seed):
    rng = np.random.default_rng(seed)
    return [oracle.f32_to_bf16(rng.standard_normal(n * p).astype(np.float32)) for _ in range(p)]


def _to_dev(bits, dtype):
    t = torch.from_numpy(bits.view(np.int16) if dtype == torch.bfloat16 else bits)
    return t.view(dtype).cuda()


def _from_dev(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


@pytest.mark.parametrize("p", [2, 4, 8, 16])
@pytest.mark.parametrize("algo", ["ring", "recursive", "direct"])
@pytest.mark.parametrize("n", [8, 1000, 4096 + 24])
def test_bf16_reduce_scatter(p, algo, n):
    pkg = _pkg()
    ins = _bf16_inputs(p, n, seed=p * 1000 + n)
    fns = {
        "ring": pkg.ring_reduce_scatter,
        "recursive": pkg.rechalf_reduce_scatter,
        "direct": lambda c, x: pkg.direct_reduce_scatter(c, x, order="ring"),
    }
    outs = pkg.run_ranks(p, lambda c: _from_dev(fns[algo](c, _to_dev(ins[c.rank], torch.bfloat16))))
    if algo == "direct":
        want = oracle.direct_reduce_scatter(ins, "bf16", "ring")
    else:
        want = (oracle.ring_reduce_scatter if algo == "ring" else oracle.rechalf_reduce_scatter)(ins, "bf16")
    # exact float64 sum for the tolerance bound |y - s| <= p * 2^-8 * sum|x|
    f = [oracle.bf16_to_f32(x).astype(np.float64) for x in ins]
    for r in range(p):
        assert np.array_equal(outs[r], want[r]), (algo, p, r)
        exact = sum(x[r * n : (r + 1) * n] for x in f)
        mag = sum(np.abs(x[r * n : (r + 1) * n]) for x in f)
        err = np.abs(oracle.bf16_to_f32(outs[r]).astype(np.float64) - exact)
        assert np.all(err <= p * 2.0**-8 * mag + 1e-30)


@pytest.mark.parametrize("p", [2, 8])
@pytest.mark.parametrize("algo", ["ring", "recursive", "direct"])
def test_f16_reduce_scatter(p, algo):
    pkg = _pkg()
    rng = np.random.default_rng(p)
    n = 520
    ins = [rng.standard_normal(n * p).astype(np.float16) for _ in range(p)]
    fns = {
        "ring": pkg.ring_reduce_scatter,
        "recursive": pkg.rechalf_reduce_scatter,
        "direct": lambda c, x: pkg.direct_reduce_scatter(c, x, order="recursive"),
    }
    outs = pkg.run_ranks(p, lambda c: fns[algo](c, torch.from_numpy(ins[c.rank]).cuda()).cpu().numpy())
    if algo == "direct":
        want = oracle.direct_reduce_scatter(ins, "f16", "recursive")
    else:
        want = (oracle.ring_reduce_scatter if algo == "ring" else oracle.rechalf_reduce_scatter)(ins, "f16")
    for r in range(p):
        assert _bits_equal(outs[r], want[r])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.int64, torch.uint8, torch.float64])
@pytest.mark.parametrize("algo", ["ring", "recursive", "direct"])
def test_all_gather_any_dtype_byte_exact(dtype, algo):
    pkg = _pkg()
    p, n = 8, 333
    g = torch.Generator().manual_seed(5)
    ins = [torch.randint(0, 200, (n,), generator=g).to(dtype) for _ in range(p)]
    fn = {"ring": pkg.ring_all_gather, "recursive": pkg.recdbl_all_gather, "direct": pkg.direct_all_gather}[algo]
    outs = pkg.run_ranks(p, lambda c: fn(c, ins[c.rank].cuda()).cpu())
    want = torch.cat(ins)
    for r in range(p):
        assert outs[r].dtype == dtype and torch.equal(outs[r], want)


# ---------------------------------------------------------------------------
# large sizes: size-independent properties (vectorised, pipelined path)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("algo", ["ring", "recursive", "direct"])
def test_large_fp32_integer_sums_exact(p, algo):
    """Integer-valued fp32 (the reference's test domain) sums are exact in any
    order: RS chunks must equal the exact sum; AG must reassemble the inputs."""
    pkg = _pkg()
    n = (1 << 20) + 96
    g = torch.Generator().manual_seed(p)
    ins = [torch.randint(-1024, 1025, (n * p,), generator=g).float().cuda() for _ in range(p)]
    rs = {"ring": pkg.ring_reduce_scatter, "recursive": pkg.rechalf_reduce_scatter,
          "direct": pkg.direct_reduce_scatter}[algo]
    outs = pkg.run_ranks(p, lambda c: rs(c, ins[c.rank]))
    total = sum(x.double() for x in ins)
    for r in range(p):
        assert torch.equal(outs[r].double(), total[r * n : (r + 1) * n])
    ag = {"ring": pkg.ring_all_gather, "recursive": pkg.recdbl_all_gather, "direct": pkg.direct_all_gather}[algo]
    outs = pkg.run_ranks(p, lambda c: ag(c, ins[c.rank][:n]))
    want = torch.cat([x[:n] for x in ins])
    for r in range(p):
        assert torch.equal(outs[r], want)


@pytest.mark.parametrize("p", [4, 8])
def test_large_fp32_normal_bit_exact_vs_oracle(p):
    pkg = _pkg()
    n = 300_000
    rng = np.random.default_rng(99)
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    for algo, fn, ref in [
        ("ring", pkg.ring_reduce_scatter, oracle.ring_reduce_scatter),
        ("recursive", pkg.rechalf_reduce_scatter, oracle.rechalf_reduce_scatter),
    ]:
        outs = pkg.run_ranks(p, lambda c: fn(c, ins[c.rank]))
        want = ref(ins)
        for r in range(p):
            assert _bits_equal(outs[r], want[r]), (algo, r)


@pytest.fixture
def small_pipeline(monkeypatch):
    """Pipelined host path with small slices (several slices per call), and
    a spy that records how many slices each pipelined call used."""
    from paper_2504_18658_b200 import collectives as C

    monkeypatch.setattr(C, "PIPE_MIN_BYTES", 256 << 10)
    monkeypatch.setattr(C, "PIPE_SLICE_BYTES", 64 << 10)
    used = []
    real = C._pipeline_slices

    def spy(*a):
        sl = real(*a)
        used.append(0 if sl is None else len(sl))
        return sl

    monkeypatch.setattr(C, "_pipeline_slices", spy)
    return used


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("algo", ["ring", "recursive", "direct"])
def test_host_pipeline_reduce_scatter_bit_exact(p, algo, small_pipeline):
    """Host inputs large enough to be sliced: numpy (pageable) and pinned
    tensors give the same bits as the oracle of the named algorithm."""
    pkg = _pkg()
    n = 50_003  # ragged: the last slice is short and unaligned
    rng = np.random.default_rng(p)
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    fn = {"ring": pkg.ring_reduce_scatter, "recursive": pkg.rechalf_reduce_scatter,
          "direct": pkg.direct_reduce_scatter}[algo]
    want = (oracle.rechalf_reduce_scatter if algo == "recursive" else oracle.ring_reduce_scatter)(ins)
    outs = pkg.run_ranks(p, lambda c: fn(c, ins[c.rank]))
    pins = [torch.from_numpy(x).pin_memory() for x in ins]
    outs_pinned = pkg.run_ranks(p, lambda c: fn(c, pins[c.rank]))
    assert small_pipeline and min(small_pipeline) >= 3, small_pipeline
    for r in range(p):
        assert _bits_equal(outs[r], want[r]), r
        assert outs_pinned[r].is_pinned() and _bits_equal(outs_pinned[r].numpy(), want[r]), r


@pytest.mark.parametrize("p", [2, 4, 8])
def test_host_pipeline_bf16_matches_device_path(p, small_pipeline):
    pkg = _pkg()
    n = 70_001
    g = torch.Generator().manual_seed(p)
    ins = [torch.randn(n * p, generator=g).to(torch.bfloat16) for _ in range(p)]
    host = pkg.run_ranks(p, lambda c: pkg.rechalf_reduce_scatter(c, ins[c.rank].pin_memory()))
    dev = pkg.run_ranks(p, lambda c: pkg.rechalf_reduce_scatter(c, ins[c.rank].cuda()))
    assert small_pipeline and max(small_pipeline) >= 3
    for r in range(p):
        assert torch.equal(host[r].view(torch.int16), dev[r].cpu().view(torch.int16)), r


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("dtype", [np.float32, np.int32, np.uint8])
def test_host_pipeline_all_gather_byte_exact(p, dtype, small_pipeline):
    pkg = _pkg()
    n = 300_007 if dtype == np.uint8 else 200_011
    rng = np.random.default_rng(7)
    ins = [rng.integers(0, 255, n).astype(dtype) for _ in range(p)]
    fns = [pkg.ring_all_gather, pkg.direct_all_gather] + ([pkg.recdbl_all_gather] if p & (p - 1) == 0 else [])
    for fn in fns:
        outs = pkg.run_ranks(p, lambda c: fn(c, torch.from_numpy(ins[c.rank]).pin_memory()))
        want = np.concatenate(ins)
        for r in range(p):
            assert np.array_equal(outs[r].numpy(), want), (fn.__name__, r)
    assert small_pipeline and min(small_pipeline) >= 3


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("item_kib", [16, 64])
def test_direct_dynamic_work_items_bit_exact(p, item_kib):
    """Direct kernels with dynamically claimed work items (param item_kib):
    AG pull / push and RS pull / push give the oracle's bits."""
    pkg = _pkg()
    n = 300_001
    rng = np.random.default_rng(p + item_kib)
    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    want_ag = np.concatenate(ag_in)
    want_rs = oracle.ring_reduce_scatter(rs_in)

    def body(c):
        w = c.world
        w.set_param("item_kib", item_kib)
        res = []
        try:
            for v in (0, 1):
                w.set_param("ag_variant", v)
                w.set_param("rs_variant", v)
                res.append(pkg.direct_all_gather(c, torch.from_numpy(ag_in[c.rank]).cuda()).cpu().numpy())
                res.append(pkg.direct_reduce_scatter(c, torch.from_numpy(rs_in[c.rank]).cuda()).cpu().numpy())
        finally:
            w.set_param("item_kib", 0)
            w.set_param("ag_variant", -1)
            w.set_param("rs_variant", -1)
        return res

    outs = pkg.run_ranks(p, body)
    for r in range(p):
        for i, got in enumerate(outs[r]):
            assert _bits_equal(got, want_ag if i % 2 == 0 else want_rs[r]), (r, i)


@pytest.mark.parametrize("p", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("order", ["ring", "recursive", "rank"])
def test_direct_pipelined_push_bit_exact(p, order):
    """rs_variant 5 (pusher / folder CTAs, sub-slice pipelined): fp32 in every
    fold order and bf16 give the oracle's bits; odd and even grids."""
    if order == "recursive" and p & (p - 1):
        pytest.skip("recursive order needs a power of two")
    pkg = _pkg()
    n = 100_003 if p < 16 else 20_011
    rng = np.random.default_rng(p * 7 + len(order))
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    ins_bf = [oracle.f32_to_bf16(x) for x in ins]
    want = oracle.direct_reduce_scatter(ins, "f32", order)
    want_bf = oracle.direct_reduce_scatter(ins_bf, "bf16", order)

    def body(c):
        w = c.world
        w.set_param("rs_variant", 5)
        try:
            out = []
            for ctas in (0, 7):  # auto (even) and an odd grid (spare CTA)
                w.set_param("ctas", ctas)
                out.append(pkg.direct_reduce_scatter(c, torch.from_numpy(ins[c.rank]).cuda(), order=order).cpu().numpy())
                xb = torch.from_numpy(ins_bf[c.rank].view(np.int16)).view(torch.bfloat16).cuda()
                yb = pkg.direct_reduce_scatter(c, xb, order=order)
                out.append(yb.view(torch.int16).cpu().numpy().view(np.uint16))
        finally:
            w.set_param("rs_variant", -1)
            w.set_param("ctas", 0)
        return out

    outs = pkg.run_ranks(p, body)
    for r in range(p):
        for i, got in enumerate(outs[r]):
            assert _bits_equal(got, (want if i % 2 == 0 else want_bf)[r]), (r, i)


def test_back_to_back_calls_reuse_buffers():
    """Epoch flags never reset: many consecutive calls stay correct."""
    pkg = _pkg()
    p, n = 8, 50_000
    g = torch.Generator().manual_seed(3)

    def body(c):
        res = []
        for it in range(20):
            x = torch.full((n * p,), float(it + c.rank), device="cuda")
            algo = ["direct", "ring", "recursive"][it % 3]
            y = pkg.reduce_scatter(c, x, algorithm=algo)
            res.append(float(y[0].item()))
        return res

    outs = pkg.run_ranks(p, body)
    for r in range(p):
        for it in range(20):
            assert outs[r][it] == sum(it + q for q in range(p))


# ---------------------------------------------------------------------------
# edge cases and errors (reference contract)
# ---------------------------------------------------------------------------
def test_p1_returns_copy():
    pkg = _pkg()
    x = np.array([5.0], np.float32)
    out = pkg.run_ranks(1, lambda c: pkg.ring_all_gather(c, x))
    assert np.array_equal(out[0], [5.0]) and out[0] is not x


def test_empty_payloads():
    pkg = _pkg()
    for fn in (pkg.ring_all_gather, pkg.recdbl_all_gather, pkg.direct_all_gather):
        outs = pkg.run_ranks(4, lambda c: fn(c, np.zeros(0, np.float32)))
        assert all(o.size == 0 for o in outs)
    for fn in (pkg.ring_reduce_scatter, pkg.rechalf_reduce_scatter, pkg.direct_reduce_scatter):
        outs = pkg.run_ranks(4, lambda c: fn(c, np.zeros(0, np.float32)))
        assert all(o.size == 0 for o in outs)
    # device tensors too (no host round trip)
    outs = pkg.run_ranks(4, lambda c: pkg.all_gather(c, torch.zeros(0, device="cuda"), algorithm="direct"))
    assert all(o.numel() == 0 for o in outs)


def test_errors():
    pkg = _pkg()
    from paper_2504_18658_b200.errors import LengthMismatch, NonPowerOfTwo, NotDivisible

    with pytest.raises(NotDivisible):
        pkg.run_ranks(2, lambda c: pkg.ring_reduce_scatter(c, np.zeros(3, np.float32)))
    with pytest.raises(NonPowerOfTwo):
        pkg.run_ranks(3, lambda c: pkg.recdbl_all_gather(c, np.zeros(2, np.float32)))
    with pytest.raises(NonPowerOfTwo):
        pkg.run_ranks(6, lambda c: pkg.rechalf_reduce_scatter(c, np.zeros(12, np.float32)))
    sizes = [4, 2]
    with pytest.raises(LengthMismatch):
        pkg.run_ranks(2, lambda c: pkg.ring_all_gather(c, np.zeros(sizes[c.rank], np.float32)))
    # still usable afterwards
    outs = pkg.run_ranks(2, lambda c: pkg.ring_all_gather(c, np.full(2, c.rank, np.float32)))
    assert np.array_equal(outs[1], [0, 0, 1, 1])


@pytest.mark.parametrize("algo,n", [("direct", 4096), ("direct", 1 << 22), ("ring", 4096), ("recursive", 4096)])
def test_device_side_signature_mismatch_aborts_cleanly(algo, n):
    """A rank whose call signature differs (what a cross-rank size mismatch
    looks like on a real multi-GPU job) must make every rank raise
    LengthMismatch via the device flag protocol — not hang."""
    pkg = _pkg()
    from paper_2504_18658_b200 import _lib
    from paper_2504_18658_b200.errors import LengthMismatch

    w = pkg.emulated_world(4)
    _lib.lib().pccl_emu_debug_meta_skew(w.handle, 2, 0x1234)
    try:
        with pytest.raises(LengthMismatch):
            pkg.run_ranks(4, lambda c: pkg.reduce_scatter(c, torch.ones(n, device="cuda"), algorithm=algo))
        with pytest.raises(LengthMismatch):  # all-gather too (LL header / READY word)
            pkg.run_ranks(4, lambda c: pkg.all_gather(c, torch.ones(n // 4, device="cuda"), algorithm=algo))
    finally:
        _lib.lib().pccl_emu_debug_meta_skew(w.handle, 2, 0)
        w.reset_flags()
    outs = pkg.run_ranks(4, lambda c: pkg.reduce_scatter(c, torch.ones(n, device="cuda"), algorithm=algo))
    assert all(torch.all(o == 4) for o in outs)


def test_shuffles_match_reference_golden():
    pkg = _pkg()
    for key in [k[: -len("/in")] for k in Z.files if k.startswith("shuffle_") and k.endswith("/in")]:
        dims, b = key[len("shuffle_"):].split("_b")
        N, M = map(int, dims.split("x"))
        buf = Z[key + "/in"]
        assert np.array_equal(pkg.shuffle_local_major_to_global(buf, N, M, int(b)), Z[key + "/l2g"])
        assert np.array_equal(pkg.shuffle_global_to_local_major(buf, N, M, int(b)), Z[key + "/g2l"])


def test_reduce_inplace_matches_scalar_loop():
    pkg = _pkg()
    rng = np.random.default_rng(3)
    a = rng.standard_normal(64).astype(np.float32)
    b = rng.standard_normal(64).astype(np.float32)
    want = np.array([float(a[i]) + float(b[i]) for i in range(64)], dtype=np.float32)
    acc = a.copy()
    assert pkg.reduce_inplace(acc, b) is acc
    assert np.array_equal(acc, want)


def test_hier_block_trace_and_all_ones():
    pkg = _pkg()
    plan = pkg.HierPlan(topo=pkg.Topology(2, 2), inter_alg="ring")
    outs = pkg.run_ranks(4, lambda c: pkg.hier_all_gather(plan, c, np.array([float(c.rank)], np.float32)))
    assert all(np.array_equal(o, [0, 1, 2, 3]) for o in outs)
    outs = pkg.run_ranks(4, lambda c: pkg.hier_reduce_scatter(pkg.HierPlan(topo=pkg.Topology(2, 2)), c,
                                                              np.ones(4, np.float32)))
    assert all(np.array_equal(o, [4.0]) for o in outs)


@pytest.mark.parametrize("members", [(1, 3, 5, 7), (4, 5, 6, 7), (6, 2, 4, 0)])
@pytest.mark.parametrize("inter", ["ring", "recursive"])
def test_hierarchical_on_a_sub_communicator(members, inter):
    """hierarchy.py:129-134 only requires the communicator's size to match the
    topology: a 4-member sub-communicator of an 8-rank world runs a 2x2
    hierarchical AG / RS whose topology rank g is member g."""
    pkg = _pkg()
    p, n = len(members), 1000
    rng = np.random.default_rng(5)
    ag_in = {m: rng.standard_normal(n).astype(np.float32) for m in members}
    rs_in = {m: rng.standard_normal(n * p).astype(np.float32) for m in members}
    plan = pkg.HierPlan(topo=pkg.Topology(2, 2), inter_alg=inter)

    def body(c):
        sub = c.subgroup(members, 9)
        if sub is None:
            return None
        me = members[sub.rank]
        return (pkg.hier_all_gather(plan, sub, ag_in[me]), pkg.hier_reduce_scatter(plan, sub, rs_in[me]))

    outs = pkg.run_ranks(8, body)
    want_ag = oracle.hier_all_gather([ag_in[m] for m in members], 2, 2, inter)
    want_rs = oracle.hier_reduce_scatter([rs_in[m] for m in members], 2, 2, inter)
    for w in range(8):
        if w not in members:
            assert outs[w] is None
            continue
        g = members.index(w)
        assert _bits_equal(outs[w][0], want_ag[g]), (w, "ag")
        assert _bits_equal(outs[w][1], want_rs[g]), (w, "rs")


def test_hierarchical_world_size_mismatch_raises():
    pkg = _pkg()
    plan = pkg.HierPlan(topo=pkg.Topology(2, 2))
    with pytest.raises(pkg.errors.LengthMismatch):
        pkg.run_ranks(2, lambda c: pkg.hier_all_gather(plan, c, np.zeros(2, np.float32)))


def test_registered_torch_tensors_are_zero_copy():
    """World.register (emulation: one caching-allocator tensor per rank):
    collectives bind the registered buffers without staging and stay exact."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    p, n = 4, 70001
    w = emulated_world(p, 0)
    rng = np.random.default_rng(11)
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    xs = [torch.from_numpy(x).cuda() for x in ins]
    ys = [torch.empty(n, device="cuda") for _ in range(p)]
    zs = [torch.empty(n * p, device="cuda") for _ in range(p)]
    with w.register(xs), w.register(ys), w.register(zs):
        w.set_param("staged_bytes", 0)
        for algo in ("direct", "ring", "recursive"):
            order = "recursive" if algo == "recursive" else "ring"
            pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, xs[c.rank], algorithm=algo, order=order, out=ys[c.rank]))
            want = oracle.rechalf_reduce_scatter(ins) if algo == "recursive" else oracle.ring_reduce_scatter(ins)
            for r in range(p):
                assert _bits_equal(ys[r].cpu().numpy(), want[r]), (algo, r)
            pkg.run_ranks(p, lambda c: pkg.all_gather(c, ys[c.rank], algorithm=algo, out=zs[c.rank]))
            for r in range(p):
                assert _bits_equal(zs[r].cpu().numpy(), np.concatenate([y.cpu().numpy() for y in ys])), (algo, r)
        torch.cuda.synchronize()
        assert w.get_param("staged_bytes") == 0
    # (emulated rows bind every rank's own pointer, so unregistered buffers are
    # not staged here either; the real-mode worker checks the staging counter)


def test_symmetric_heap_allocates_deterministically_and_reuses():
    from paper_2504_18658_b200.communicator import emulated_world

    pkg = _pkg()
    p = 4
    w = emulated_world(p, 0)
    heap = w.heap(8 << 20)
    free0 = heap.bytes_free()
    a = heap.empty(1000, torch.float32)
    b = heap.empty(3000, torch.bfloat16)
    assert len(a) == p and a[0].data_ptr() - heap.segment.ptr(0) == 0
    assert b[0].data_ptr() - heap.segment.ptr(0) == 4096  # 4000 B rounded to 256
    for r in range(p):  # every rank's block at the same offset
        assert a[r].data_ptr() - heap.segment.ptr(r) == 0 and b[r].data_ptr() - heap.segment.ptr(r) == 4096
    x = heap.empty(4096 * p, torch.float32)
    y = heap.empty(4096, torch.float32)
    for r in range(p):
        x[r].fill_(float(r + 1))
    w.set_param("staged_bytes", 0)
    pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, x[c.rank], algorithm="direct", out=y[c.rank]))
    torch.cuda.synchronize()
    assert w.get_param("staged_bytes") == 0
    assert all(float(y[r][0]) == p * (p + 1) / 2 for r in range(p))
    del a, b, x, y
    import gc

    gc.collect()
    heap.empty(16, torch.float32)  # runs the queued releases
    assert heap.bytes_free() == free0 - 256
    with pytest.raises(pkg.errors.OutOfMemory):
        heap.empty(16 << 20, torch.float32)


def test_world_empty_segments_are_released():
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(2, 0)
    before = len(w._segments)
    for _ in range(100):  # more than the old 64-segment table without releases
        t = w.empty(1 << 16, torch.float32)
        del t
    import gc

    gc.collect()
    w._run_pending()
    assert len(w._segments) <= before + 1


@pytest.mark.parametrize("p", [2, 4, 8, 16])
@pytest.mark.parametrize("items_per_cta", [1, 2, 4])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_rechalf_work_items_bit_exact(p, items_per_cta, dtype):
    """rs_variant 7 (recursive halving with per-step dynamic work items):
    bit-identical to the oracle's butterfly (fp32) / wire rounding (bf16)."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(p, 0)
    rng = np.random.default_rng(p * 10 + items_per_cta)
    n = 70001 * 8 // p * p // p + 5
    ins32 = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    ins = [oracle.f32_to_bf16(x) for x in ins32] if dtype == "bf16" else ins32
    want = oracle.rechalf_reduce_scatter(ins, dtype)
    w.set_param("rs_variant", 7)
    w.set_param("items_per_cta", items_per_cta)
    w.set_param("ll_max", 0)
    try:
        for _ in range(2):
            if dtype == "bf16":
                outs = pkg.run_ranks(p, lambda c: pkg.rechalf_reduce_scatter(
                    c, torch.from_numpy(ins[c.rank].view(np.int16)).view(torch.bfloat16).cuda())
                    .view(torch.int16).cpu().numpy().view(np.uint16))
            else:
                outs = pkg.run_ranks(p, lambda c: pkg.rechalf_reduce_scatter(c, ins[c.rank]))
            for r in range(p):
                assert _bits_equal(outs[r], want[r]), r
    finally:
        w.set_param("rs_variant", -1)
        w.set_param("items_per_cta", 2)
        w.set_param("ll_max", -1)


@pytest.mark.parametrize("grid", [(2, 4), (4, 2), (2, 8), (1, 4), (4, 4)])
@pytest.mark.parametrize("intra", [-1, 0, 1])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_hierarchical_intra_direct_is_bit_identical(grid, intra, dtype):
    """The intra phase as the one-step direct kernel (param hier_intra, auto
    for M >= 3): ring add order and, in bf16, the ring's per-step rounding —
    bit-identical to the oracle's hier_reduce_scatter / hier_all_gather."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    N, M = grid
    p = N * M
    w = emulated_world(p, 0)
    rng = np.random.default_rng(p + 10 * (intra + 1) + (dtype == "bf16"))
    n = 777
    rs32 = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    ag32 = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    rs = [oracle.f32_to_bf16(x) for x in rs32] if dtype == "bf16" else rs32
    ag = [oracle.f32_to_bf16(x) for x in ag32] if dtype == "bf16" else ag32

    def dev(x):
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda() if dtype == "bf16" else \
            torch.from_numpy(x).cuda()

    def host(t):
        return t.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else t.cpu().numpy()

    w.set_param("hier_intra", intra)
    try:
        for inter in ["ring"] + (["recursive"] if N & (N - 1) == 0 else []):
            plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=inter)
            got = pkg.run_ranks(p, lambda c: host(pkg.hier_reduce_scatter(plan, c, dev(rs[c.rank]))))
            want = oracle.hier_reduce_scatter(rs, N, M, inter, dtype)
            for r in range(p):
                assert _bits_equal(got[r], want[r]), ("rs", inter, r)
            got = pkg.run_ranks(p, lambda c: host(pkg.hier_all_gather(plan, c, dev(ag[c.rank]))))
            want = oracle.hier_all_gather(ag, N, M, inter)
            for r in range(p):
                assert _bits_equal(got[r], want[r]), ("ag", inter, r)
    finally:
        w.set_param("hier_intra", -1)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("n", [40, 70001])  # LL protocol / flag protocol
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("order", ["ring", "recursive"])
def test_direct_wire_rounding_equals_stepwise(p, n, dtype, order):
    """order "<name>/wire": the one-step direct kernel rounds where the
    step-wise algorithm does — bit-identical to ring / recursive halving."""
    pkg = _pkg()
    rng = np.random.default_rng(p * n)
    x32 = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    if dtype == "bf16":
        ins = [oracle.f32_to_bf16(x) for x in x32]
        dev = lambda x: torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()  # noqa: E731
        host = lambda t: t.view(torch.int16).cpu().numpy().view(np.uint16)  # noqa: E731
    else:
        ins = [x.astype(np.float16) for x in x32]
        dev = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
        host = lambda t: t.cpu().numpy()  # noqa: E731
    want = (oracle.ring_reduce_scatter(ins, dtype) if order == "ring" else oracle.rechalf_reduce_scatter(ins, dtype))
    got = pkg.run_ranks(p, lambda c: host(pkg.direct_reduce_scatter(c, dev(ins[c.rank]), order=order + "/wire")))
    for r in range(p):
        assert _bits_equal(got[r], want[r]), r
    # auto never changes bits with the data movement it picks
    got = pkg.run_ranks(p, lambda c: host(pkg.reduce_scatter(c, dev(ins[c.rank]), algorithm="auto", order=order)))
    for r in range(p):
        assert _bits_equal(got[r], want[r]), r
