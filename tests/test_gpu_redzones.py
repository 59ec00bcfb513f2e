"""Out-of-bounds write detection without compute-sanitizer (closed on this
pool): every buffer a collective touches sits between two guard regions
filled with a byte pattern; after the call the guards must be intact and the
output must match the oracle. Covers every algorithm x data-movement variant
x dtype, odd element counts (scalar tail paths), misaligned views (the
non-vectorised kernels and LL bounce buffers) and symmetric buffers (zero-copy
push / pull paths), emulated p = 2, 3, 4, 8."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
PAT = 0xA5


def _pkg():
    import paper_2504_18658_b200 as pkg

    return pkg


def _guarded(numel, dtype, kind, world=None):
    """(buffers, check) — buffers[r] is the payload view of rank r."""
    es = torch.empty(0, dtype=dtype).element_size()
    g = GUARD // es
    p = world.nranks
    if kind == "sym":
        bases = world.empty(numel + 2 * g, dtype)
    else:
        shift = 1 if kind == "misaligned" else 0
        bases = [torch.empty(numel + 2 * g + shift, dtype=dtype, device="cuda")[shift:] for _ in range(p)]
    for b in bases:
        b.view(torch.uint8).fill_(PAT)
    bufs = [b[g: g + numel] for b in bases]

    def intact():
        for b in bases:
            u = b.view(torch.uint8)
            head, tail = u[: g * es], u[(g + numel) * es:]
            if not (bool((head == PAT).all()) and bool((tail == PAT).all())):
                return False
        return True

    return bufs, intact


def _bits(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 3, 1001, 4099, 70001])
@pytest.mark.parametrize("kind", ["sym", "plain", "misaligned"])
def test_all_gather_writes_only_its_output(p, n, kind):
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(p, 0)
    rng = np.random.default_rng(n + p)
    ins = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    algos = ["direct", "ring"] + (["recursive"] if p & (p - 1) == 0 else [])
    for algo in algos:
        xs, x_ok = _guarded(n, torch.float32, kind, w)
        ys, y_ok = _guarded(n * p, torch.float32, kind, w)
        for r in range(p):
            xs[r].copy_(torch.from_numpy(ins[r]))
        pkg.run_ranks(p, lambda c: pkg.all_gather(c, xs[c.rank], algorithm=algo, out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), (algo, "guard overwritten")
        want = np.concatenate(ins)
        for r in range(p):
            assert np.array_equal(_bits(ys[r]).view(np.uint8), want.view(np.uint8)), (algo, r)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 3, 1001, 4099, 70001])
@pytest.mark.parametrize("kind", ["sym", "plain", "misaligned"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_reduce_scatter_writes_only_its_output(p, n, kind, dtype):
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(p, 0)
    rng = np.random.default_rng(n * 7 + p)
    ins32 = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    dn = "bf16" if dtype == torch.bfloat16 else "f32"
    ins = [oracle.f32_to_bf16(x) for x in ins32] if dn == "bf16" else ins32
    algos = ["direct", "ring"] + (["recursive"] if p & (p - 1) == 0 else [])
    for algo in algos:
        xs, x_ok = _guarded(n * p, dtype, kind, w)
        ys, y_ok = _guarded(n, dtype, kind, w)
        for r in range(p):
            src = torch.from_numpy(ins[r].view(np.int16)).view(torch.bfloat16) if dn == "bf16" else \
                torch.from_numpy(ins[r])
            xs[r].copy_(src)
        order = "recursive" if algo == "recursive" else "ring"
        pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, xs[c.rank], algorithm=algo, order=order, out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), (algo, "guard overwritten")
        want = {"ring": oracle.ring_reduce_scatter(ins, dn), "recursive": oracle.rechalf_reduce_scatter(ins, dn)
                if algo == "recursive" else None,
                "direct": oracle.direct_reduce_scatter(ins, dn, order="ring")}[algo]
        for r in range(p):
            assert np.array_equal(_bits(ys[r]).view(np.uint8), np.asarray(want[r]).view(np.uint8)), (algo, r)


@pytest.mark.parametrize("variant", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [3, 4099, 70001])
def test_all_gather_variants_write_only_their_output(variant, n):
    """push / pull / TMA pull / TMA push data movement (flag protocol)."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    p = 4
    w = emulated_world(p, 0)
    rng = np.random.default_rng(n)
    ins = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    w.set_param("ll_max", 0)
    w.set_param("ag_variant", variant)
    try:
        for algo in (["direct"] if variant >= 2 else ["direct", "ring", "recursive"]):
            xs, x_ok = _guarded(n, torch.float32, "sym", w)
            ys, y_ok = _guarded(n * p, torch.float32, "sym", w)
            for r in range(p):
                xs[r].copy_(torch.from_numpy(ins[r]))
            pkg.run_ranks(p, lambda c: pkg.all_gather(c, xs[c.rank], algorithm=algo, out=ys[c.rank]))
            torch.cuda.synchronize()
            assert x_ok() and y_ok(), (algo, variant)
            for r in range(p):
                assert np.array_equal(_bits(ys[r]), np.concatenate(ins)), (algo, variant, r)
    finally:
        w.set_param("ag_variant", -1)
        w.set_param("ll_max", -1)


@pytest.mark.parametrize("kind", ["sym", "plain", "misaligned"])
@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("words", [1, 15, 61, 4099, 70000])
def test_ll128_all_gather_writes_only_its_output(kind, p, words):
    """LL128 line protocol: the last line's padding never reaches the output
    (every output, and every misaligned buffer bounced through staging, keeps
    its guards), and the payload is exact."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(p, 0)
    n = words * 2
    rng = np.random.default_rng(words + p)
    ins = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    w.set_param("ag_variant", 8)
    try:
        xs, x_ok = _guarded(n, torch.float32, kind, w)
        ys, y_ok = _guarded(n * p, torch.float32, kind, w)
        for r in range(p):
            xs[r].copy_(torch.from_numpy(ins[r]))
        pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, xs[c.rank], out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), (kind, p, words)
        for r in range(p):
            assert np.array_equal(_bits(ys[r]), np.concatenate(ins)), (kind, p, words, r)
    finally:
        w.set_param("ag_variant", -1)


@pytest.mark.parametrize("kind", ["sym", "plain", "misaligned"])
@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("words", [1, 61, 70000])
def test_ll128_reduce_scatter_writes_only_its_output(kind, p, words):
    """LL128 reduce-scatter: no write past the output chunk (padding of the
    last line), guards of inputs / outputs intact, result equal to the
    oracle's direct ring-order fold."""
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    w = emulated_world(p, 0)
    n = words * 2
    rng = np.random.default_rng(words * 7 + p)
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    w.set_param("rs_variant", 8)
    try:
        xs, x_ok = _guarded(n * p, torch.float32, kind, w)
        ys, y_ok = _guarded(n, torch.float32, kind, w)
        for r in range(p):
            xs[r].copy_(torch.from_numpy(ins[r]))
        pkg.run_ranks(p, lambda c: pkg.direct_reduce_scatter(c, xs[c.rank], order="ring", out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), (kind, p, words)
        want = oracle.direct_reduce_scatter(ins, "f32", order="ring")
        for r in range(p):
            assert np.array_equal(_bits(ys[r]).view(np.uint32), np.asarray(want[r]).view(np.uint32)), (kind, p, words, r)
    finally:
        w.set_param("rs_variant", -1)


@pytest.mark.parametrize("variant", [0, 1, 5])
@pytest.mark.parametrize("n", [3, 4099, 70001])
def test_reduce_scatter_variants_write_only_their_output(variant, n):
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    p = 4
    w = emulated_world(p, 0)
    rng = np.random.default_rng(n + 1)
    ins = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    w.set_param("ll_max", 0)
    w.set_param("rs_variant", variant)
    try:
        for algo in (["direct"] if variant == 5 else ["direct", "ring", "recursive"]):
            xs, x_ok = _guarded(n * p, torch.float32, "sym", w)
            ys, y_ok = _guarded(n, torch.float32, "sym", w)
            for r in range(p):
                xs[r].copy_(torch.from_numpy(ins[r]))
            order = "recursive" if algo == "recursive" else "ring"
            pkg.run_ranks(p, lambda c: pkg.reduce_scatter(c, xs[c.rank], algorithm=algo, order=order,
                                                          out=ys[c.rank]))
            torch.cuda.synchronize()
            assert x_ok() and y_ok(), (algo, variant)
            want = oracle.rechalf_reduce_scatter(ins) if algo == "recursive" else oracle.ring_reduce_scatter(ins)
            for r in range(p):
                assert np.array_equal(_bits(ys[r]), want[r]), (algo, variant, r)
    finally:
        w.set_param("rs_variant", -1)
        w.set_param("ll_max", -1)


@pytest.mark.parametrize("grid", [(2, 2), (2, 4), (4, 2)])
@pytest.mark.parametrize("n", [3, 4099])
def test_hierarchical_writes_only_its_output(grid, n):
    pkg = _pkg()
    from paper_2504_18658_b200.communicator import emulated_world

    N, M = grid
    p = N * M
    w = emulated_world(p, 0)
    rng = np.random.default_rng(n + 3)
    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    for inter in ("ring", "recursive"):
        plan = pkg.HierPlan(topo=pkg.Topology(N, M), inter_alg=inter)
        xs, x_ok = _guarded(n, torch.float32, "plain", w)
        ys, y_ok = _guarded(n * p, torch.float32, "plain", w)
        for r in range(p):
            xs[r].copy_(torch.from_numpy(ag_in[r]))
        pkg.run_ranks(p, lambda c: pkg.hier_all_gather(plan, c, xs[c.rank], out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), ("hier ag", inter)
        want = oracle.hier_all_gather(ag_in, N, M, inter)
        for r in range(p):
            assert np.array_equal(_bits(ys[r]), want[r])
        xs, x_ok = _guarded(n * p, torch.float32, "plain", w)
        ys, y_ok = _guarded(n, torch.float32, "plain", w)
        for r in range(p):
            xs[r].copy_(torch.from_numpy(rs_in[r]))
        pkg.run_ranks(p, lambda c: pkg.hier_reduce_scatter(plan, c, xs[c.rank], out=ys[c.rank]))
        torch.cuda.synchronize()
        assert x_ok() and y_ok(), ("hier rs", inter)
        want = oracle.hier_reduce_scatter(rs_in, N, M, inter)
        for r in range(p):
            assert np.array_equal(_bits(ys[r]), want[r])
