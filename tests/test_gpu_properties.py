"""GPU parity, property-based and per data-movement variant (emulation mode):
random group sizes, lengths (including non-16-byte-aligned ones), dtypes and
algorithms, each checked bit-for-bit against the oracle; explicit push / pull
variants; zero-copy symmetric buffers; the torch.distributed-shaped FSDP
wrappers; sub-communicators."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_2504_18658_b200 as pkg

    return pkg


def _np_dev(x, dtype):
    if dtype == "bf16":
        return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(x).cuda()


def _dev_np(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _inputs(rng, p, length, dtype):
    if dtype == "bf16":
        return [oracle.f32_to_bf16(rng.standard_normal(length).astype(np.float32)) for _ in range(p)]
    if dtype == "f16":
        return [rng.standard_normal(length).astype(np.float16) for _ in range(p)]
    return [rng.standard_normal(length).astype(np.float32) for _ in range(p)]


RS = {"ring": ("ring_reduce_scatter", oracle.ring_reduce_scatter),
      "recursive": ("rechalf_reduce_scatter", oracle.rechalf_reduce_scatter)}


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(p=st.sampled_from([2, 3, 4, 5, 8]), n=st.integers(0, 3000), dtype=st.sampled_from(["f32", "bf16", "f16"]),
       algo=st.sampled_from(["ring", "recursive", "direct"]), seed=st.integers(0, 10**6))
def test_reduce_scatter_property(p, n, dtype, algo, seed):
    pkg = _pkg()
    if algo == "recursive" and p & (p - 1):
        return
    rng = np.random.default_rng(seed)
    ins = _inputs(rng, p, n * p, dtype)
    if algo == "direct":
        fn = lambda c, x: pkg.direct_reduce_scatter(c, x, order="ring")  # noqa: E731
        want = oracle.direct_reduce_scatter(ins, dtype, "ring")
    else:
        fn = getattr(pkg, RS[algo][0])
        want = RS[algo][1](ins, dtype)
    outs = pkg.run_ranks(p, lambda c: _dev_np(fn(c, _np_dev(ins[c.rank], dtype)), dtype))
    for r in range(p):
        assert np.array_equal(np.ascontiguousarray(outs[r]).view(np.uint8),
                              np.ascontiguousarray(want[r]).view(np.uint8)), (p, n, dtype, algo, r)


@settings(max_examples=30, deadline=None, suppress_health_check=list(HealthCheck))
@given(p=st.sampled_from([2, 3, 4, 6, 8]), n=st.integers(0, 5000),
       dtype=st.sampled_from([torch.uint8, torch.bfloat16, torch.float32, torch.int64]),
       algo=st.sampled_from(["ring", "recursive", "direct"]), seed=st.integers(0, 10**6))
def test_all_gather_property(p, n, dtype, algo, seed):
    pkg = _pkg()
    if algo == "recursive" and p & (p - 1):
        return
    g = torch.Generator().manual_seed(seed)
    ins = [torch.randint(0, 255, (n,), generator=g).to(dtype) for _ in range(p)]
    fn = {"ring": pkg.ring_all_gather, "recursive": pkg.recdbl_all_gather, "direct": pkg.direct_all_gather}[algo]
    outs = pkg.run_ranks(p, lambda c: fn(c, ins[c.rank].cuda()).cpu())
    want = torch.cat(ins)
    for o in outs:
        assert torch.equal(o, want)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("algo", ["direct", "ring", "recursive"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_explicit_data_movement_variants(variant, algo, p):
    """Push and pull implementations of every algorithm are bit-identical."""
    pkg = _pkg()
    w = pkg.emulated_world(p)
    rng = np.random.default_rng(p * 10 + variant)
    n = 40_000 + 8
    rs_in = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
    ag_in = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
    try:
        w.set_param("ag_variant", variant)
        w.set_param("rs_variant", variant)
        rs = {"direct": lambda c, x: pkg.direct_reduce_scatter(c, x, order="ring"),
              "ring": pkg.ring_reduce_scatter, "recursive": pkg.rechalf_reduce_scatter}[algo]
        want = (oracle.rechalf_reduce_scatter if algo == "recursive" else oracle.ring_reduce_scatter)(rs_in)
        outs = pkg.run_ranks(p, lambda c: rs(c, torch.from_numpy(rs_in[c.rank]).cuda()).cpu().numpy())
        for r in range(p):
            assert np.array_equal(outs[r].view(np.uint32), want[r].view(np.uint32))
        ag = {"direct": pkg.direct_all_gather, "ring": pkg.ring_all_gather, "recursive": pkg.recdbl_all_gather}[algo]
        outs = pkg.run_ranks(p, lambda c: ag(c, torch.from_numpy(ag_in[c.rank]).cuda()).cpu().numpy())
        want = np.concatenate(ag_in)
        for o in outs:
            assert np.array_equal(o, want)
    finally:
        w.set_param("ag_variant", -1)
        w.set_param("rs_variant", -1)


def test_zero_copy_symmetric_buffers_and_fsdp_wrappers():
    """Tensors from world.empty are used in place (no staging); the
    torch.distributed-shaped wrappers fill caller-provided outputs."""
    pkg = _pkg()
    p, n = 4, 65536
    w = pkg.emulated_world(p)
    shards = w.empty(n, torch.bfloat16)
    full = w.empty(n * p, torch.bfloat16)
    grads = w.empty(n * p, torch.bfloat16)
    gsh = w.empty(n, torch.bfloat16)
    for r in range(p):
        shards[r].copy_(torch.arange(n, dtype=torch.float32).to(torch.bfloat16) + r)
        grads[r].fill_(float(r + 1))

    def body(c):
        pkg.all_gather_into_tensor(full[c.rank], shards[c.rank], c, algorithm="direct")
        pkg.reduce_scatter_tensor(gsh[c.rank], grads[c.rank], c, algorithm="recursive")
        return None

    pkg.run_ranks(p, body)
    want = torch.cat([s.cpu() for s in shards])
    for r in range(p):
        assert torch.equal(full[r].cpu(), want)
        assert torch.all(gsh[r].float() == sum(range(1, p + 1)))


def test_subgroup_collectives_and_barrier():
    pkg = _pkg()
    p = 8

    def body(c):
        c.barrier()
        sub = c.subgroup([m for m in range(p) if m % 2 == c.rank % 2], 1 + c.rank % 2)
        x = np.full(6, float(c.rank), np.float32)
        g = pkg.ring_all_gather(sub, x)
        s = pkg.rechalf_reduce_scatter(sub, np.ones(4 * 4, np.float32) * c.rank)
        c.barrier()
        return g, s

    outs = pkg.run_ranks(p, body)
    for r, (g, s) in enumerate(outs):
        members = [m for m in range(p) if m % 2 == r % 2]
        assert np.array_equal(g, np.repeat(np.array(members, np.float32), 6))
        assert np.all(s == sum(members))


@pytest.mark.parametrize("algo", ["direct", "ring", "recursive"])
def test_cuda_graph_capture_and_replay(algo):
    """Epochs live in device memory, so collectives captured into a CUDA graph
    replay correctly, and eager calls interleave with replays."""
    pkg = _pkg()
    from paper_2504_18658_b200 import _lib
    from paper_2504_18658_b200.communicator import _emu_group

    p, n = 4, 1 << 16
    w = pkg.emulated_world(p)
    group, _ = _emu_group(w, tuple(range(p)), 0)
    L = _lib.lib()
    a = _lib.ALGOS[algo]
    ins = w.empty(n * p, torch.float32)
    outs = w.empty(n, torch.float32)
    ag_out = w.empty(n * p, torch.float32)
    for r in range(p):
        ins[r].copy_(torch.arange(n * p, dtype=torch.float32) * (r + 1))
    w.ensure_staging(int(L.pccl_staging_bytes(1, a, p, n, 0)) + int(L.pccl_staging_bytes(0, a, p, n, 0)))
    sp = _lib.ptr_array([t.data_ptr() for t in ins])
    rp = _lib.ptr_array([t.data_ptr() for t in outs])
    ap = _lib.ptr_array([t.data_ptr() for t in ag_out])
    stream = torch.cuda.Stream()
    order = _lib.ORDERS["recursive" if algo == "recursive" else "ring"]

    def step(s):
        _lib.check(L.pccl_emu_reduce_scatter(group.handle, a, order, sp, rp, n, 0, s))
        _lib.check(L.pccl_emu_all_gather(group.handle, a, rp, ap, n, 0, s))

    torch.cuda.synchronize()
    step(stream.cuda_stream)  # eager warm-up (also grows nothing during capture)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step(stream.cuda_stream)
        step(stream.cuda_stream)
    with torch.cuda.stream(stream):  # replay() launches on the current stream: keep one stream
        for _ in range(25):
            g.replay()
    step(stream.cuda_stream)  # eager after replays
    torch.cuda.synchronize()
    w.check()
    total = sum(range(1, p + 1))
    want_rs = [torch.arange(n * p, dtype=torch.float32)[r * n:(r + 1) * n] * total for r in range(p)]
    for r in range(p):
        assert torch.equal(outs[r].cpu(), want_rs[r])
        assert torch.equal(ag_out[r].cpu(), torch.cat(want_rs))


@pytest.mark.parametrize("p", [4, 8])
@pytest.mark.parametrize("coll,algo", [("rs", "ring"), ("rs", "recursive"), ("rs", "direct"),
                                       ("ag", "ring"), ("ag", "recursive"), ("ag", "direct")])
def test_device_step_structure_matches_schedule(p, coll, algo):
    """The kernels' own event trace (per CTA: waits on a peer, signals to a
    peer) has exactly the step count of the algorithm's schedule
    (pccl_schedule == collkit.simnet.build_schedule, tests/test_abi.py):
    ring p-1 steps, recursive log2 p, direct 1."""
    pkg = _pkg()
    from paper_2504_18658_b200 import _lib
    from paper_2504_18658_b200.communicator import _emu_group

    w = pkg.emulated_world(p)
    group, _ = _emu_group(w, tuple(range(p)), 0)
    L = _lib.lib()
    n = 1 << 14
    a = _lib.ALGOS[algo]
    ins = w.empty(n * p if coll == "rs" else n, torch.float32)
    outs = w.empty(n if coll == "rs" else n * p, torch.float32)
    w.ensure_staging(int(L.pccl_staging_bytes(1 if coll == "rs" else 0, a, p, n, 0)))
    sp = _lib.ptr_array([t.data_ptr() for t in ins])
    rp = _lib.ptr_array([t.data_ptr() for t in outs])
    steps = len(_lib.schedule(1 if coll == "rs" else 0, a, 1, 1, p, n * p * 4))
    ll_max = w.get_param("ll_max")
    try:
        w.set_param("trace", 1)
        w.set_param("nsub", 1)
        w.set_param("ll_max", 0)  # the bulk (flag) protocol: LL / LL128 have no per-step waits
        w.set_param("ll128_max", 0)
        s = torch.cuda.current_stream().cuda_stream
        if coll == "rs":
            _lib.check(L.pccl_emu_reduce_scatter(group.handle, a, 0, sp, rp, n, 0, s))
        else:
            _lib.check(L.pccl_emu_all_gather(group.handle, a, sp, rp, n, 0, s))
        torch.cuda.synchronize()
        tr = w.trace()
    finally:
        w.set_param("trace", 0)
        w.set_param("ll_max", ll_max)
        w.set_param("ll128_max", 1 << 30)  # back to "whatever a region holds"
    assert len(tr) == p
    # default data movement for symmetric buffers: AG push, RS pull. Waits
    # per CTA = the algorithm's steps plus the push handshakes ("your buffer
    # is free" before the first store, and the final arrival of the last
    # forwarded block for AG; direct AG waits for each peer's "free"
    # separately, just before its stores into that peer).
    L = steps
    expect = {("rs", "ring"): L, ("rs", "recursive"): L, ("rs", "direct"): L,
              ("ag", "ring"): L + 1, ("ag", "recursive"): 2 * L, ("ag", "direct"): p}[(coll, algo)]
    for row in tr:
        for ev in row:
            kinds = [k for _, k, _ in ev if k not in (5, 6, 7, 8)]  # (exit, resident, epilogue, PDL release: timing only)
            assert kinds[0] == 1 and kinds.count(2) == expect, (coll, algo, p, kinds)


# ---------------------------------------------------------------------------
# maximum sizes: byte offsets and element indices beyond 2^32 / 2^31
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("algo", ["direct", "ring", "recursive"])
def test_offsets_beyond_4gib(algo):
    """AG of 4 GiB + 4112 B per rank (output offsets past 2^33) and RS of
    2^31 + 2^16 + 8 bf16 elements per rank (element indices past 2^31)."""
    pkg = _pkg()
    p = 2
    torch.cuda.empty_cache()
    n = (1 << 32) + 4112
    g = torch.Generator(device="cuda").manual_seed(11)
    ins = [torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g) for _ in range(p)]
    ag = {"direct": pkg.direct_all_gather, "ring": pkg.ring_all_gather, "recursive": pkg.recdbl_all_gather}[algo]
    outs = [torch.empty(n * p, dtype=torch.uint8, device="cuda") for _ in range(p)]
    pkg.run_ranks(p, lambda c: ag(c, ins[c.rank], out=outs[c.rank]))
    for r in range(p):
        for q in range(p):
            assert torch.equal(outs[r][q * n:(q + 1) * n], ins[q]), (algo, r, q)
    del ins, outs
    torch.cuda.empty_cache()

    m = (1 << 31) + (1 << 16) + 8  # RS input elements per rank (bf16)
    ins = []
    for r in range(p):
        x = torch.empty(m, dtype=torch.bfloat16, device="cuda")
        for s in range(0, m, 1 << 28):  # small integers: exact in bf16 under any fold order
            e = min(m, s + (1 << 28))
            x[s:e] = ((torch.arange(s, e, device="cuda") % 61 - 30) * (r + 1)).to(torch.bfloat16)
        ins.append(x)
    rs = {"direct": pkg.direct_reduce_scatter, "ring": pkg.ring_reduce_scatter,
          "recursive": pkg.rechalf_reduce_scatter}[algo]
    outs = [torch.empty(m // p, dtype=torch.bfloat16, device="cuda") for _ in range(p)]
    pkg.run_ranks(p, lambda c: rs(c, ins[c.rank], out=outs[c.rank]))
    k = m // p
    for r in range(p):
        for s in range(0, k, 1 << 28):
            e = min(k, s + (1 << 28))
            want = ((torch.arange(r * k + s, r * k + e, device="cuda") % 61 - 30) * 3).to(torch.bfloat16)
            assert torch.equal(outs[r][s:e], want), (algo, r, s)
    del ins, outs
    torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# LL protocol (small direct collectives): same results as the bulk path and
# the oracle; channel parity across groups; misaligned buffers
# ---------------------------------------------------------------------------
def _with_ll(world, value, fn):
    old = world.get_param("ll_max")
    world.set_param("ll_max", value)
    try:
        return fn()
    finally:
        world.set_param("ll_max", old)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 16])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_ll_direct_matches_bulk_and_oracle(p, dtype):
    pkg = _pkg()
    world = pkg.emulated_world(p)
    rng = np.random.default_rng(p * 7 + len(dtype))
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    per8 = {"f32": 2, "bf16": 4, "f16": 4}[dtype]
    for n in (per8, per8 * 3, per8 * 1000, (64 << 10) // (8 // per8)):
        xs = [torch.from_numpy(rng.standard_normal(n * p).astype(np.float32)).to(tdt).cuda() for _ in range(p)]
        orders = ["ring", "rank"] + (["recursive"] if p & (p - 1) == 0 else [])
        for order in orders:
            run = lambda: pkg.run_ranks(p, lambda c: pkg.direct_reduce_scatter(c, xs[c.rank], order=order).cpu())  # noqa: E731
            ll = _with_ll(world, 1 << 20, run)
            bulk = _with_ll(world, 0, run)
            if dtype != "f16":
                want = oracle.direct_reduce_scatter([_dev_np(x.cpu(), dtype) for x in xs], dtype if dtype == "bf16" else "f32",
                                                    order)
            for r in range(p):
                assert torch.equal(ll[r].view(torch.int16 if tdt != torch.float32 else torch.int32),
                                   bulk[r].view(torch.int16 if tdt != torch.float32 else torch.int32)), (order, r, n)
                if dtype != "f16":
                    assert np.array_equal(_dev_np(ll[r], dtype).view(np.uint8), np.asarray(want[r]).view(np.uint8))
        ag = lambda: pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, xs[c.rank][:n]).cpu())  # noqa: E731
        ll = _with_ll(world, 1 << 20, ag)
        want = torch.cat([x[:n].cpu() for x in xs])
        for r in range(p):
            assert torch.equal(ll[r], want)


def test_ll_channels_alternate_across_groups_and_protocols():
    """Back-to-back LL calls on the world and on overlapping sub-groups,
    interleaved with bulk calls: each channel's two regions alternate by its
    own message count, so every result stays exact."""
    pkg = _pkg()
    p, n = 4, 512

    def body(c):
        lo = c.subgroup([0, 1], 1) if c.rank < 2 else c.subgroup([2, 3], 2)
        odd = c.subgroup([1, 2, 3], 3) if c.rank > 0 else None
        bad = []
        for it in range(40):
            x = torch.full((n * p,), float(it * 10 + c.rank + 1), device="cuda")
            y = pkg.direct_reduce_scatter(c, x)
            if float(y[0]) != sum(it * 10 + q + 1 for q in range(p)):
                bad.append(("world_rs", it))
            z = pkg.direct_all_gather(lo, x[:n])
            if [float(z[0]), float(z[-1])] != [float(it * 10 + lo.members[0] + 1), float(it * 10 + lo.members[1] + 1)]:
                bad.append(("pair_ag", it))
            if odd is not None and it % 3 == 0:
                w = pkg.direct_all_gather(odd, x[:n])
                if float(w[-1]) != float(it * 10 + 4):
                    bad.append(("odd_ag", it))
            if it % 5 == 0:  # bulk protocol in between (4 MiB)
                big = torch.full(((1 << 20) * p,), 1.0, device="cuda")
                if float(pkg.reduce_scatter(c, big, algorithm="direct")[0]) != p:
                    bad.append(("bulk", it))
        torch.cuda.synchronize()
        return bad

    outs = pkg.run_ranks(p, body)
    assert outs == [[]] * p


def test_ll_misaligned_buffers_are_bounced():
    pkg = _pkg()
    p, n = 4, 1000
    base = [torch.arange(n * p + 1, dtype=torch.float32, device="cuda") * (r + 1) for r in range(p)]
    xs = [b[1:] for b in base]  # 4-byte offset: not 8-byte aligned
    assert xs[0].data_ptr() % 8 == 4
    outs_raw = [torch.zeros(n + 1, device="cuda") for _ in range(p)]
    outs = [o[1:] for o in outs_raw]
    pkg.run_ranks(p, lambda c: pkg.direct_reduce_scatter(c, xs[c.rank], out=outs[c.rank]))
    total = sum(range(1, p + 1))
    for r in range(p):
        want = (torch.arange(n * p + 1, dtype=torch.float32)[1:] * total)[r * n:(r + 1) * n]
        assert torch.equal(outs[r].cpu(), want)
    ag_raw = [torch.zeros(n * p + 1, device="cuda") for _ in range(p)]
    ags = [a[1:] for a in ag_raw]
    pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, xs[c.rank][:n], out=ags[c.rank]))
    want = torch.cat([x[:n].cpu() for x in xs])
    for r in range(p):
        assert torch.equal(ags[r].cpu(), want)


def test_param_validation():
    """Tuning knobs: documented ranges accepted, the rest rejected (include/pccl_b200.h)."""
    pkg = _pkg()
    w = pkg.emulated_world(2)
    cases = [("ll_max", [-1, 0, 8, 1 << 20], [-2]), ("ag_variant", [-1, 0, 1, 2, 3, 4, 5, 8], [-2, 6, 7, 9]),
             ("rs_variant", [-1, 0, 1, 4, 5, 7, 8], [6, 9]), ("ll128_max", [0, 8, 1 << 20], [-1]), ("items_per_cta", [1, 16], [0, 17]), ("hier_intra", [-1, 0, 1], [-2, 2]), ("ctas", [0, 1, 320], [-1, 321]), ("nsub", [1, 32], [0, 33]),
             ("threads", [64, 512], [32, 100, 1024]), ("timeout_ms", [1, 20000], [0]), ("pdl", [0, 1], [-1]),
             ("local_fence", [0, 1], [-1]), ("item_kib", [0, 16, 64], [-1])]
    for key, good, bad in cases:
        old = w.get_param(key)
        try:
            for v in good:
                w.set_param(key, v)
                assert w.get_param(key) == v
            for v in bad:
                with pytest.raises(ValueError):
                    w.set_param(key, v)
        finally:
            w.set_param(key, old)
    with pytest.raises(ValueError):
        w.set_param("no_such_knob", 1)


def test_nvls_needs_real_mode():
    """NVLS segments are a real-mode (one process per GPU) feature: an
    emulated world reports no support and refuses to create one."""
    pkg = _pkg()
    from paper_2504_18658_b200 import nvls
    from paper_2504_18658_b200.errors import Unsupported

    w = pkg.emulated_world(2)
    assert not nvls.nvls_supported(w)
    with pytest.raises(Unsupported):
        nvls.create_nvls_segment(w, 1 << 20)


@pytest.mark.parametrize("algo", ["direct", "ring", "recursive"])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_push_all_gather_mixed_in_place_rows(algo, dtype):
    """Push all-gathers store the own block into the output from the first
    push's loads (no tail local copy). In one emulated launch some rows run
    in place (send = own block of the output) and others do not: the copy is
    one value per launch (OR over the rows), a self-copy is harmless, and
    every output is exact."""
    pkg = _pkg()
    p, n = 4, 40000 + 8
    w = pkg.emulated_world(p)
    full = w.empty(n * p, dtype)
    sends = w.empty(n, dtype)
    g = torch.Generator(device="cuda").manual_seed(5)
    blocks = [torch.randn(n, generator=g, device="cuda").to(dtype) for _ in range(p)]
    for r in range(p):
        full[r].fill_(float("nan"))
        if r % 2 == 0:
            full[r][r * n:(r + 1) * n].copy_(blocks[r])  # in place
        else:
            sends[r].copy_(blocks[r])

    def body(c):
        src = full[c.rank][c.rank * n:(c.rank + 1) * n] if c.rank % 2 == 0 else sends[c.rank]
        pkg.all_gather_into_tensor(full[c.rank], src, c, algorithm=algo)
        return None

    pkg.run_ranks(p, body)
    want = torch.cat(blocks)
    for r in range(p):
        assert torch.equal(full[r].view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                           want.view(torch.int16 if dtype == torch.bfloat16 else torch.int32)), (algo, r)


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.uint8])
def test_ll128_all_gather_matches_oracle(p, dtype):
    """LL128 line protocol (ag_variant 8): 120 payload bytes + an 8-byte tag
    per 128-byte line, no handshakes. Every size class: a single word, a
    partial last line, exact line multiples, ragged warp groups, and the
    largest message one region holds; alternated with LL and flag-protocol
    calls on the same group (separate regions and channel counters), in
    place and not, bit-exact against the reference's all-gather."""
    pkg = _pkg()
    w = pkg.emulated_world(p)
    es = torch.empty(0, dtype=dtype).element_size()
    cap_words = (1 << 14) * 15  # PCCL_LL128_LINES * 15 eight-byte words
    g = torch.Generator(device="cuda").manual_seed(17 + p)
    try:
        for words in (1, 14, 15, 16, 60, 61, 1000, 4099, 40000, cap_words):
            n = words * 8 // es
            blocks = [torch.randint(0, 255, (n * es,), dtype=torch.uint8, generator=g, device="cuda").view(dtype)
                      for _ in range(p)]
            want = torch.cat(blocks)
            for variant in (8, 4, -1, 8):
                if variant == 4 and words * 8 > (1 << 20):
                    continue
                w.set_param("ag_variant", variant)
                outs = [torch.full((n * p,), 0, dtype=dtype, device="cuda") for _ in range(p)]
                pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, blocks[c.rank], out=outs[c.rank]))
                for r in range(p):
                    assert torch.equal(outs[r].view(torch.uint8), want.view(torch.uint8)), (p, dtype, words, variant, r)
        # in place: my block already sits in the output
        w.set_param("ag_variant", 8)
        n = 4099 * 8 // es
        blocks = [torch.randint(0, 255, (n * es,), dtype=torch.uint8, generator=g, device="cuda").view(dtype)
                  for _ in range(p)]
        outs = [torch.zeros(n * p, dtype=dtype, device="cuda") for _ in range(p)]
        for r in range(p):
            outs[r][r * n:(r + 1) * n].copy_(blocks[r])
        pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, outs[c.rank][c.rank * n:(c.rank + 1) * n],
                                                          out=outs[c.rank]))
        for r in range(p):
            assert torch.equal(outs[r].view(torch.uint8), torch.cat(blocks).view(torch.uint8))
    finally:
        w.set_param("ag_variant", -1)


def test_ll128_too_large_is_rejected_not_truncated():
    """A message larger than one LL128 region is not sent as LL128: with the
    variant forced the call falls back to the flag protocol (the LL rule),
    and the result is exact."""
    pkg = _pkg()
    p = 2
    w = pkg.emulated_world(p)
    words = (1 << 14) * 15 + 8
    blocks = [torch.arange(words * 2, dtype=torch.float32, device="cuda") + 1000 * r for r in range(p)]
    outs = [torch.empty(words * 2 * p, device="cuda") for _ in range(p)]
    try:
        w.set_param("ag_variant", 8)
        pkg.run_ranks(p, lambda c: pkg.direct_all_gather(c, blocks[c.rank], out=outs[c.rank]))
    finally:
        w.set_param("ag_variant", -1)
    for r in range(p):
        assert torch.equal(outs[r], torch.cat(blocks))


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_ll128_reduce_scatter_matches_oracle(p, dtype):
    """LL128 reduce-scatter (rs_variant 8): chunk q travels to member q as
    128-byte lines; the owner folds its own chunk and the p - 1 line streams
    in the named order (ring / butterfly / rank, with the wire rounding
    points when asked) — bit-identical to the direct kernel in that order and
    to the reference where the order is the reference's. Sizes from one word
    to a full region, alternated with LL and flag-protocol calls."""
    pkg = _pkg()
    w = pkg.emulated_world(p)
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    es = torch.empty(0, dtype=tdt).element_size()
    rng = np.random.default_rng(23 + p)
    orders = ["ring", "rank"] + (["recursive"] if p & (p - 1) == 0 else [])
    try:
        for words in (1, 15, 61, 4099, (1 << 14) * 15):
            n = words * 8 // es
            ins32 = [rng.standard_normal(n * p).astype(np.float32) for _ in range(p)]
            xs = [torch.from_numpy(x).to(tdt).cuda() for x in ins32]
            for order in orders:
                ref = None
                for variant in (8, -1, 4, 8):
                    if variant == 4 and words * 8 > (1 << 20):
                        continue
                    w.set_param("rs_variant", variant)
                    outs = pkg.run_ranks(p, lambda c: pkg.direct_reduce_scatter(c, xs[c.rank], order=order).cpu())
                    bits = [o.view(torch.int16 if es == 2 else torch.int32) for o in outs]
                    if ref is None:
                        ref = bits
                    for r in range(p):
                        assert torch.equal(bits[r], ref[r]), (p, dtype, words, order, variant, r)
                if dtype == "f32" and order != "rank":
                    want = (oracle.rechalf_reduce_scatter if order == "recursive" else oracle.direct_reduce_scatter)(
                        ins32, "f32", **({} if order == "recursive" else {"order": "ring"}))
                    for r in range(p):
                        assert np.array_equal(ref[r].numpy().view(np.uint32), np.asarray(want[r]).view(np.uint32))
    finally:
        w.set_param("rs_variant", -1)
