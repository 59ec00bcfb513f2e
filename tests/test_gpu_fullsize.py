"""GPU parity at the BASELINE configs' FULL sizes (VERDICT r1 "next" item 2):
p = 8 ranks emulated on cuda:0 in one cooperative launch per collective,
through the C ABI (pccl_emu_*), exactly the kernels the 8-GPU path runs.

Every output is compared bit for bit over its whole length with the device
restatement of the algorithm's reduction order (``bench.expected_rs``, pinned
against the oracle by tests/test_bench.py), and a sampled sub-problem (a
column slice of every chunk: the collectives are elementwise, so slicing
every chunk the same way is again a valid input) is checked against the
numpy oracle itself.

* C1  all-gather fp32, 64 MiB output, ring                     (collectives.py:55-76)
* C2  reduce-scatter bf16, 128 MiB input, recursive halving     (collectives.py:132-165)
* C3  hierarchical AG + RS fp32, 256 MiB, 2x4 ring / 4x2 rec.   (hierarchy.py:158-195)
* C5  GPT-3-style 7B per-layer bf16 (402,759,680 B), direct AG + RS
"""
import numpy as np
import pytest
import torch

import bench
import oracle

pytestmark = pytest.mark.gpu

MiB = 1 << 20
P8 = 8


@pytest.fixture(scope="module")
def rig():
    r = bench.Rig(False, P8, 0, torch.device("cuda", 0))
    yield r
    r.world.check()


def _np_bits(t: torch.Tensor) -> np.ndarray:
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def _dn(dtype):
    return "bf16" if dtype == torch.bfloat16 else "f32"


def _sub_inputs(ins, n, lo, hi, p):
    """Every rank's input restricted to columns [lo, hi) of each of its p chunks."""
    return [_np_bits(torch.cat([x[c * n + lo: c * n + hi] for c in range(p)])) for x in ins]


def _run(rig, call):
    call()
    torch.cuda.synchronize()
    rig.world.check()


def test_c1_all_gather_f32_64MiB_ring(rig):
    p, S = P8, 64 * MiB
    n = S // 4 // p
    bi, bo = rig.sym(n, torch.float32), rig.sym(n * p, torch.float32)
    seed = rig.new_seed()
    rig.fill(bi, seed)
    for t in bo:
        t.fill_(float("nan"))
    _run(rig, rig.ag("ring", bi, bo, n, 0))
    assert rig.verify_ag(bi, bo, seed, n, torch.float32)
    lo, hi = n // 3, n // 3 + 65536
    want = oracle.ring_all_gather([_np_bits(x[lo:hi]) for x in bi])
    for r in range(p):
        got = np.concatenate([_np_bits(bo[r][q * n + lo: q * n + hi]) for q in range(p)])
        assert np.array_equal(got.view(np.uint8), want[r].view(np.uint8)), r


@pytest.mark.parametrize("algo", ["recursive", "direct"])
def test_c2_reduce_scatter_bf16_128MiB(rig, algo):
    p, S = P8, 128 * MiB
    n = S // 2 // p
    order = "recursive" if algo == "recursive" else "ring"
    bi, bo = rig.sym(n * p, torch.bfloat16), rig.sym(n, torch.bfloat16)
    seed = rig.new_seed()
    rig.fill(bi, seed)
    _run(rig, rig.rs(algo, order, bi, bo, n, 1))
    # whole output, bit-exact vs the per-step-rounding restatement
    assert rig.verify_rs(bi, bo, seed, n, torch.bfloat16, algo, order)
    # sampled sub-problem vs the numpy oracle
    lo, hi = 1234567, 1234567 + 49152
    sub = _sub_inputs(bi, n, lo, hi, p)
    want = (oracle.rechalf_reduce_scatter(sub, "bf16") if algo == "recursive"
            else oracle.direct_reduce_scatter(sub, "bf16", order="ring"))
    for r in range(p):
        assert np.array_equal(_np_bits(bo[r][lo:hi]), want[r]), r
    # the stated bf16 bound vs the exact sum: |y - sum| <= p * 2^-8 * sum|x|
    for r in range(p):
        leaves = torch.stack([bi[q][r * n: (r + 1) * n].double() for q in range(p)])
        exact, mag = leaves.sum(0), leaves.abs().sum(0)
        assert bool(((bo[r].double() - exact).abs() <= p * 2.0 ** -8 * mag + 1e-30).all()), r


@pytest.mark.parametrize("grid,inter", [((2, 4), "ring"), ((4, 2), "recursive")])
def test_c3_hierarchical_256MiB(rig, grid, inter):
    p, S = P8, 256 * MiB
    N, M = grid
    n = S // 4 // p
    ai, ao = rig.sym(n, torch.float32), rig.sym(n * p, torch.float32)
    sa = rig.new_seed()
    rig.fill(ai, sa)
    _run(rig, rig.hier("ag", N, M, inter, ai, ao, n, 0))
    assert rig.verify_ag(ai, ao, sa, n, torch.float32)
    del ai, ao
    ri, ro = rig.sym(n * p, torch.float32), rig.sym(n, torch.float32)
    sr = rig.new_seed()
    rig.fill(ri, sr)
    _run(rig, rig.hier("rs", N, M, inter, ri, ro, n, 0))
    assert rig.verify_rs(ri, ro, sr, n, torch.float32, "hierarchical", grid=grid, inter=inter)
    lo, hi = n - 40000, n
    want = oracle.hier_reduce_scatter(_sub_inputs(ri, n, lo, hi, p), N, M, inter, "f32")
    for r in range(p):
        assert np.array_equal(_np_bits(ro[r][lo:hi]).view(np.uint8), want[r].view(np.uint8)), r


def test_c5_fsdp_7b_layer_direct_bf16(rig):
    p = P8
    n7 = bench.P7 // p
    prm, full = rig.sym(n7, torch.bfloat16), rig.sym(n7 * p, torch.bfloat16)
    s_p = rig.new_seed()
    rig.fill(prm, s_p)
    _run(rig, rig.ag("direct", prm, full, n7, 1))
    assert rig.verify_ag(prm, full, s_p, n7, torch.bfloat16)
    del prm, full
    grad, gsh = rig.sym(n7 * p, torch.bfloat16), rig.sym(n7, torch.bfloat16)
    s_g = rig.new_seed()
    rig.fill(grad, s_g)
    _run(rig, rig.rs("direct", "ring", grad, gsh, n7, 1))
    assert rig.verify_rs(grad, gsh, s_g, n7, torch.bfloat16, "direct", "ring")
    lo, hi = 777, 777 + 32768
    want = oracle.direct_reduce_scatter(_sub_inputs(grad, n7, lo, hi, p), "bf16", order="ring")
    for r in range(p):
        assert np.array_equal(_np_bits(gsh[r][lo:hi]), want[r]), r
