"""CPU: the C-ABI library loads, exports every symbol include/pccl_b200.h
declares, maps status codes to the reference's exceptions, and its host-only
step tables (the structure the kernels execute) equal the reference
simulator's schedules (pkg/tests/test_acceptance.py:229-281)."""
import os
import re

import pytest

from tests.golden import fixtures

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pccl_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pccl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding knows every one of them
    assert set(names) <= set(_lib._SIGS), set(names) - set(_lib._SIGS)


def test_status_codes_map_to_reference_exceptions():
    from paper_2504_18658_b200 import _lib, errors

    expect = {2: errors.NonPowerOfTwo, 3: errors.NotDivisible, 4: errors.LengthMismatch, 5: errors.Timeout,
              6: errors.PeerUnreachable, 7: errors.Unsupported, 8: errors.InvalidTopology}
    for code, cls in expect.items():
        with pytest.raises(cls):
            _lib.check(code)
        assert _lib.error_string(code)


@pytest.mark.parametrize("cell", fixtures.schedules(), ids=lambda c: f"{c['collective']}-{c['algorithm']}-{c['N']}x{c['M']}")
def test_kernel_step_structure_matches_reference_simulator(cell):
    from paper_2504_18658_b200 import _lib

    algo = {"ring": 1, "recursive": 2, "hierarchical": 3}[cell["algorithm"]]
    inter = {"ring": 1, "recursive": 2}[cell["inter"]]
    coll = 0 if cell["collective"] == "all_gather" else 1
    got = _lib.schedule(coll, algo, inter, cell["N"], cell["M"], cell["m_bytes"])
    want = [sorted(tuple(m) for m in s) for s in cell["steps"]]
    assert got == want


@pytest.mark.parametrize("p", [2, 4, 8])
def test_byte_totals_per_rank(p):
    """Ring and recursive both move (p-1)/p * S per rank (test_collectives.py:198-220);
    direct moves the same bytes in one step."""
    from paper_2504_18658_b200 import _lib

    S = 4096 * p
    for coll in (0, 1):
        for algo in (0, 1, 2):
            steps = _lib.schedule(coll, algo, 1, 1, p, S)
            sent = {}
            for st in steps:
                for src, dst, nb in st:
                    sent[src] = sent.get(src, 0) + nb
            assert all(v == (p - 1) * S // p for v in sent.values()), (coll, algo)
            assert len(steps) == {0: 1, 1: p - 1, 2: p.bit_length() - 1}[algo]


def test_schedule_errors():
    from paper_2504_18658_b200 import _lib, errors

    with pytest.raises(errors.NonPowerOfTwo):
        _lib.schedule(0, 2, 1, 1, 6, 6 * 64)
    with pytest.raises(errors.NotDivisible):
        _lib.schedule(1, 1, 1, 1, 4, 10)


def test_staging_bytes_is_spmd_uniform_and_sufficient():
    from paper_2504_18658_b200 import _lib

    L = _lib.lib()
    for algo in (0, 1, 2, 3):
        a = L.pccl_staging_bytes(1, algo, 8, 1 << 20, 1)
        b = L.pccl_staging_bytes(1, algo, 8, 1 << 20, 1)
        assert a == b and a >= 8 * (1 << 20) * 2


def test_header_is_plain_c():
    """No torch / CUDA types in the boundary signatures."""
    raw = open(HEADER).read()
    code = re.sub(r"/\*.*?\*/", "", raw, flags=re.S)
    for bad in ("torch", "at::", "cudaStream_t", "#include <cuda"):
        assert bad not in code
    assert 'extern "C"' in code
