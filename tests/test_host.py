"""CPU: host-side logic that does not need a GPU — topology/groups, plans,
selectors, the emulation rendezvous, and the multi-process bootstrap exchange
(world_size 2 over gloo, 127.0.0.1)."""
import os
import threading

import pytest

from paper_2504_18658_b200 import errors
from paper_2504_18658_b200.communicator import Rendezvous
from paper_2504_18658_b200.hierarchy import BlockLayout, HierPlan, inter_comm_id, intra_comm_id
from paper_2504_18658_b200.selector import (
    CalibrationEntry,
    CalibrationTable,
    CostParams,
    FlatEntry,
    FlatTable,
    choose_inter_algorithm,
    t_rec,
    t_ring,
)
from paper_2504_18658_b200.topology import (
    RankId,
    Topology,
    build_topology,
    inter_node_group,
    intra_node_group,
    nic_of,
)


def test_topology_groups_match_reference_examples():
    # SPEC.md topology examples
    t = Topology(2, 2, 1)
    assert inter_node_group(t, 0).members == (0, 2)
    assert inter_node_group(t, 1).members == (1, 3)
    assert intra_node_group(t, 1).members == (2, 3)
    assert intra_node_group(Topology(1, 4, 1), 0).members == (0, 1, 2, 3)
    with pytest.raises(errors.IndexOutOfRange):
        inter_node_group(Topology(3, 2, 1), 2)
    with pytest.raises(errors.IndexOutOfRange):
        intra_node_group(t, 2)
    with pytest.raises(errors.InvalidTopology):
        build_topology(2, 8, 3)
    assert build_topology(2, 8, 4).world_size == 16
    t8 = Topology(2, 8, 4)
    assert [nic_of(t8, g) for g in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]
    assert RankId.of(t8, 13) == RankId(13, 1, 5)
    # node-major numbering; groups partition the world
    for N, M in [(2, 4), (4, 2), (1, 8), (8, 1)]:
        t = Topology(N, M)
        inter = sorted(g for j in range(M) for g in inter_node_group(t, j).members)
        intra = sorted(g for n in range(N) for g in intra_node_group(t, n).members)
        assert inter == intra == list(range(N * M))


def test_comm_ids_follow_reference():
    t = Topology(2, 4)
    assert [inter_comm_id(t, j) for j in range(4)] == [1, 2, 3, 4]
    assert [intra_comm_id(t, n) for n in range(2)] == [5, 6]


def test_plan_validation_and_auto_resolution():
    with pytest.raises(errors.NonPowerOfTwo):
        HierPlan(topo=Topology(3, 2), inter_alg="recursive")
    with pytest.raises(ValueError):
        HierPlan(topo=Topology(2, 2), inter_alg="tree")
    with pytest.raises(ValueError):
        HierPlan(topo=Topology(2, 2), collective="broadcast")
    assert HierPlan(topo=Topology(2, 2)).resolve_inter(1 << 20) == "ring"     # tie -> ring
    assert HierPlan(topo=Topology(64, 2)).resolve_inter(1 << 20) == "recursive"
    assert HierPlan(topo=Topology(3, 2)).resolve_inter(1 << 20) == "ring"     # non-pow2
    assert HierPlan(topo=Topology(1, 8)).resolve_inter(1 << 20) == "ring"     # single node
    table = CalibrationTable()
    table.add(CalibrationEntry(4, 1 << 20, 1.0, 2.0, "ring"))
    assert HierPlan(topo=Topology(4, 2), selector_mode="table", table=table).resolve_inter(1 << 20) == "ring"
    with pytest.raises(errors.EmptyTable):
        HierPlan(topo=Topology(4, 2), selector_mode="table", table=CalibrationTable()).resolve_inter(1)
    layout = BlockLayout(block_count=8, block_len=16, ordering="local_major")
    assert layout.total_elems == 128
    with pytest.raises(ValueError):
        BlockLayout(8, 16, "diagonal")


def test_cost_model_properties():
    P = CostParams()
    for p in (2, 4, 8, 16):
        for m in (1 << 10, 1 << 20, 1 << 28):
            assert t_ring(p, m, P) >= t_rec(p, m, P)          # equal bandwidth term, more steps
            assert t_ring(p, 2 * m, P) > t_ring(p, m, P)       # monotone in size
    with pytest.raises(errors.NonPowerOfTwo):
        t_rec(6, 100, P)
    assert choose_inter_algorithm(2, 1 << 20, P) == "ring"
    assert choose_inter_algorithm(8, 1 << 20, P) == "recursive"


def test_calibration_tables_roundtrip(tmp_path):
    t = CalibrationTable()
    t.add(CalibrationEntry(4, 1 << 20, 1e-3, 2e-3, "ring"))
    t.add(CalibrationEntry(4, 1 << 26, 3e-3, 2e-3, "recursive"))
    path = tmp_path / "cal.csv"
    t.save_csv(path)
    t2 = CalibrationTable.load_csv(path)
    assert t2.entries == t.entries
    assert t2.lookup(4, 1 << 25) == "recursive"
    ft = FlatTable()
    ft.add(FlatEntry("all_gather", 8, 1 << 26, "direct", 600.0))
    ft.add(FlatEntry("all_gather", 8, 1 << 26, "ring", 500.0))
    ft.add(FlatEntry("all_gather", 8, 1 << 20, "ring", 100.0))
    ft.add(FlatEntry("all_gather", 8, 1 << 20, "direct", 90.0))
    fp = tmp_path / "flat.csv"
    ft.save_csv(fp)
    ft2 = FlatTable.load_csv(fp)
    assert ft2.best("all_gather", 8, 1 << 27) == "direct"
    assert ft2.best("all_gather", 8, 1 << 19) == "ring"
    with pytest.raises(errors.EmptyTable):
        ft2.best("reduce_scatter", 8, 1)


def test_rendezvous_runs_once_and_distributes():
    rdv = Rendezvous(timeout=10)
    calls = []
    out = [None] * 4

    def execute(payloads):
        calls.append(list(payloads))
        return [x * 10 for x in payloads]

    def worker(r):
        for it in range(5):
            out[r] = rdv.arrive(("k", it), 4, r, r + it, execute)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert len(calls) == 5 and out == [(r + 4) * 10 for r in range(4)]


def test_rendezvous_reuses_keys_safely_and_propagates_errors():
    rdv = Rendezvous(timeout=10)
    errs = []

    def execute(payloads):
        raise errors.LengthMismatch("sizes differ")

    def worker(r):
        try:
            rdv.arrive("same", 2, r, r, execute)
        except errors.LengthMismatch:
            errs.append(r)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert sorted(errs) == [0, 1]
    with pytest.raises(errors.Timeout):
        Rendezvous(timeout=0.2).arrive("lonely", 2, 0, None, execute)


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the bootstrap exchange init_from_torch uses for IPC handles
    blob = bytes([rank]) * 64
    out = [None] * world
    dist.all_gather_object(out, blob)
    q.put((rank, [o[0] for o in out], all(len(o) == 64 for o in out)))
    dist.destroy_process_group()


def test_bootstrap_exchange_world_size_2_gloo():
    """Handles are exchanged in rank order over the process group (the only
    host-side collective the GPU path performs)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29000 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, [0, 1], True), (1, [0, 1], True)]


# ---------------------------------------------------------------------------
# sliced host-buffer path: slice geometry (collectives._pipeline_slices)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("row_len,es", [(1, 4), (1000, 4), (262144, 4), (300_007, 2), (1 << 24, 2), (5_000_011, 1),
                                        (33_554_432, 4)])
def test_pipeline_slices_cover_rows_exactly(row_len, es):
    from paper_2504_18658_b200 import collectives as C

    for in_bytes in (row_len * es, row_len * es * 8):
        sl = C._pipeline_slices(row_len, es, in_bytes)
        if in_bytes < C.PIPE_MIN_BYTES:
            assert sl is None
            continue
        if sl is None:  # a row too short to split
            assert row_len * es <= 256
            continue
        assert 2 <= len(sl) <= C.PIPE_MAX_SLICES
        assert sl[0][0] == 0 and sum(n for _, n in sl) == row_len
        for (a, n), (b, _) in zip(sl, sl[1:]):
            assert a + n == b  # contiguous, no overlap
        assert all((off * es) % 256 == 0 for off, _ in sl)  # vector-aligned slice starts
        assert all(n > 0 for _, n in sl)


def test_pipeline_slices_follow_the_size_knobs(monkeypatch):
    from paper_2504_18658_b200 import collectives as C

    monkeypatch.setattr(C, "PIPE_MIN_BYTES", 1 << 20)
    monkeypatch.setattr(C, "PIPE_SLICE_BYTES", 1 << 20)
    assert C._pipeline_slices(1 << 18, 4, (1 << 20) - 4) is None  # below the threshold
    assert len(C._pipeline_slices(1 << 18, 4, 4 << 20)) == 4
    assert len(C._pipeline_slices(1 << 24, 4, 1 << 30)) == C.PIPE_MAX_SLICES  # capped


def test_cost_params_defaults_and_formulas_match_reference():
    """CostParams() keeps collkit's defaults (costmodel.py:35-41); numbers
    below were produced by collkit.costmodel in this container."""
    import math

    from paper_2504_18658_b200 import B200_NVLINK, t_hierarchical

    P = CostParams()
    assert (P.alpha_inter, P.beta_inter, P.alpha_intra, P.beta_intra) == (10e-6, 0.04e-9, 3e-6, 0.01e-9)
    assert (P.gamma("fast"), P.gamma("slow"), P.packet_bytes) == (0.002e-9, 0.4e-9, 2048)
    assert math.isclose(t_ring(8, 1e6, P), 0.000105, rel_tol=1e-12)
    assert math.isclose(t_rec(8, 1e6, P), 6.500000000000001e-05, rel_tol=1e-12)
    assert math.isclose(t_ring(4, 2 ** 27, P, "intra"), 0.0010156329599999999, rel_tol=1e-12)
    for (N, M, alg), want in {(2, 4, "ring"): 0.0033744431999999996, (4, 2, "recursive"): 0.00539170912,
                              (4, 2, "auto"): 0.00539170912, (2, 4, "auto"): 0.0033744431999999996,
                              (3, 2, "auto"): 0.004944316693333333}.items():
        assert math.isclose(t_hierarchical(Topology(N, M, 1), 2 ** 28, alg, P), want, rel_tol=1e-12), (N, M, alg)
    with pytest.raises(ValueError):
        t_hierarchical(Topology(2, 2, 1), 1e6, "bogus", P)
    # the B200 preset changes the numbers, not the analytic decisions
    for N in (2, 3, 4, 8):
        for m in (1e3, 1e6, 1e9):
            assert choose_inter_algorithm(N, m, B200_NVLINK) == choose_inter_algorithm(N, m, P)


def test_auto_reduce_scatter_keeps_the_requested_add_order():
    """algorithm="auto" only picks among data movements that add in the
    requested order (fp32 bits never depend on message size / table)."""
    from paper_2504_18658_b200 import selector

    t = FlatTable()
    for m, (d, r, rec) in {1 << 20: (100, 50, 400), 1 << 27: (100, 300, 500)}.items():
        t.add(FlatEntry("reduce_scatter", 4, m, "direct", d))
        t.add(FlatEntry("reduce_scatter", 4, m, "ring", r))
        t.add(FlatEntry("reduce_scatter", 4, m, "recursive", rec))
    saved = selector._flat_table
    selector._flat_table = t
    selector._choice_cache.clear()
    try:
        assert selector.choose_algorithm("reduce_scatter", 4, 1 << 27) == "ring"
        assert selector.choose_algorithm("reduce_scatter", 4, 1 << 20) == "direct"
        assert selector.choose_algorithm("reduce_scatter", 4, 1 << 27, "recursive") == "recursive"
        assert selector.choose_algorithm("reduce_scatter", 4, 1 << 27, "rank") == "direct"
        assert selector.choose_algorithm("all_gather", 4, 1 << 27) == "direct"  # nothing measured: one-shot
    finally:
        selector._flat_table = saved
        selector._choice_cache.clear()


def test_torch_distributed_backend_registers():
    import torch.distributed as dist

    from paper_2504_18658_b200 import c10d

    assert c10d.BACKEND in dist.Backend.backend_list
    assert issubclass(c10d.PcclProcessGroup, dist.ProcessGroup)


def test_symmetric_heap_allocator_is_deterministic_and_coalesces():
    """The heap's first-fit allocator (no GPU: the segment is faked)."""
    from paper_2504_18658_b200.world import SymmetricHeap

    h = SymmetricHeap.__new__(SymmetricHeap)
    h.nbytes = 1 << 20
    h._free = [(0, h.nbytes)]
    h._lock = threading.Lock()
    a = h._alloc(1000)
    b = h._alloc(1)
    c = h._alloc(4096)
    assert a == (0, 1024) and b == (1024, 256) and c == (1280, 4096)
    h._release(*b)
    assert h._alloc(200) == (1024, 256)  # first fit reuses the hole
    h._release(1024, 256)
    h._release(*a)
    h._release(*c)
    assert h._free == [(0, 1 << 20)]  # everything coalesced back
    with pytest.raises(errors.OutOfMemory):
        h._alloc(2 << 20)


def test_auto_calibrates_uncovered_gpu_counts_once_per_size_bucket(monkeypatch):
    """algorithm="auto" on a real communicator whose GPU count / size bucket
    the table lacks runs tuning.autotune once (SPMD-uniform decision), then
    uses the table; emulated communicators never calibrate."""
    import torch

    from paper_2504_18658_b200 import collectives as C
    from paper_2504_18658_b200 import selector, tuning

    calls = []

    def fake_autotune(comm, collective, m, dtype=None):
        calls.append((collective, m))
        tuning._table().add(selector.FlatEntry(collective, comm.size, m, "ring", 100.0))
        return {"ring": 100.0}

    class FakeComm:
        size, emulated = 6, False

    def bucket(m_bytes, p=6):
        m = 1 << max(20, min(28, (m_bytes - 1).bit_length()))
        return m // (16 * p * 4) * (16 * p * 4)

    saved = selector._flat_table
    selector._flat_table = selector.FlatTable()
    selector._choice_cache.clear()
    monkeypatch.setattr(tuning, "autotune", fake_autotune)
    monkeypatch.setattr(torch.cuda, "is_current_stream_capturing", lambda: False)
    try:
        assert C._resolve_auto(FakeComm(), "all_gather", 100 << 20) == "ring"
        assert calls == [("all_gather", bucket(100 << 20))]
        C._resolve_auto(FakeComm(), "all_gather", 50 << 20)    # within 8x of the measured bucket
        C._resolve_auto(FakeComm(), "all_gather", 1 << 30)     # clamped to 256 MiB: within 8x
        assert len(calls) == 1
        C._resolve_auto(FakeComm(), "all_gather", 1 << 10)     # clamped to 1 MiB: 128x away
        assert calls[-1] == ("all_gather", bucket(1 << 10)) and len(calls) == 2
        C._resolve_auto(FakeComm(), "all_gather", 1 << 10)     # now measured
        assert len(calls) == 2
        FakeComm.emulated = True
        C._resolve_auto(FakeComm(), "reduce_scatter", 1 << 20)
        assert len(calls) == 2
    finally:
        selector._flat_table = saved
        selector._choice_cache.clear()
