"""Per-step message multisets of each algorithm — TEST INFRASTRUCTURE ONLY.

Restates ``collkit/simnet.py:209-345`` (``build_schedule``): for a collective of
``m_bytes`` (AG output / RS input per rank) it yields, per synchronous step, the
sorted list of ``(src_world, dst_world, nbytes)`` messages. Used to check the
step structure the CUDA kernels declare through ``pccl_schedule`` (C-ABI),
the same check the reference runs against its instrumented transport
(``pkg/tests/conftest.py:8-44``, ``pkg/tests/test_acceptance.py:229-281``).
"""
from __future__ import annotations


def _flat(collective: str, algorithm: str, members, m_bytes: int):
    p = len(members)
    if m_bytes % p:
        raise ValueError("not divisible")
    block = m_bytes // p
    if p == 1:
        return []
    steps = []
    if algorithm == "ring":
        for _ in range(p - 1):
            steps.append([(members[r], members[(r + 1) % p], block) for r in range(p)])
    elif algorithm == "recursive":
        if p & (p - 1):
            raise ValueError("recursive needs power-of-two p")
        if collective == "all_gather":
            for k in range(p.bit_length() - 1):
                w = 1 << k
                steps.append([(members[r], members[r ^ w], w * block) for r in range(p)])
        else:
            half = p // 2
            while half >= 1:
                steps.append([(members[r], members[r ^ half], half * block) for r in range(p)])
                half //= 2
    elif algorithm == "direct":
        steps.append([(members[r], members[q], block) for r in range(p) for q in range(p) if q != r])
    else:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    return steps


def build_schedule(
    collective: str,
    algorithm: str,
    m_bytes: int,
    num_nodes: int = 1,
    gpus_per_node: int | None = None,
    inter: str = "ring",
):
    """List of steps, each a sorted list of (src, dst, nbytes)."""
    if algorithm != "hierarchical":
        p = num_nodes * gpus_per_node if gpus_per_node else num_nodes
        return [sorted(s) for s in _flat(collective, algorithm, tuple(range(p)), m_bytes)]
    N, M = num_nodes, gpus_per_node
    sub_m = m_bytes // M

    def inter_phase():
        per = [_flat(collective, inter, tuple(nd * M + j for nd in range(N)), sub_m) for j in range(M)]
        return [sorted(m for g in steps for m in g) for steps in zip(*per)]

    def intra_phase():
        per = [_flat(collective, "ring", tuple(nd * M + l for l in range(M)), m_bytes) for nd in range(N)]
        return [sorted(m for g in steps for m in g) for steps in zip(*per)]

    if collective == "all_gather":
        return inter_phase() + intra_phase()
    return intra_phase() + inter_phase()
