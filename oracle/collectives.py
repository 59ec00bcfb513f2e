"""Numpy restatement of the reference's collectives — TEST INFRASTRUCTURE ONLY.

Every function takes the list of per-rank inputs (rank order) and returns the
list of per-rank outputs, executing the reference algorithm's steps for all
ranks in one process. Floating-point reductions happen in exactly the order
the reference performs them, so fp32 results are bit-identical to running
collkit itself (pinned by ``tests/test_oracle.py`` against
``tests/golden/*.npz``, generated from collkit by ``tests/golden/make_golden.py``).

``dtype`` is "f32", "bf16" or "f16". bf16 arrays are ``uint16`` bit patterns
(see ``oracle/bf16.py``); f16 arrays are numpy ``float16``. For the step-wise
algorithms (ring, recursive halving, hierarchical) a low-precision partial is
rounded back to its storage type after every step ("wire" semantics, exactly
what the CUDA kernels store between steps). ``direct_reduce_scatter``
accumulates in fp32 and rounds once.
"""
from __future__ import annotations

import numpy as np

from .bf16 import bf16_to_f32, f32_to_bf16

_STORAGE = {"f32": np.float32, "bf16": np.uint16, "f16": np.float16}


def _check_dtype(dtype: str) -> None:
    if dtype not in _STORAGE:
        raise ValueError(f"unknown dtype {dtype!r}")


def _to_f32(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return bf16_to_f32(x)
    return np.asarray(x).astype(np.float32)


def _from_f32(x: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return f32_to_bf16(x)
    if dtype == "f16":
        return x.astype(np.float16)
    return x.astype(np.float32)


def _add(a: np.ndarray, b: np.ndarray, dtype: str) -> np.ndarray:
    """One reduction step, ``collkit/collectives.py:45-52`` (``np.add``):
    fp32 IEEE RNE add; low-precision operands are upcast exactly and the sum is
    rounded back to the storage type."""
    if dtype == "f32":
        return np.add(a, b, dtype=np.float32)
    return _from_f32(np.add(_to_f32(a, dtype), _to_f32(b, dtype), dtype=np.float32), dtype)


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _flat(inputs) -> list:
    return [np.ascontiguousarray(x).reshape(-1) for x in inputs]


# --------------------------------------------------------------------------
# all-gather
# --------------------------------------------------------------------------


def ring_all_gather(inputs) -> list:
    """``collkit/collectives.py:55-76``: step s, rank r forwards block (r-s)
    to r+1 and receives block (r-s-1) from r-1."""
    src = _flat(inputs)
    p = len(src)
    n = src[0].size
    outs = []
    for r in range(p):
        out = np.empty(p * n, dtype=src[0].dtype)
        out[r * n : (r + 1) * n] = src[r]
        outs.append(out)
    for s in range(p - 1):
        sent = [outs[r][((r - s) % p) * n : ((r - s) % p + 1) * n].copy() for r in range(p)]
        for r in range(p):
            blk = (r - s - 1) % p
            outs[r][blk * n : (blk + 1) * n] = sent[(r - 1) % p]
    return outs


def recdbl_all_gather(inputs) -> list:
    """``collkit/collectives.py:107-129``: step k swaps the 2^k gathered
    blocks with partner r XOR 2^k."""
    src = _flat(inputs)
    p = len(src)
    if not _is_pow2(p):
        raise ValueError(f"recursive doubling requires power-of-two ranks, got {p}")
    n = src[0].size
    outs = []
    for r in range(p):
        out = np.empty(p * n, dtype=src[0].dtype)
        out[r * n : (r + 1) * n] = src[r]
        outs.append(out)
    for k in range(p.bit_length() - 1):
        width = 1 << k
        sent = []
        for r in range(p):
            start = (r >> k) << k
            sent.append(outs[r][start * n : (start + width) * n].copy())
        for r in range(p):
            partner = r ^ width
            pstart = (partner >> k) << k
            outs[r][pstart * n : (pstart + width) * n] = sent[partner]
    return outs


def direct_all_gather(inputs) -> list:
    """One-shot all-gather (new algorithm name): same output
    contract as ``ring_all_gather``."""
    src = _flat(inputs)
    cat = np.concatenate(src) if src else np.empty(0, np.float32)
    return [cat.copy() for _ in src]


def expected_all_gather(inputs) -> np.ndarray:
    """``collkit/bench/oracles.py:7-9``."""
    return np.concatenate(_flat(inputs))


# --------------------------------------------------------------------------
# reduce-scatter
# --------------------------------------------------------------------------


def ring_reduce_scatter(inputs, dtype: str = "f32") -> list:
    """``collkit/collectives.py:79-104``. The carry for chunk (r-1) starts at
    rank r; at step s rank r computes carry = chunk(r-s-1) + received, so
    chunk c ends as ((x_{c+1} + x_{c+2}) + ...) + x_c (indices mod p)."""
    _check_dtype(dtype)
    src = _flat(inputs)
    p = len(src)
    if src[0].size % p:
        raise ValueError(f"input of {src[0].size} elements not divisible by p={p}")
    n = src[0].size // p
    if p == 1:
        return [src[0].copy()]

    def chunk(r, j):
        return src[r][j * n : (j + 1) * n]

    carry = [chunk(r, (r - 1) % p).copy() for r in range(p)]
    for s in range(1, p):
        received = [carry[(r - 1) % p] for r in range(p)]
        carry = [_add(chunk(r, (r - s - 1) % p), received[r], dtype) for r in range(p)]
    return carry


def rechalf_reduce_scatter(inputs, dtype: str = "f32") -> list:
    """``collkit/collectives.py:132-165``: step k exchanges half of the active
    region with partner r XOR (p >> (k+1)) and adds the received partials into
    the kept half (butterfly T_{k+1}(i) = T_k(i) + T_k(i ^ (p >> (k+1))))."""
    _check_dtype(dtype)
    src = _flat(inputs)
    p = len(src)
    if not _is_pow2(p):
        raise ValueError(f"recursive halving requires power-of-two ranks, got {p}")
    if src[0].size % p:
        raise ValueError(f"input of {src[0].size} elements not divisible by p={p}")
    n = src[0].size // p
    if p == 1:
        return [src[0].copy()]
    work = [s.copy() for s in src]
    lo = [0] * p
    hi = [p] * p
    while hi[0] - lo[0] > 1:
        sent = []
        plan = []
        for r in range(p):
            half = (hi[r] - lo[r]) // 2
            mid = lo[r] + half
            mine, theirs = ((lo[r], mid), (mid, hi[r])) if r < mid else ((mid, hi[r]), (lo[r], mid))
            sent.append(work[r][theirs[0] * n : theirs[1] * n].copy())
            plan.append((r ^ half, mine))
        for r in range(p):
            partner, mine = plan[r]
            a, b = mine[0] * n, mine[1] * n
            work[r][a:b] = _add(work[r][a:b], sent[partner], dtype)
            lo[r], hi[r] = mine
    return [work[r][r * n : (r + 1) * n].copy() for r in range(p)]


def _order_ring(p: int, c: int) -> list:
    return [(c + 1 + i) % p for i in range(p)]


def _fold_butterfly(vals: list, c: int, add) -> np.ndarray:
    """T_L(c) of the recursive-halving butterfly over leaves vals[i] = x_i."""
    p = len(vals)
    t = list(vals)
    h = p >> 1
    while h >= 1:
        t = [add(t[i], t[i ^ h]) for i in range(p)]
        h >>= 1
    return t[c]


def _fold(vals: list, order: list, add):
    acc = vals[order[0]]
    for i in order[1:]:
        acc = add(acc, vals[i])
    return acc


def direct_reduce_scatter(
    inputs,
    dtype: str = "f32",
    order: str = "ring",
    num_nodes: int | None = None,
    gpus_per_node: int | None = None,
    inter: str = "ring",
) -> list:
    """One-shot reduce-scatter: chunk c gathers x_q[c] from
    every rank and folds them in fp32, in the order of the named algorithm:

    * ``ring``: the left fold of ``ring_reduce_scatter``;
    * ``recursive``: the butterfly of ``rechalf_reduce_scatter``;
    * ``hierarchical``: outer {ring | butterfly over nodes} of the inner ring
      over local ranks (``hier_reduce_scatter``, ``collkit/hierarchy.py:176-195``);
    * ``rank``: rank order from zeros, ``collkit/bench/oracles.py:12-19``.

    Low-precision inputs are upcast once and the fp32 result is rounded once,
    so for fp32 the result is bit-identical to the named step-wise algorithm.
    """
    _check_dtype(dtype)
    src = _flat(inputs)
    p = len(src)
    if src[0].size % p:
        raise ValueError(f"input of {src[0].size} elements not divisible by p={p}")
    n = src[0].size // p
    f = [_to_f32(x, dtype) for x in src]

    def add(a, b):
        return np.add(a, b, dtype=np.float32)

    outs = []
    for c in range(p):
        vals = [f[q][c * n : (c + 1) * n] for q in range(p)]
        if order == "ring":
            acc = _fold(vals, _order_ring(p, c), add)
        elif order == "recursive":
            if not _is_pow2(p):
                raise ValueError("recursive order requires power-of-two p")
            acc = _fold_butterfly(vals, c, add)
        elif order == "rank":
            acc = np.zeros(n, np.float32)
            for v in vals:
                acc = add(acc, v)
        elif order == "hierarchical":
            N, M = num_nodes, gpus_per_node
            if N is None or M is None or N * M != p:
                raise ValueError("hierarchical order needs num_nodes * gpus_per_node == p")
            node, j = divmod(c, M)
            partials = []
            for nd in range(N):
                local = [vals[nd * M + l] for l in range(M)]
                partials.append(_fold(local, _order_ring(M, j), add))
            if inter == "recursive" and N > 1:
                acc = _fold_butterfly(partials, node, add)
            else:
                acc = _fold(partials, _order_ring(N, node), add)
        else:
            raise ValueError(f"unknown order {order!r}")
        outs.append(_from_f32(np.asarray(acc, np.float32), dtype))
    return outs


def expected_reduce_scatter(inputs) -> list:
    """``collkit/bench/oracles.py:12-19``: rank-order fold from zeros (equal to
    every algorithm only for integer-valued inputs)."""
    src = [np.asarray(x, np.float32).reshape(-1) for x in inputs]
    p = len(src)
    total = np.zeros_like(src[0])
    for b in src:
        total = total + b
    n = total.size // p
    return [total[r * n : (r + 1) * n].copy() for r in range(p)]


# --------------------------------------------------------------------------
# hierarchical
# --------------------------------------------------------------------------


def shuffle_local_major_to_global(buf, num_nodes: int, gpus_per_node: int, block_len: int) -> np.ndarray:
    """``collkit/hierarchy.py:103-114``: output block n*M + j = input block j*N + n."""
    arr = np.ascontiguousarray(buf).reshape(-1)
    if arr.size != num_nodes * gpus_per_node * block_len:
        raise ValueError("length mismatch")
    if block_len == 0:
        return arr.copy()
    return np.ascontiguousarray(
        arr.reshape(gpus_per_node, num_nodes, block_len).transpose(1, 0, 2)
    ).reshape(-1)


def shuffle_global_to_local_major(buf, num_nodes: int, gpus_per_node: int, block_len: int) -> np.ndarray:
    """``collkit/hierarchy.py:117-126`` (inverse of the above)."""
    arr = np.ascontiguousarray(buf).reshape(-1)
    if arr.size != num_nodes * gpus_per_node * block_len:
        raise ValueError("length mismatch")
    if block_len == 0:
        return arr.copy()
    return np.ascontiguousarray(
        arr.reshape(num_nodes, gpus_per_node, block_len).transpose(1, 0, 2)
    ).reshape(-1)


def _resolve_inter(inter: str, num_nodes: int) -> str:
    """``collkit/hierarchy.py:87-100`` with the analytic selector of
    ``collkit/costmodel.py:169-196``: N<2 or non-pow2 -> ring, N=2 ties -> ring,
    pow2 N>=4 -> recursive (size-independent with default CostParams)."""
    if inter != "auto":
        return inter
    if num_nodes < 2 or not _is_pow2(num_nodes) or num_nodes == 2:
        return "ring"
    return "recursive"


def hier_all_gather(inputs, num_nodes: int, gpus_per_node: int, inter: str = "ring") -> list:
    """``collkit/hierarchy.py:158-173``: inter all-gather on the stride-M
    groups, intra ring all-gather, then the local-major -> global shuffle."""
    src = _flat(inputs)
    N, M = num_nodes, gpus_per_node
    if len(src) != N * M:
        raise ValueError("world size mismatch")
    inter = _resolve_inter(inter, N)
    n = src[0].size
    gathered = [None] * (N * M)
    for j in range(M):
        members = [nd * M + j for nd in range(N)]
        fn = recdbl_all_gather if inter == "recursive" else ring_all_gather
        res = fn([src[g] for g in members])
        for i, g in enumerate(members):
            gathered[g] = res[i]
    local_major = [None] * (N * M)
    for nd in range(N):
        members = [nd * M + l for l in range(M)]
        res = ring_all_gather([gathered[g] for g in members])
        for i, g in enumerate(members):
            local_major[g] = res[i]
    return [shuffle_local_major_to_global(x, N, M, n) for x in local_major]


def hier_reduce_scatter(
    inputs, num_nodes: int, gpus_per_node: int, inter: str = "ring", dtype: str = "f32"
) -> list:
    """``collkit/hierarchy.py:176-195``: global -> local-major shuffle, intra
    ring reduce-scatter, then the inter reduce-scatter (ring or halving)."""
    _check_dtype(dtype)
    src = _flat(inputs)
    N, M = num_nodes, gpus_per_node
    p = N * M
    if len(src) != p:
        raise ValueError("world size mismatch")
    if src[0].size % p:
        raise ValueError("not divisible")
    inter = _resolve_inter(inter, N)
    n = src[0].size // p
    local_major = [shuffle_global_to_local_major(x, N, M, n) for x in src]
    partials = [None] * p
    for nd in range(N):
        members = [nd * M + l for l in range(M)]
        res = ring_reduce_scatter([local_major[g] for g in members], dtype)
        for i, g in enumerate(members):
            partials[g] = res[i]
    outs = [None] * p
    for j in range(M):
        members = [nd * M + j for nd in range(N)]
        fn = rechalf_reduce_scatter if inter == "recursive" else ring_reduce_scatter
        res = fn([partials[g] for g in members], dtype)
        for i, g in enumerate(members):
            outs[g] = res[i]
    return outs
