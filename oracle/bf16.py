"""bfloat16 helpers for the oracle (TEST INFRASTRUCTURE ONLY).

bf16 values are carried as ``uint16`` bit patterns (numpy has no bf16).
Conversion float32 -> bf16 is IEEE round-to-nearest-even, the same rounding as
CUDA's ``__float2bfloat16_rn``; NaNs are quietened. The reference itself has no
bf16 (``collkit/collectives.py:26-29`` casts everything to float32), so the
bf16 semantics here are the ones SURVEY.md §8(c) fixes: upcast to fp32, add
with one fp32 RNE rounding, round back to bf16 whenever a partial is stored in
the wire format.
"""
from __future__ import annotations

import numpy as np


def bf16_to_f32(bits) -> np.ndarray:
    """uint16 bf16 bit patterns -> float32 (exact)."""
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x) -> np.ndarray:
    """float32 -> uint16 bf16 bit patterns, round-to-nearest-even."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        out[nan] = ((f.view(np.uint32)[nan] >> 16) | 0x40).astype(np.uint16)
    return out


def bf16_add(a, b) -> np.ndarray:
    """bf16 + bf16 -> bf16 via one fp32 add (exact operands) and one RNE."""
    return f32_to_bf16(bf16_to_f32(a) + bf16_to_f32(b))
