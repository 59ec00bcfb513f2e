"""CPU oracle for the all-gather / reduce-scatter hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference's algorithms
(``/root/reference/pkg/src/collkit/collectives.py`` and ``hierarchy.py``) that
executes every rank's steps in one process and reproduces the exact
floating-point reduction order of each algorithm. It exists to *check* the
CUDA path: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it. The product
package ``paper_2504_18658_b200`` never imports it and has no CPU fallback.

Parity is pinned: ``tests/test_oracle.py`` checks this restatement bit-for-bit
against fixtures produced by running the real reference (collkit) in this
container (``tests/golden/make_golden.py``).
"""
from .bf16 import bf16_to_f32, f32_to_bf16, bf16_add
from .collectives import (
    direct_all_gather,
    direct_reduce_scatter,
    expected_all_gather,
    expected_reduce_scatter,
    hier_all_gather,
    hier_reduce_scatter,
    rechalf_reduce_scatter,
    recdbl_all_gather,
    ring_all_gather,
    ring_reduce_scatter,
    shuffle_global_to_local_major,
    shuffle_local_major_to_global,
)
from .schedule import build_schedule

__all__ = [
    "bf16_to_f32",
    "f32_to_bf16",
    "bf16_add",
    "direct_all_gather",
    "direct_reduce_scatter",
    "expected_all_gather",
    "expected_reduce_scatter",
    "hier_all_gather",
    "hier_reduce_scatter",
    "rechalf_reduce_scatter",
    "recdbl_all_gather",
    "ring_all_gather",
    "ring_reduce_scatter",
    "shuffle_global_to_local_major",
    "shuffle_local_major_to_global",
    "build_schedule",
]
