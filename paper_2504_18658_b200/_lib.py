"""ctypes binding of ``lib/libpccl_b200.so`` (the C ABI in
``include/pccl_b200.h``). There is no fallback: if the library is missing the
import of any collective fails loudly with the build command to run.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import STATUS_TO_ERROR, CollkitError

LIB_PATH = os.environ.get("PCCL_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libpccl_b200.so")
IPC_HANDLE_BYTES = 64
REG_HANDLE_BYTES = 80  # allocation IPC handle + offset + allocation size
MAX_RANKS = 16

# pccl_dtype_t / pccl_algo_t / pccl_order_t
DTYPES = {"f32": 0, "bf16": 1, "f16": 2, "u8": 3, "i32": 4, "i64": 5, "f64": 6}
ALGOS = {"direct": 0, "ring": 1, "recursive": 2}
ORDERS = {"ring": 0, "recursive": 1, "rank": 2,
          # direct only: the partial is rounded after every add, where the
          # step-wise algorithm of that name stores it (PCCL_ORDER_WIRE)
          "ring/wire": 16, "recursive/wire": 17}
ALL_GATHER, REDUCE_SCATTER = 0, 1

_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i = ctypes.c_int
_sz = ctypes.c_size_t
_SIGS = {
    "pccl_error_string": (ctypes.c_char_p, [_i]),
    "pccl_version": (_i, []),
    "pccl_world_create": (_i, [_i, _i, _i, ctypes.POINTER(_vp)]),
    "pccl_emu_world_create": (_i, [_i, _i, ctypes.POINTER(_vp)]),
    "pccl_world_destroy": (_i, [_vp]),
    "pccl_world_check": (_i, [_vp]),
    "pccl_world_error_detail": (_i, [_vp, ctypes.POINTER(_i)]),
    "pccl_world_reset_flags": (_i, [_vp]),
    "pccl_world_set_tuning": (_i, [_vp, _i, _i, _i]),
    "pccl_world_set_timeout_ms": (_i, [_vp, ctypes.c_int64]),
    "pccl_world_set_param": (_i, [_vp, ctypes.c_char_p, ctypes.c_int64]),
    "pccl_world_trace": (_i, [_vp, ctypes.POINTER(ctypes.c_uint64), _sz, ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "pccl_world_trace_at": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_uint64), _sz, ctypes.POINTER(_i),
                                 ctypes.POINTER(_i)]),
    "pccl_world_get_param": (_i, [_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64)]),
    "pccl_segment_create": (_i, [_vp, _sz, ctypes.POINTER(_i)]),
    "pccl_segment_export": (_i, [_vp, _i, _vp]),
    "pccl_segment_import": (_i, [_vp, _i, _vp]),
    "pccl_segment_ptr": (_i, [_vp, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_sz)]),
    "pccl_segment_register": (_i, [_vp, _vp, _sz, ctypes.POINTER(_i)]),
    "pccl_segment_register_export": (_i, [_vp, _i, _vp]),
    "pccl_segment_register_import": (_i, [_vp, _i, _vp]),
    "pccl_emu_segment_register": (_i, [_vp, ctypes.POINTER(_vp), _sz, ctypes.POINTER(_i)]),
    "pccl_segment_destroy": (_i, [_vp, _i]),
    "pccl_world_set_staging": (_i, [_vp, _i]),
    "pccl_staging_bytes": (_sz, [_i, _i, _i, _sz, _i]),
    "pccl_comm_create": (_i, [_vp, ctypes.POINTER(_i), _i, _i, ctypes.POINTER(_vp)]),
    "pccl_comm_destroy": (_i, [_vp]),
    "pccl_comm_size": (_i, [_vp, ctypes.POINTER(_i)]),
    "pccl_comm_rank": (_i, [_vp, ctypes.POINTER(_i)]),
    "pccl_comm_epoch": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_uint64)]),
    "pccl_send": (_i, [_vp, _i, _i, ctypes.c_int64, _vp, _sz, _i]),
    "pccl_recv": (_i, [_vp, _i, _i, ctypes.c_int64, _vp, _sz, _i, ctypes.POINTER(_sz)]),
    "pccl_all_gather": (_i, [_vp, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_reduce_scatter": (_i, [_vp, _i, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_hier_all_gather": (_i, [_vp, _i, _i, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_hier_reduce_scatter": (_i, [_vp, _i, _i, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_emu_all_gather": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _vp]),
    "pccl_emu_reduce_scatter": (_i, [_vp, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _vp]),
    "pccl_emu_hier_all_gather": (_i, [_vp, _i, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _vp]),
    "pccl_emu_hier_reduce_scatter": (_i, [_vp, _i, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _vp]),
    "pccl_hier_all_gather_comm": (_i, [_vp, _i, _i, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_hier_reduce_scatter_comm": (_i, [_vp, _i, _i, _i, _vp, _vp, _sz, _i, _vp]),
    "pccl_emu_hier_all_gather_comm": (_i, [_vp, _i, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i, _vp]),
    "pccl_emu_hier_reduce_scatter_comm": (_i, [_vp, _i, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _sz, _i,
                                               _vp]),
    "pccl_emu_debug_meta_skew": (_i, [_vp, _i, ctypes.c_uint32]),
    "pccl_probe": (_i, [_vp, _i, _i, ctypes.c_uint32, _sz, _i, _vp]),
    "pccl_shuffle": (_i, [_i, _vp, _vp, _i, _i, _sz, _i, _vp]),
    "pccl_reduce_inplace": (_i, [_vp, _vp, _sz, _i, _vp]),
    "pccl_copy2d": (_i, [_vp, _sz, _vp, _sz, _sz, _sz, _vp]),
    "pccl_ce_available": (_i, [_i]),
    "pccl_nvls_supported": (_i, [_vp]),
    "pccl_nvls_create": (_i, [_vp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "pccl_nvls_import": (_i, [_vp, _i, _sz, ctypes.POINTER(_i)]),
    "pccl_nvls_add_device": (_i, [_vp, _i]),
    "pccl_nvls_bind": (_i, [_vp, _i]),
    "pccl_nvls_ptr": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_sz)]),
    "pccl_nvls_destroy": (_i, [_vp, _i]),
    "pccl_nvls_all_gather": (_i, [_vp, _i, _vp, _sz, _sz, _i, _vp]),
    "pccl_nvls_reduce_scatter": (_i, [_vp, _i, _sz, _vp, _sz, _i, _vp]),
    "pccl_schedule": (_i, [_i, _i, _i, _i, _i, _sz, ctypes.POINTER(ctypes.c_int64), _i, ctypes.POINTER(_i)]),
}


def lib():
    """The loaded C library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with `make` (or "
                        "`python -c 'import __graft_entry__ as g; g.build()'`) — there is no CPU fallback"
                    )
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def error_string(status: int) -> str:
    return lib().pccl_error_string(status).decode()


def check(status: int, what: str = "") -> None:
    """Raise the reference exception class for a non-zero status."""
    if status == 0:
        return
    cls = STATUS_TO_ERROR.get(status, CollkitError)
    msg = error_string(status)
    raise cls(f"{what}: {msg}" if what else msg)


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def schedule(collective: int, algo: int, inter: int, n_nodes: int, m_gpus: int, m_bytes: int):
    """Kernel step structure as a list of steps of sorted (src, dst, nbytes)."""
    cap = 1 << 16
    rows = (ctypes.c_int64 * (4 * cap))()
    n = ctypes.c_int(0)
    check(lib().pccl_schedule(collective, algo, inter, n_nodes, m_gpus, m_bytes, rows, cap, ctypes.byref(n)), "schedule")
    steps: dict[int, list] = {}
    for i in range(n.value):
        s, src, dst, nb = rows[4 * i : 4 * i + 4]
        steps.setdefault(s, []).append((int(src), int(dst), int(nb)))
    return [sorted(steps[k]) for k in sorted(steps)]
