"""ctypes binding of libbiluk (include/biluk.h) and status -> exception mapping.

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1703_01325_b200.build``) into ``_lib/libbiluk.so``.  There is
no fallback: if the library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import FactorizationError, SingularBlockError, StructuralError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libbiluk.so")
# A/B experiments (tools/exp.sh) load another build of the same library
LIB_PATH = os.environ.get("BILUK_LIB_PATH", LIB_PATH)

OK, ESTRUCT, ESINGULAR, EZEROPIVOT, ECUDA, ETIMEOUT, EARG, ENOMEM, EUNSUPPORTED = range(9)

_lib = None
_lock = threading.Lock()

c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_dbl = ctypes.POINTER(ctypes.c_double)

PRECOND_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class CudaPathError(RuntimeError):
    """A CUDA call inside the library failed (or the device timed out)."""


_SIGS = {
    "biluk_last_error": (ctypes.c_char_p, []),
    "biluk_version": (ctypes.c_char_p, []),
    "biluk_set_device": (ctypes.c_int, [c_i32]),
    "biluk_symbolic": (ctypes.c_int, [c_i64, c_vp, c_vp, c_i32, ctypes.POINTER(c_vp), P_i64]),
    "biluk_pattern_nnz": (c_i64, [c_vp]),
    "biluk_pattern_copy": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "biluk_pattern_free": (None, [c_vp]),
    "biluk_level_schedule": (ctypes.c_int, [c_i64, c_vp, c_vp, c_i32, c_vp, P_i64]),
    "biluk_plan_create": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_i32, ctypes.POINTER(c_vp), P_i64]),
    "biluk_plan_destroy": (None, [c_vp]),
    "biluk_plan_create_ex": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_i32, c_i32, ctypes.POINTER(c_vp), P_i64]),
    "biluk_plan_factor_lu": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, P_i64]),
    "biluk_plan_load_factored": (ctypes.c_int, [c_vp, c_vp, c_vp, P_i64]),
    "biluk_block_invert": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, P_i64, c_vp]),
    "biluk_block_diag_apply": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "biluk_scatter_blocks": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "biluk_plan_workspace_bytes": (c_u64, [c_vp]),
    "biluk_plan_bind": (ctypes.c_int, [c_vp, c_vp, c_u64, c_vp]),
    "biluk_plan_factor": (ctypes.c_int, [c_vp, c_vp, c_vp, P_i64]),
    "biluk_plan_apply": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "biluk_plan_status": (ctypes.c_int, [c_vp, c_vp]),
    "biluk_plan_tune": (ctypes.c_int, [c_vp, ctypes.c_char_p, c_i64]),
    "biluk_plan_set_trace": (ctypes.c_int, [c_vp, c_vp]),
    "biluk_plan_tile_levels": (ctypes.c_int, [c_vp, c_vp]),
    "biluk_plan_set_timing": (ctypes.c_int, [c_vp, c_i32]),
    "biluk_plan_sweep_ms": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_float)]),
    "biluk_plan_records": (ctypes.c_int, [c_vp, c_vp, c_i64]),
    "biluk_plan_info": (ctypes.c_int, [c_vp, P_i64, c_i32]),
    "biluk_plan_copy_factors": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "biluk_op_create": (ctypes.c_int, [c_i32, c_i64, c_i64, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "biluk_op_destroy": (None, [c_vp]),
    "biluk_op_workspace_bytes": (c_u64, [c_vp]),
    "biluk_op_bind": (ctypes.c_int, [c_vp, c_vp, c_u64, c_vp]),
    "biluk_op_set_values": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "biluk_op_spmv": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "biluk_krylov_workspace_bytes": (c_u64, [c_i64, c_i32]),
    "biluk_bicgstab": (ctypes.c_int, [c_vp, c_vp, PRECOND_FN, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl,
                                      P_dbl, P_dbl, c_i64, c_vp]),
    "biluk_gmres": (ctypes.c_int, [c_vp, c_vp, PRECOND_FN, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_dbl, c_dbl,
                                   P_dbl, P_dbl, c_i64, c_vp]),
    "biluk_krylov_batched_workspace_bytes": (c_u64, [c_i64, c_i32]),
    "biluk_bicgstab_batched": (ctypes.c_int, [c_vp, c_vp, PRECOND_FN, c_vp, c_i32, P_i64, c_vp, c_vp, c_vp, c_i64,
                                              c_dbl, P_dbl, c_vp]),
    "biluk_dot": (ctypes.c_int, [c_vp, c_vp, c_i64, P_dbl, c_vp, c_vp]),
}


def declared_symbols():
    """Names of every entry point the header declares (for the export test)."""
    return list(_SIGS)


def lib():
    """The loaded library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: the CUDA library was not built "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
            handle = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().biluk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, stage: str | None = None, row: int | None = None) -> None:
    """Raise the reference's exception type for a failing status code.

    Messages are stage-prefixed like the reference pipeline (factor.py:292-299).
    """
    if rc == OK:
        return
    msg = last_error() or f"status {rc}"
    if stage:
        msg = f"{stage}: {msg}"
    if rc == ESTRUCT:
        raise StructuralError(msg)
    if rc == ESINGULAR:
        raise SingularBlockError(msg, row=row)
    if rc == EZEROPIVOT:
        raise FactorizationError(msg, row=row)
    if rc == EARG:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    if rc == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaPathError(msg)


def ptr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array."""
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def current_stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def set_device(device_index: int) -> None:
    check(lib().biluk_set_device(int(device_index)))
