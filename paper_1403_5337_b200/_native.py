"""ctypes binding of libhodlr_b200.so (the C ABI declared in include/hodlr_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import errors

_LIB = None
_LOCK = threading.Lock()
LIB_PATH = Path(os.environ.get("HK_LIB_PATH") or Path(__file__).resolve().with_name("libhodlr_b200.so"))

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double
PI64 = C.POINTER(C.c_int64)
PI32 = C.POINTER(C.c_int32)
PD = C.POINTER(C.c_double)

# name -> (restype, argtypes); every symbol of include/hodlr_b200.h
SIGNATURES = {
    "hk_last_error": (C.c_char_p, []),
    "hk_version": (C.c_char_p, []),
    "hk_device_count": (C.c_int, []),
    "hk_plan_create": (C.c_int, [I64, I64, I64, C.POINTER(P)]),
    "hk_plan_destroy": (C.c_int, [P]),
    "hk_plan_num_nodes": (I64, [P]),
    "hk_plan_tree": (C.c_int, [P, PI32, PI64, PI64, PI32, PI32]),
    "hk_build_aca": (C.c_int, [P, P, I64, I64, D, D, I64, C.c_int, P]),
    "hk_build_bdlr": (C.c_int, [P, P, I64, I64, D, I32, I64, PI64, PI64, P]),
    "hk_build_external_begin": (C.c_int, [P, P, I64, I64, P]),
    "hk_set_block_factor": (C.c_int, [P, I64, I64, I64, P, I64, P, I64, P]),
    "hk_get_ranks": (C.c_int, [P, PI32]),
    "hk_get_aca_trace": (C.c_int, [P, I64, I64, PI32, PI64, PI32, PI64]),
    "hk_get_skeleton": (C.c_int, [P, I64, I64, PI64, PI64, PI64, I64]),
    "hk_get_block_factor": (C.c_int, [P, I64, I64, PD, PD]),
    "hk_block_shape": (C.c_int, [P, I64, PI64, PI64, PI64]),
    "hk_factor": (C.c_int, [P, P]),
    "hk_factor_ext": (C.c_int, [P, P, I64, I64, P]),
    "hk_get_extension": (C.c_int, [P, I64, C.POINTER(P), C.POINTER(I64), C.POINTER(I64)]),
    "hk_copy_extension": (C.c_int, [P, I64, I64, I64, P, I64, P]),
    "hk_copy_h2d_streaming": (C.c_int, [P, P, I64, C.c_int, P]),
    "hk_gmres_batch": (C.c_int, [P, I64, P, I64, I64, P, I64, D, I64, C.c_int, P, P, PI64, PD, PD, PI32, P]),
    "hk_dgemm": (C.c_int, [C.c_int, I64, I64, I64, D, P, I64, P, I64, D, P, I64, P]),
    "hk_gj_inverse": (C.c_int, [P, I64, I64, I64, I64, P, P, P]),
    "hk_get_leaf_lu": (C.c_int, [P, I64, I64, PD, PI32, PD]),
    "hk_get_coupling": (C.c_int, [P, I64, I64, PD, PD, PD, PI32, PD]),
    "hk_solve": (C.c_int, [P, P, I64, I64, I64, P]),
    "hk_solve_front": (C.c_int, [P, I64, P, I64, I64, P]),
    "hk_gmres": (C.c_int, [P, I64, P, I64, I64, P, D, I64, C.c_int, P, P, PI64, PD, PD, PI32, P]),
    "hk_arnoldi_step": (C.c_int, [I64, I64, I64, P, P, P, P, P, P, D, PD, P]),
    "hk_gmres_combine": (C.c_int, [I64, I64, I64, P, P, P, P, P]),
    "hk_arnoldi_step_batch": (C.c_int, [I64, I64, I64, P, I64, P, I64, P, P, P, P, P, P, P, I64, P]),
    "hk_gemv": (C.c_int, [P, I64, I64, I64, P, I64, I64, P, I64, P]),
    "hk_lu_full": (C.c_int, [P, I64, I64, I64, P, P, P, PI64, P]),
    "hk_lu_partial": (C.c_int, [P, I64, I64, P, P, P]),
    "hk_aca_block": (C.c_int, [P, I64, I64, I64, D, I64, P, P, PI64, PI32, PI64, PI32, PI64, P]),
    "hk_skeleton_block": (C.c_int, [P, I64, I64, I64, PI64, I64, PI64, I64, D, I64, P, P, PI64,
                                    PI64, PI64, P]),
    "hk_graph_distance": (C.c_int, [I64, PI64, PI64, PI64, I64, PI64, I64, PI64]),
    "hk_select_by_depth": (C.c_int, [I64, PI64, PI64, PI64, I64, PI64, I64, I32, PI64, PI64,
                                     PI64, PI64]),
    "hk_get_timings": (C.c_int, [P, PD, PD, PD]),
    "hk_get_aca_time": (C.c_int, [P, PD]),
    "hk_launch_count": (I64, []),
    "hk_debug_violations": (I64, [C.POINTER(I64)]),
    "hk_spd_inverse": (C.c_int, [P, I64, I64, I64, I64, PI32, P]),
}

HK_OK = 0
_STATUS = {
    1: ValueError,
    2: errors.DimensionMismatchError,
    3: errors.SingularMatrixError,
    4: errors.SingularLeafError,
    5: errors.SingularSchurError,
    6: errors.DegenerateSkeletonError,
    7: errors.GmresBreakdownError,
    8: errors.EmptySelectionError,
    20: RuntimeError,
    21: RuntimeError,
}


def lib():
    """Load the library once; raise ImportError if it was never built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH.name} is not built; run "
                    "`python -m paper_1403_5337_b200.build_native` (no CPU fallback exists)")
            L = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = L
    return _LIB


def last_error() -> str:
    msg = lib().hk_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status == HK_OK:
        return
    exc = _STATUS.get(status, RuntimeError)
    raise exc(last_error() or f"hodlr_b200 status {status}")


def device_count() -> int:
    return int(lib().hk_device_count())


def require_cuda():
    """The compute path runs only on a CUDA device: fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available() or device_count() == 0:
        raise RuntimeError("paper_1403_5337_b200 needs a CUDA device (sm_100a B200); "
                           "there is no CPU fallback")
    return torch


def stream_handle():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    """Device pointer of a torch tensor."""
    return C.c_void_p(t.data_ptr())


def arr_ptr(a, ctype):
    """Host pointer of a contiguous numpy array."""
    return a.ctypes.data_as(C.POINTER(ctype))


def launch_count() -> int:
    return int(lib().hk_launch_count())
