"""ctypes binding of libintscale_b200.so (include/intscale_b200.h).

The shared library is built in-tree by ``paper_2405_14597_b200.build``
(nvcc, sm_100a). There is no fallback: if the library is missing or cannot be
loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ISB_LIB_PATH") or os.path.join(_HERE, "libintscale_b200.so")

ISB_OK, ISB_PARAM, ISB_DIMENSION, ISB_VALUE, ISB_OVERFLOW, ISB_LENGTH, ISB_FORMAT, ISB_ERROR, \
    ISB_CUDA = range(9)
ISB_F32, ISB_BF16, ISB_F16, ISB_I32 = 0, 1, 2, 3
ISB_PATH_FLOAT_SCALE, ISB_PATH_INTEGER_SCALE, ISB_PATH_COARSE = 0, 1, 2


class IntscaleError(Exception):
    """Base of the reference's exception taxonomy (types.hpp:29-31)."""


class ParamError(IntscaleError):
    pass


class DimensionError(IntscaleError):
    pass


class ValueError_(IntscaleError):
    """ValueError (types.hpp:44); named with a trailing underscore to keep Python's builtin."""


class OverflowError_(IntscaleError):
    pass


class LengthError(IntscaleError):
    pass


class FormatError(IntscaleError):
    pass


class CudaError(IntscaleError):
    pass


_ERRORS = {
    ISB_PARAM: ParamError, ISB_DIMENSION: DimensionError, ISB_VALUE: ValueError_,
    ISB_OVERFLOW: OverflowError_, ISB_LENGTH: LengthError, ISB_FORMAT: FormatError,
    ISB_ERROR: IntscaleError, ISB_CUDA: CudaError,
}


class WeightInfo(C.Structure):
    _fields_ = [
        ("k", C.c_int64), ("n", C.c_int64), ("group", C.c_int64), ("groups", C.c_int64),
        ("amplifier", C.c_int64), ("exponent", C.c_int32), ("has_int_scales", C.c_int32),
        ("packed_bytes", C.c_int64), ("scale_bytes", C.c_int64), ("max_int_scale", C.c_int32),
        ("tensor_core_ok", C.c_int32),
    ]


class GroupProblem(C.Structure):
    _fields_ = [("w", C.c_void_p), ("m", C.c_int64), ("x", C.c_void_p), ("x_dtype", C.c_int32),
                ("xq", C.c_void_p), ("sa", C.c_void_p), ("out", C.c_void_p)]


class GroupInfo(C.Structure):
    _fields_ = [("grid", C.c_int32), ("cluster", C.c_int32), ("tile_tokens", C.c_int32),
                ("quantize", C.c_int32), ("makespan_steps", C.c_double)]


class GemmStats(C.Structure):
    _fields_ = [
        ("max_abs_accumulator", C.c_int64), ("overflow_detected", C.c_int32),
        ("hard_limit_hit", C.c_int32), ("overflow_i", C.c_int64), ("overflow_j", C.c_int64),
    ]


# Every symbol include/intscale_b200.h declares, with its ctypes signature.
_VP, _I64, _I32, _INT = C.c_void_p, C.c_int64, C.c_int32, C.c_int
SIGNATURES = {
    "isb_last_error": (C.c_char_p, []),
    "isb_version": (_INT, []),
    "isb_launch_count": (_I64, []),
    "isb_quantize_per_token": (_INT, [_VP, _INT, _I64, _I64, _VP, _VP, _INT, _VP]),
    "isb_quantize_weight_groups": (_INT, [_VP, _I64, _I64, _I64, _INT, _VP, _VP, _VP]),
    "isb_weight_pack_codes": (_INT, [_VP, _I64, _I64, _I64, _VP, _VP, _I64, _VP,
                                     C.POINTER(_VP)]),
    "isb_weight_pack_signed4": (_INT, [_VP, _I64, _I64, _I64, _I64, _VP, _VP, _I64, _VP,
                                       C.POINTER(_VP)]),
    "isb_weight_unpack_codes": (_INT, [_VP, _VP, _VP]),
    "isb_weight_repack_signed4": (_INT, [_VP, _VP, _VP]),
    "isb_weight_destroy": (_INT, [_VP]),
    "isb_weight_info": (_INT, [_VP, C.POINTER(WeightInfo)]),
    "isb_gemm_workspace_size": (_INT, [_I64, _VP, C.POINTER(_I64)]),
    "isb_gemm_act_fused_workspace_size": (_INT, [_I64, _VP, C.POINTER(_I64)]),
    "isb_gemm_integer_scale": (_INT, [_VP, _VP, _I64, _I64, _VP, _VP, _INT, _VP, _I64, _VP]),
    "isb_gemm_float_scale": (_INT, [_VP, _VP, _I64, _I64, _VP, _VP, _INT, _VP, _I64, _VP]),
    "isb_gemm_checked": (_INT, [_INT, _VP, _VP, _I64, _I64, _VP, _INT, _VP, _VP, _VP, _VP,
                                C.POINTER(GemmStats), _VP]),
    "isb_overflow_analyzer": (_INT, [_I64, _I64, _INT, _INT, _VP, _I64, C.POINTER(_I64),
                                     C.POINTER(C.c_double), C.POINTER(_I32)]),
    "isb_search_amplifier_exponent": (_INT, [_VP, _I64, C.POINTER(_I32)]),
    "isb_integerize_scales": (_INT, [_VP, _I64, _I64, _VP, C.POINTER(_I32)]),
    "isb_finalize_acc": (_INT, [_VP, _VP, _I64, _I64, _I64, _VP, _INT, _VP]),
    "isb_gemm_coarse": (_INT, [_VP, _VP, _I64, _I64, _VP, _VP, _INT, _VP, _I64, _VP]),
    "isb_gemm_act_fused": (_INT, [_INT, _VP, _INT, _I64, _I64, _VP, _VP, _INT, _VP, _VP, _I64,
                                  _VP]),
    "isb_dual_inner_quantize": (_INT, [_VP, _I64, _I64, _I64, _VP, _VP, _VP, _VP]),
    "isb_gemm_dual_quant": (_INT, [_VP, _VP, _I64, _I64, _VP, _VP, _VP, _I64, _VP, _I64, _VP, _VP,
                                    _VP]),
    "isb_gemm_dense": (_INT, [_VP, _VP, _INT, _I64, _I64, _I64, _VP, _INT, _VP]),
    "isb_group_plan_create": (_INT, [C.POINTER(GroupProblem), _I32, _I32, _I32,
                                     C.POINTER(_VP)]),
    "isb_group_run": (_INT, [_VP, _VP]),
    "isb_group_plan_info": (_INT, [_VP, C.POINTER(GroupInfo)]),
    "isb_group_nonfinite": (_INT, [_VP, _I32, C.POINTER(_I32)]),
    "isb_group_plan_destroy": (_INT, [_VP]),
    "isb_row_absmax": (_INT, [_VP, _INT, _I64, _I64, _VP, _VP]),
    "isb_quantize_per_token_amax": (_INT, [_VP, _INT, _I64, _I64, _VP, _VP, _VP, _VP]),
}

_lib = None


def load():
    """Load the in-tree library (raises if it is missing — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int):
    if rc != ISB_OK:
        msg = load().isb_last_error().decode()
        raise _ERRORS.get(rc, IntscaleError)(msg)
