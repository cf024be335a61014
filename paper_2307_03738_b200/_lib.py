"""ctypes binding of libqigen_b200.so (include/qigen_b200.h).

The library is the only compute path: if it is missing or no CUDA device is
present, every op raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .config import ConfigError

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("QIGEN_B200_LIB", _HERE / "libqigen_b200.so"))

OK, ERR_CONFIG, ERR_PACK, ERR_PLAN, ERR_CUDA, ERR_ARG, ERR_UNSUPPORTED = range(7)
F32, F16, BF16 = 0, 1, 2


class QigenCudaError(RuntimeError):
    """A CUDA runtime failure inside libqigen_b200."""


class UnsupportedError(ValueError):
    """The combination is valid for the reference but not implemented here."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int

class ChainOpts(ctypes.Structure):
    """qigen_gemv_chain_opts (include/qigen_b200.h)."""
    _fields_ = [("x_digits", _P), ("ss_in", _P), ("ss_count", _I32), ("eps", ctypes.c_float),
                ("y_digits", _P), ("out_scale", _P), ("out_group", _I64), ("ss_out", _P)]


class StackLayer(ctypes.Structure):
    """qigen_stack_layer (include/qigen_b200.h)."""
    _fields_ = [("qw", _P * 4), ("qsz", _P * 4), ("norm1", _P), ("norm2", _P),
                ("k_cache", _P), ("v_cache", _P)]


class StackDesc(ctypes.Structure):
    """qigen_stack_desc (include/qigen_b200.h)."""
    _fields_ = [("layers", _I32), ("d_model", _I32), ("heads", _I32), ("head_dim", _I32),
                ("ffn", _I32), ("bits", _I32), ("group_size", _I64), ("ctx", _I64),
                ("eps", ctypes.c_float)]


class GemvDesc(ctypes.Structure):
    """qigen_gemv_desc (include/qigen_b200.h)."""
    _fields_ = [("qw", _P), ("qsz", _P), ("n", _I64), ("m", _I64), ("bits", _I32),
                ("group_size", _I64), ("x", _P), ("x_dtype", _I32), ("tokens", _I64),
                ("ldx", _I64), ("y", _P), ("ldy", _I64)]


# name -> (restype, argtypes)
SIGNATURES = {
    "qigen_version": (_I32, []),
    "qigen_last_error": (ctypes.c_char_p, []),
    "qigen_quantize": (_I32, [_P, _I64, _I64, _I32, _I64, _I32, _P, _P, _P, _P]),
    "qigen_dequantize": (_I32, [_P, _P, _P, _I64, _I64, _I64, _P, _P]),
    "qigen_pack_rowseq": (_I32, [_P, _I64, _I64, _I32, _P, _P]),
    "qigen_unpack_rowseq": (_I32, [_P, _I64, _I64, _I32, _P, _P]),
    "qigen_permute_zcurve": (_I32, [_P, _P, _I64, _I64, _I32, _I64, _I64, _P, _I64, _I32, _P]),
    "qigen_panel_words": (_I64, [_I64, _I64, _I32]),
    "qigen_panel_params": (_I64, [_I64, _I64, _I64]),
    "qigen_panels_from_codes": (_I32, [_P, _P, _P, _I64, _I64, _I32, _I64, _P, _P, _P]),
    "qigen_panels_to_codes": (_I32, [_P, _I64, _I64, _I32, _P, _P]),
    "qigen_panels_from_rowseq": (_I32, [_P, _P, _P, _I64, _I64, _I32, _I64, _P, _P, _P]),
    "qigen_input_sums": (_I32, [_P, _I64, _I64, _P, _P]),
    "qigen_gemv": (_I32, [_P, _P, _I64, _I64, _I32, _I64, _P, _I32, _I64, _I64, _P, _I64,
                          _I32, _I32, _P]),
    "qigen_gemv_workspace_size": (_I64, [_I64, _I64]),
    "qigen_gemv_ex": (_I32, [_P, _P, _I64, _I64, _I32, _I64, _P, _I32, _I64, _I64, _P, _I64,
                             _I32, _I32, _I32, _P, ctypes.c_float, _P, _I64, _P]),
    "qigen_debug_max_split": (_I32, [_I32]),
    "qigen_debug_norm_prep": (_I32, [_I32]),
    "qigen_gemv_group_create": (_I32, [_I32, _P, ctypes.POINTER(_P)]),
    "qigen_gemv_group_run": (_I32, [_P, _P]),
    "qigen_gemv_group_destroy": (_I32, [_P]),
    "qigen_gemv_group_run_rebased": (_I32, [_P, _P, _P, _P]),
    "qigen_gemv_group_run_host": (_I32, [_P, _P, _P, ctypes.c_size_t, _P, _P, ctypes.c_size_t, _P]),
    "qigen_rope_kv": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _I64, _I64, _P]),
    "qigen_rmsnorm_f16": (_I32, [_P, _P, _I64, _I64, ctypes.c_float, _P, _P]),
    "qigen_attn_decode_workspace_size": (_I64, [_I64, _I64, _I64, _I64]),
    "qigen_attn_decode": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64,
                                 ctypes.c_float, _P, _P, _I64, _P]),
    "qigen_gemv_ss_count": (_I64, [_I64]),
    "qigen_gemv_chain": (_I32, [_P, _P, _I64, _I64, _I32, _I64, _P, _I32, _I64, _I64, _P, _I64,
                                _I32, _I32, _P, ctypes.c_float, _P, _I64, _P, _P]),
    "qigen_tp_buffer_size": (_I64, [_I32, _I64, _I64]),
    "qigen_tp_alloc": (_I32, [_I64, ctypes.POINTER(_P), _P]),
    "qigen_tp_free": (_I32, [_P]),
    "qigen_tp_open_peer": (_I32, [_P, ctypes.POINTER(_P)]),
    "qigen_tp_close_peer": (_I32, [_P]),
    "qigen_tp_create": (_I32, [_I32, _I32, _I64, _I64, _I32, _P, ctypes.POINTER(_P)]),
    "qigen_tp_destroy": (_I32, [_P]),
    "qigen_tp_step_begin": (_I32, [_P, _P]),
    "qigen_gemv_tp_push": (_I32, [_P, _I32, _P, _P, _I64, _I64, _I32, _I64, _P, _I32, _I64, _I64,
                                  _I32, _P, ctypes.c_float, _P, _I64, _P]),
    "qigen_tp_reduce": (_I32, [_P, _I32, _I32, _P, _I64, _P]),
    "qigen_tp_error": (_I32, [_P, ctypes.POINTER(_I32)]),
    "qigen_lm_head_workspace_size": (_I64, [_I64, _I64, _I64]),
    "qigen_lm_head": (_I32, [_P, _P, ctypes.c_float, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P,
                             _I64, _P]),
    "qigen_attn_decode_chain": (_I32, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64,
                                       ctypes.c_float, _P, _P, _I64, _P, _I64, _P]),
    "qigen_gemm_tc_workspace_size": (_I64, [_I64, _I64]),
    "qigen_gemm_tc": (_I32, [_P, _P, _I64, _I64, _I32, _I64, _P, _I32, _I64, _I64, _P, _I64, _I32,
                             _I32, _P, _I64, _P]),
    "qigen_debug_trace": (_I32, [_P]),
    "qigen_debug_trace_clk": (_I32, [_P]),
    "qigen_debug_prefetch": (_I32, [_I32]),
    "qigen_debug_force_prep": (_I32, [_I32]),
    "qigen_debug_early_trigger": (_I32, [_I32]),
    "qigen_debug_gemv_tuning": (_I32, [_I32, _I32, _I32, _I32]),
    "qigen_debug_tc_mode": (_I32, [_I32]),
    "qigen_debug_group_mode": (_I32, [_I32]),
    "qigen_debug_attn_trace": (_I32, [_P]),
    "qigen_debug_attn_splits": (_I32, [_I32]),
    "qigen_decode_stack_create": (_I32, [_P, _P, ctypes.POINTER(_P)]),
    "qigen_decode_stack_run": (_I32, [_P, _P, _P, _P, _P, _I64, ctypes.c_float, _P]),
    "qigen_decode_stack_error": (_I32, [_P, ctypes.POINTER(_I32)]),
    "qigen_decode_stack_info": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                       ctypes.POINTER(_I32)]),
    "qigen_decode_stack_destroy": (_I32, [_P]),
    "qigen_debug_stack_tuning": (_I32, [_I32, _I32, _I32]),
    "qigen_debug_stack_mode": (_I32, [_I32]),
    "qigen_weights_create": (_I32, [_P, _I32, _I64, _I64, _I32, _I64, _I64, _I64, _P, _I64,
                                    _P, _P, _P, ctypes.POINTER(_P)]),
    "qigen_weights_destroy": (_I32, [_P]),
    "qigen_weights_gemv": (_I32, [_P, _P, _I32, _I64, _P, _I32, _P]),
    "qigen_weights_gemv_host": (_I32, [_P, _P, _I64, _P, _P]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    """Map a qigen_status onto the reference's exception classes."""
    if status == OK:
        return
    msg = lib().qigen_last_error().decode(errors="replace")
    if status == ERR_CONFIG:
        raise ConfigError(msg)
    if status == ERR_PACK:
        from .packing import PackError
        raise PackError(msg)
    if status == ERR_PLAN:
        from .perfmodel import PlanError
        raise PlanError(msg)
    if status == ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == ERR_CUDA:
        raise QigenCudaError(msg)
    raise ValueError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
