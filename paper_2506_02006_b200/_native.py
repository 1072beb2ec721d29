"""ctypes binding of the C ABI in include/morphserve.h (libmorphserve.so).

The product path is this library; there is no CPU or PyTorch fallback.  If the
library is missing the import fails loudly (build it with
``python -m paper_2506_02006_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

_LIB_PATH = os.path.join(os.environ.get("MS_LIB_DIR") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib"),
                         "libmorphserve.so")

MS_OK, MS_EVALIDATION, MS_ERUNTIME, MS_ELOGIC = 0, 2, 3, 4


class MsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class MsValidationError(MsError, ValueError):
    """std::invalid_argument in the reference (exit code 2)."""


class MsLogicError(MsError):
    """std::logic_error in the reference (broken invariant)."""


class ModelDesc(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("hidden", C.c_int32), ("num_heads", C.c_int32),
        ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("block_tokens", C.c_int32), ("max_batch", C.c_int32), ("max_prefill_tokens", C.c_int32),
        ("max_pos", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_double),
        ("arena_pages", C.c_int64),
    ]


class DecodeBatch(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("slots", C.POINTER(C.c_int32)), ("positions", C.POINTER(C.c_int32)),
        ("tokens", C.POINTER(C.c_int32)), ("block_ids", C.POINTER(C.c_int64)), ("max_blocks", C.c_int32),
    ]


# (name, restype, argtypes) -- every symbol include/morphserve.h declares
_P = C.c_void_p
SIGNATURES = [
    ("ms_last_error", C.c_char_p, []),
    ("ms_page_bytes", C.c_int64, [C.POINTER(ModelDesc)]),
    ("ms_layer_pages", C.c_int64, [C.POINTER(ModelDesc), C.c_int]),
    ("ms_ctx_create", C.c_int, [C.c_int, C.POINTER(ModelDesc), C.POINTER(_P)]),
    ("ms_ctx_destroy", C.c_int, [_P]),
    ("ms_sync", C.c_int, [_P]),
    ("ms_num_sms", C.c_int, [_P]),
    ("ms_weights_synthetic", C.c_int, [_P, C.c_uint64]),
    ("ms_weights_upload", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int64]),
    ("ms_weights_finalize", C.c_int, [_P]),
    ("ms_variant_enable", C.c_int, [_P, C.c_int]),
    ("ms_variant_bytes", C.c_int64, [_P, C.c_int]),
    ("ms_variant_export", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int64]),
    ("ms_variant_register", C.c_int, [_P, C.c_int, C.c_int, _P, C.c_int64, C.c_int]),
    ("ms_swap_begin", C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    ("ms_swap_begin_peer", C.c_int, [_P, C.c_int, C.c_int, _P, C.POINTER(C.c_uint64)]),
    ("ms_swap_poll", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_int)]),
    ("ms_swap_wait", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_float)]),
    ("ms_swap_commit", C.c_int, [_P, C.c_uint64, C.POINTER(C.c_int64)]),
    ("ms_layer_bits", C.c_int, [_P, C.c_int]),
    ("ms_reset_state", C.c_int, [_P]),
    ("ms_kv_attach", C.c_int, [_P, C.c_int64, C.c_int64]),
    ("ms_kv_detach", C.c_int, [_P, C.POINTER(C.c_int64), C.c_int64]),
    ("ms_free_pages", C.c_int64, [_P]),
    ("ms_kv_page_of", C.c_int64, [_P, C.c_int64]),
    ("ms_kv_export", C.c_int, [_P, C.c_int64, _P, C.c_int64]),
    ("ms_graph_captures", C.c_int64, [_P]),
    ("ms_hist_reserve", C.c_int, [_P, C.c_int32, C.c_int32]),
    ("ms_hist_write", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32]),
    ("ms_hist_read", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32]),
    ("ms_set_stream", C.c_int, [_P, _P]),
    ("ms_decode_step", C.c_int, [_P, C.POINTER(DecodeBatch), C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    ("ms_decode_submit", C.c_int, [_P, C.POINTER(DecodeBatch)]),
    ("ms_decode_collect", C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    ("ms_prefill", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.c_int32,
                             C.POINTER(C.c_int32), C.POINTER(C.c_float)]),
    ("ms_prefill_trace", C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.c_int32,
                                   C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    ("ms_last_step_ms", C.c_int, [_P, C.POINTER(C.c_float)]),
    ("ms_kv_fill_synthetic", C.c_int, [_P, C.POINTER(C.c_int64), C.c_int64, C.c_uint64]),
    ("ms_launch_count", C.c_int64, [_P]),
    ("ms_timer_start", C.c_int, [_P]),
    ("ms_timer_stop", C.c_int, [_P, C.POINTER(C.c_float)]),
    ("ms_prof_attention", C.c_int, [_P, C.c_int]),
    ("ms_prof_kernels", C.c_int, [_P, C.c_int]),
    ("ms_prof_kernels_read", C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_int64)]),
    ("ms_prof_attention_read", C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_int64)]),
    ("ms_k_gen_weight", C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double, _P, _P]),
    ("ms_k_pack_bf16", C.c_int, [_P, C.c_int, C.c_int, _P, _P]),
    ("ms_k_quant", C.c_int, [C.c_int, _P, C.c_int, C.c_int, _P, _P, _P]),
    ("ms_k_quant_w4", C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P]),
    ("ms_k_pack_act", C.c_int, [_P, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("ms_k_gemm", C.c_int, [C.c_int, _P, C.c_int, C.c_int, _P, C.c_int, C.c_int, C.c_int, _P,
                            C.POINTER(C.c_int), _P]),
    ("ms_k_attn_prefill", C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P, C.c_int,
                                    _P, _P]),
    ("ms_k_attn_decode", C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P,
                                   C.c_int, _P, C.c_int, C.c_int, _P, _P, _P]),
]

_lib = None


def lib():
    """Loads libmorphserve.so (raises if it was not built: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(
                f"{_LIB_PATH} is missing; build it with `python -m paper_2506_02006_b200.build` "
                "(the serving hot path has no CPU fallback)")
        L = C.CDLL(_LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == MS_OK:
        return
    msg = lib().ms_last_error().decode()
    if rc == MS_EVALIDATION:
        raise MsValidationError(rc, msg)
    if rc == MS_ELOGIC:
        raise MsLogicError(rc, msg)
    raise MsError(rc, msg)


def i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32)) if a is not None else None


def i64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64)) if a is not None else None


def f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float)) if a is not None else None
