"""ctypes binding of the C-ABI library `libzq_b200.so` (include/zq_b200.h).

This is the only path to compute in the package: there is no CPU or eager
PyTorch fallback.  If the library is missing, or no CUDA device is present, the
first call raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ShapeError, UsageError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZQ_LIB") or os.path.join(_HERE, "libzq_b200.so")  # ZQ_LIB: experiment builds

ZQ_OK, ZQ_ERR_USAGE, ZQ_ERR_SHAPE, ZQ_ERR_CUDA, ZQ_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
OUT_F32, OUT_F16, OUT_BF16 = 0, 1, 2

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f32 = ctypes.c_float
_f64 = ctypes.c_double

# name -> argtypes (all return int status, except the two string getters)
_SIGS = {
    "zq_quantize_tokenwise": [_p, _i64, _i64, _i64, _i32, _p, _i64, _p, _p, _p],
    "zq_quantize_static": [_p, _i64, _i64, _i64, _f64, _i32, _p, _i64, _p, _p],
    "zq_quantize_weight_groupwise": [_p, _i64, _i64, _i64, _i32, _p, _i64, _p, _p, _p, _p, _p],
    "zq_pack_int4": [_p, _i64, _i64, _p, _p],
    "zq_layer_norm_quantize": [_p, _p, _p, _p, _i64, _i64, _f32, _i32, _p, _p, _i64, _p, _p, _p],
    "zq_gelu_quantize": [_p, _i64, _i64, _i64, _i32, _p, _p, _i64, _p, _p, _p],
    "zq_igemm_s32": [_p, _i64, _p, _i64, _i32, _i64, _i64, _i64, _p, _i64, _p],
    "zq_linear": [_p, _i64, _p, _f32, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _i32, _p],
    "zq_linear_ln_quantize": [_p, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _p, _p, _f32, _i32, _p,
                              _p, _i64, _p, _p, _i64, _p, _p],
    "zq_dequant_epilogue": [_p, _i64, _p, _f32, _p, _p, _i64, _i64, _p, _i64, _i32, _p],
    "zq_linear_full": [_p, _i64, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _p],
    "zq_row_absmax": [_p, _i64, _i64, _i64, _p, _p, _p],
    "zq_row_absmax_f64": [_p, _i64, _i64, _i64, _p, _p, _p],
    "zq_quantize_array_f64": [_p, _i64, _f64, _i32, _p, _p, _p],
    "zq_quantize_with_absmax": [_p, _i64, _i64, _i64, _p, _i32, _p, _i64, _p, _p],
    "zq_gemm_set_trace": [_p],
    "zq_attention_debug": [_i32],
    "zq_attention_set_trace": [_p],
    "zq_gelu_estimate": [_p, _i64, _p, _p, _p],
    "zq_attention_f32": [_p, _i64, _i32, _i32, _i32, _i32, _i32, _f32, _p, _i64, _p],
    "zq_kv_append": [_p, _i64, _i32, _i32, _i32, _p, _p, _p, _i64, _p],
    "zq_decode_attention_f32": [_p, _i64, _p, _p, _i64, _i32, _i32, _i32, _p, _f32, _p, _i64, _i32, _p],
    "zq_decode_attention_chunks": [_i32, _i32, _i64],
    "zq_linear_kv": [_p, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _p, _i32, _i64,
                     _p],
    "zq_l2_persist": [_p, _p, _i64, _p],
    "zq_matmul_f32_seq": [_p, _i64, _p, _i64, _p, _i64, _i64, _i64, _p, _i64, _p],
    "zq_attention_exact_f32": [_p, _i64, _i32, _i32, _i32, _i32, _f32, _p, _p, _i64, _p],
    "zq_minmax_f32": [_p, _i64, _p, _p, _p],
    "zq_np_expf": [_p, _i64, _p, _p],
    "zq_lm_head_argmax": [_p, _i64, _i32, _p, _i64, _i64, _f32, _p, _p, _p, _p, _p, _p],
    "zq_lm_embed_split": [_p, _i64, _i64, _f32, _p, _p, _p],
    "zq_lm_head_argmax_split": [_p, _i64, _i32, _p, _p, _i64, _i64, _f32, _p, _p, _p, _p, _p, _p],
    "zq_linear_ws": [_p, _i64, _p, _f32, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _i32, _p, _i64, _p],
    "zq_linear_kv_ws": [_p, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _p, _i32, _i64,
                        _p, _i64, _p],
    "zq_linear_kv_prefill": [_p, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _p, _p, _i32, _i64,
                             _i32, _p],
    "zq_igemm_s32_ws": [_p, _i64, _p, _i64, _i32, _i64, _i64, _i64, _p, _i64, _p, _i64, _p],
    "zq_act_split16": [_p, _i64, _i64, _i64, _i32, _p, _p, _i64, _p, _p, _p],
    "zq_linear_wo": [_p, _p, _i64, _p, _p, _i64, _i32, _p, _p, _i64, _i64, _i64, _p, _i64, _i32, _p],
    "zq_qkv_attention": [_p, _i64, _p, _p, _i64, _p, _p, _i32, _i32, _i32, _i32, _i32, _f32, _p, _i64, _p],
}

_lock = threading.Lock()
_lib = None


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is missing: the product path refuses to run."""


def exported_symbols() -> list[str]:
    return sorted(_SIGS) + ["zq_version", "zq_last_error", "zq_linear_ws_bytes"]


def load(require_device: bool = True):
    """Load libzq_b200.so (once).  Raises NativeUnavailable loudly on failure."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` or `make`"
            )
        if require_device:
            import torch

            if not torch.cuda.is_available():
                raise NativeUnavailable("no CUDA device: the ZeroQuant B200 path has no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.zq_linear_ws_bytes.argtypes = [_i64, _i64]
        lib.zq_linear_ws_bytes.restype = ctypes.c_int64
        lib.zq_version.restype = ctypes.c_char_p
        lib.zq_last_error.restype = ctypes.c_char_p
        _lib = lib
        return lib


def load_for_inspection():
    """Load without requiring a GPU (symbol checks in the CPU test suite)."""
    return ctypes.CDLL(LIB_PATH)


def check(rc: int) -> None:
    if rc == ZQ_OK:
        return
    msg = _lib.zq_last_error().decode(errors="replace") if _lib is not None else ""
    if rc == ZQ_ERR_SHAPE:
        raise ShapeError(msg)
    if rc in (ZQ_ERR_USAGE, ZQ_ERR_UNSUPPORTED):
        raise UsageError(msg)
    raise RuntimeError(f"zq_b200 CUDA failure: {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args))


def call_rc(name: str, *args) -> int:
    """Like call() but hands ZQ_ERR_UNSUPPORTED back (for entry points with a
    caller-side alternative); any other failure raises."""
    rc = getattr(load(), name)(*args)
    if rc != ZQ_ERR_UNSUPPORTED:
        check(rc)
    return rc


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int | None:
    """Device pointer of a tensor, or None (NULL) for None."""
    return None if t is None else t.data_ptr()
