"""Drop-in mirror of `lowbit.igemm` (pkg/src/lowbit/igemm.py) on B200.

* `igemm` runs the tcgen05 kind::i8 tensor-core kernel with exact int32
  accumulation in TMEM (igemm.py:66-80);
* `quantized_linear` fuses igemm + `dequant_epilogue` into one kernel whose
  epilogue reads the TMEM accumulator and applies ((f32(acc)*s_tok)*s_w)+bias in
  the reference's strict float32 order (igemm.py:83-112); no dequantized matrix
  is ever materialised on this path;
* `layer_norm_quantize` / `gelu_quantize` are single fused kernels
  (igemm.py:150-161).
Optional B200 extension: `out_dtype` (float32 default, float16/bfloat16 = RN
cast of the exact float32 result).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import quant
from .errors import ShapeError, UsageError
from .quant import QuantizedActivation, QuantizedMatrix, as_device_f32, qmax

INT32_LIMIT = 1 << 31
F32 = np.float32

_OUT_CODES = {torch.float32: N.OUT_F32, torch.float16: N.OUT_F16, torch.bfloat16: N.OUT_BF16}


@dataclass(frozen=True)
class DynamicAct:
    """igemm.py:26-28"""

    bits: int = 8


@dataclass(frozen=True)
class StaticAct:
    """igemm.py:31-34"""

    scale: float
    bits: int = 8


@dataclass(frozen=True)
class FullAct:
    """igemm.py:37-39"""


ActMode = DynamicAct | StaticAct | FullAct


@dataclass
class IntAccumulator:
    """igemm.py:45-49: exact int32 accumulator (tokens x out) on device."""

    acc: torch.Tensor


def check_overflow_guard(inner_dim: int, act_bits: int, weight_bits: int) -> None:
    """igemm.py:52-63"""
    worst = inner_dim * qmax(act_bits) * qmax(weight_bits)
    if worst >= INT32_LIMIT:
        raise UsageError(
            f"igemm overflow guard: inner dim {inner_dim} with {act_bits}x{weight_bits}-bit "
            f"operands can reach {worst} >= 2^31"
        )


def igemm(xq: QuantizedActivation, wq: QuantizedMatrix, out: torch.Tensor | None = None) -> IntAccumulator:
    """igemm.py:66-80: acc[i][j] = sum_p xq[i][p] * wq[j][p], exact int32.
    `out` (B200 extension): a caller-owned int32 [tokens, n] destination."""
    if xq.values.shape[1] != wq.cols:
        raise ShapeError(
            f"igemm inner dimensions differ: activation {tuple(xq.values.shape)} vs weight "
            f"{tuple(wq.values.shape)}"
        )
    check_overflow_guard(wq.cols, xq.bits, wq.bits)
    a = xq.gemm_operand()
    m, k = a.shape
    n = wq.rows
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a.device)
    elif out.dtype != torch.int32 or tuple(out.shape) != (m, n) or out.stride(1) != 1:
        raise ShapeError(f"igemm out must be int32 {(m, n)} with unit column stride")
    acc = out
    wp, ld_w, wb = wq.weight_operand()
    N.call("zq_igemm_s32", a.data_ptr(), a.stride(0), wp, ld_w, wb, m, n, k, acc.data_ptr(),
           acc.stride(0), N.stream_ptr())
    return IntAccumulator(acc=acc)


def _act_scale_args(act_scales, tokens: int):
    """(token-scale pointer or None, static f32 scale) per igemm.py:98-106."""
    if isinstance(act_scales, (float, int, np.floating)) and not isinstance(act_scales, bool):
        return None, float(F32(act_scales)), None
    ts = act_scales if isinstance(act_scales, torch.Tensor) else torch.as_tensor(
        np.asarray(act_scales, dtype=F32))
    ts = ts.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=torch.float32).contiguous()
    if tuple(ts.shape) != (tokens,):
        raise UsageError(
            f"epilogue needs one activation scale per token: got {tuple(ts.shape)} for {tokens} tokens"
        )
    return ts.data_ptr(), 0.0, ts


def dequant_epilogue(acc: IntAccumulator, act_scales, w: QuantizedMatrix, bias=None,
                     out_dtype: torch.dtype = torch.float32, out: torch.Tensor | None = None) -> torch.Tensor:
    """igemm.py:83-112: out = acc * act_scale(i) * group_scale(group_of(j)) + bias[j].
    `out` (B200 extension): caller-owned destination (its dtype wins)."""
    a = acc.acc
    m, n = a.shape
    if w.rows != n:
        raise ShapeError(f"epilogue weight rows {w.rows} != accumulator cols {n}")
    ts_ptr, sscale, _keep = _act_scale_args(act_scales, m)
    b = None if bias is None else as_device_f32(bias).reshape(-1)
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=a.device)
    elif tuple(out.shape) != (m, n) or out.stride(1) != 1 or out.dtype not in _OUT_CODES:
        raise ShapeError(f"epilogue out must be {(m, n)} float32/float16/bfloat16 with unit column stride")
    N.call("zq_dequant_epilogue", a.data_ptr(), a.stride(0), ts_ptr, sscale,
           w.row_scales().data_ptr(), N.ptr(b), m, n, out.data_ptr(), out.stride(0),
           _OUT_CODES[out.dtype], N.stream_ptr())
    return out


def fused_linear(xq: QuantizedActivation, w: QuantizedMatrix, bias=None,
                 out_dtype: torch.dtype = torch.float32, out: torch.Tensor | None = None
                 ) -> torch.Tensor:
    """igemm + dequant_epilogue in one tcgen05 kernel (the fused hot op)."""
    if xq.values.shape[1] != w.cols:
        raise ShapeError(
            f"igemm inner dimensions differ: activation {tuple(xq.values.shape)} vs weight "
            f"{tuple(w.values.shape)}"
        )
    check_overflow_guard(w.cols, xq.bits, w.bits)
    a = xq.gemm_operand()
    m, k = a.shape
    n = w.rows
    if xq.token_scales is not None:
        ts_ptr, sscale = xq.token_scales.data_ptr(), 0.0
    else:
        ts_ptr, sscale = None, float(F32(xq.static_scale))
    b = None if bias is None else as_device_f32(bias).reshape(-1)
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=a.device)
    wp, ld_w, wb = w.weight_operand()
    N.call("zq_linear", a.data_ptr(), a.stride(0), ts_ptr, sscale, wp, ld_w, wb,
           w.row_scales().data_ptr(), N.ptr(b), m, n, k, out.data_ptr(), out.stride(0),
           _OUT_CODES[out.dtype], N.stream_ptr())
    return out


FULL_PRECISIONS = ("exact", "f16", "f16x2")


def full_linear(x, w: QuantizedMatrix, bias=None, precision: str = "exact",
                out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """FullAct: x @ dequant(w).T + bias (igemm.py:127-130).

    precision="exact": the reference's sequential float32 accumulation
    (tensor.py:37-56), bit-exact, CUDA cores.  "f16" / "f16x2" (B200 tolerance
    modes, the paper's A16 deployment): tcgen05 kind::f16 CTA pairs with the
    weights converted int8/INT4 -> f16 in shared memory and each activation row
    scaled by a power of two into 1 (fp16) or 2 (hi + lo, ~22 bits) f16 terms.
    Tolerances vs the reference (tests/test_wo_gpu.py): f16 max|err| <= 2e-3 *
    max|ref|, f16x2 <= 5e-5 * max|ref|."""
    if precision not in FULL_PRECISIONS:
        raise UsageError(f"full_linear precision must be one of {FULL_PRECISIONS}, got {precision!r}")
    xt = as_device_f32(x)
    if xt.dim() != 2 or xt.shape[1] != w.cols:
        raise ShapeError(f"matmul inner dimensions differ: {tuple(xt.shape)} x {(w.cols, w.rows)}")
    m, k = xt.shape
    n = w.rows
    b = None if bias is None else as_device_f32(bias).reshape(-1)
    wp, ld_w, wb = w.weight_operand()
    if precision == "exact":
        if out_dtype != torch.float32:
            raise UsageError("the exact FullAct path produces float32 (as the reference)")
        out = torch.empty((m, n), dtype=torch.float32, device=xt.device)
        N.call("zq_linear_full", xt.data_ptr(), xt.stride(0), wp, ld_w, wb, w.row_scales().data_ptr(),
               N.ptr(b), m, n, k, out.data_ptr(), out.stride(0), N.stream_ptr())
        return out
    terms = 1 if precision == "f16" else 2
    ld_h = (k + 7) // 8 * 8
    hi = torch.empty((m, ld_h), dtype=torch.float16, device=xt.device)
    lo = torch.empty((m, ld_h), dtype=torch.float16, device=xt.device) if terms == 2 else None
    row_inv = torch.empty(m, dtype=torch.float32, device=xt.device)
    N.call("zq_act_split16", xt.data_ptr(), xt.stride(0), m, k, terms, hi.data_ptr(), N.ptr(lo), ld_h,
           row_inv.data_ptr(), None, N.stream_ptr())
    out = torch.empty((m, n), dtype=out_dtype, device=xt.device)
    N.call("zq_linear_wo", hi.data_ptr(), N.ptr(lo), ld_h, row_inv.data_ptr(), wp, ld_w, wb,
           w.row_scales().data_ptr(), N.ptr(b), m, n, k, out.data_ptr(), out.stride(0), _OUT_CODES[out.dtype],
           N.stream_ptr())
    return out


def quantized_linear(x, w: QuantizedMatrix, bias, act_mode: ActMode,
                     out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """igemm.py:115-139: x @ dequant(w).T + bias through the fused integer path."""
    if isinstance(act_mode, FullAct):
        return full_linear(x, w, bias)
    if isinstance(act_mode, DynamicAct):
        xq = quant.quantize_activation_tokenwise(x, act_mode.bits)
        return fused_linear(xq, w, bias, out_dtype)
    if isinstance(act_mode, StaticAct):
        xq = quant.quantize_activation_static(x, act_mode.scale, act_mode.bits)
        return fused_linear(xq, w, bias, out_dtype)
    raise UsageError(f"unknown activation mode {act_mode!r}")


def layer_norm_quantize(x, gamma, beta, bits: int, eps: float = 1e-5, *, residual=None,
                        ln_out: torch.Tensor | None = None, check_finite: bool = True,
                        flag: quant.FiniteFlag | None = None) -> QuantizedActivation:
    """igemm.py:150-157 fused (K4): LN (numpy pairwise order) + token-wise quantize.
    `residual` (B200 extension) adds x + residual first, as block_forward does
    before each LayerNorm (transformer.py:477, :486); `ln_out` receives the float
    LN output when given."""
    quant._check_bits(bits)
    if eps <= 0:
        raise ValueError(f"layer_norm eps must be > 0, got {eps}")
    xt = as_device_f32(x)
    if xt.dim() != 2 or xt.shape[0] < 1:
        raise UsageError(f"activations must be (tokens x dim), got shape {tuple(xt.shape)}")
    rows, cols = xt.shape
    g = as_device_f32(gamma).reshape(-1)
    b = as_device_f32(beta).reshape(-1)
    if g.shape != (cols,) or b.shape != (cols,):
        raise ShapeError(
            f"layer_norm params {tuple(g.shape)}/{tuple(b.shape)} do not match row width {cols}")
    r = None if residual is None else as_device_f32(residual)
    if r is not None and r.shape != xt.shape:
        raise ShapeError(f"residual {tuple(r.shape)} does not match {tuple(xt.shape)}")
    q = quant.padded_int8(rows, cols)
    s = torch.empty(rows, dtype=torch.float32, device=xt.device)
    fl = flag or quant.FiniteFlag()
    N.call("zq_layer_norm_quantize", xt.data_ptr(), N.ptr(r), g.data_ptr(), b.data_ptr(), rows,
           cols, float(F32(eps)), bits, N.ptr(ln_out), q.data_ptr(), q.stride(0), s.data_ptr(),
           fl.ptr, N.stream_ptr())
    if check_finite:
        fl.check("activations")
    return QuantizedActivation(values=q, bits=bits, token_scales=s)


def gelu_quantize(x, bits: int, *, gelu_out: torch.Tensor | None = None,
                  check_finite: bool = True, flag: quant.FiniteFlag | None = None
                  ) -> QuantizedActivation:
    """igemm.py:160-161 fused (K5): exact-erf GeLU (f64, rounded once) + quantize."""
    quant._check_bits(bits)
    xt = as_device_f32(x)
    if xt.dim() != 2 or xt.shape[0] < 1:
        raise UsageError(f"activations must be (tokens x dim), got shape {tuple(xt.shape)}")
    rows, cols = xt.shape
    q = quant.padded_int8(rows, cols)
    s = torch.empty(rows, dtype=torch.float32, device=xt.device)
    fl = flag or quant.FiniteFlag()
    N.call("zq_gelu_quantize", xt.data_ptr(), rows, cols, cols, bits, N.ptr(gelu_out),
           q.data_ptr(), q.stride(0), s.data_ptr(), fl.ptr, N.stream_ptr())
    if check_finite:
        fl.check("activations")
    return QuantizedActivation(values=q, bits=bits, token_scales=s)
