"""numpy mirror of `lowbit.igemm` (pkg/src/lowbit/igemm.py) over the B200
kernels (paper_2206_01861_b200.igemm): the tcgen05 integer GEMM, the fused
dequant epilogue, and the fused LayerNorm / GeLU quantizers."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import igemm as _dev
from ..errors import ShapeError, UsageError
from ..igemm import INT32_LIMIT, DynamicAct, FullAct, StaticAct, check_overflow_guard  # noqa: F401
from .quant import QuantizedActivation, QuantizedMatrix, _host

F32 = np.float32
ActMode = DynamicAct | StaticAct | FullAct


@dataclass
class IntAccumulator:
    """igemm.py:45-49 (numpy int32)."""

    acc: np.ndarray


def _dev_w(w) -> "_dev.quant.QuantizedMatrix":
    return w.device() if isinstance(w, QuantizedMatrix) else w


def igemm(xq: QuantizedActivation, wq: QuantizedMatrix) -> IntAccumulator:
    """igemm.py:66-80"""
    if xq.values.shape[1] != wq.cols:
        raise ShapeError(
            f"igemm inner dimensions differ: activation {xq.values.shape} vs weight {wq.values.shape}")
    check_overflow_guard(wq.cols, xq.bits, wq.bits)
    return IntAccumulator(acc=_host(_dev.igemm(xq.device(), _dev_w(wq)).acc))


def dequant_epilogue(acc: IntAccumulator, act_scales, w: QuantizedMatrix, bias=None) -> np.ndarray:
    """igemm.py:83-112"""
    a = np.asarray(acc.acc, dtype=np.int32)
    if w.rows != a.shape[1]:
        raise ShapeError(f"epilogue weight rows {w.rows} != accumulator cols {a.shape[1]}")
    dacc = _dev.IntAccumulator(torch.from_numpy(np.ascontiguousarray(a)).cuda())
    return _host(_dev.dequant_epilogue(dacc, act_scales, _dev_w(w), bias))


def quantized_linear(x, w: QuantizedMatrix, bias, act_mode: ActMode) -> np.ndarray:
    """igemm.py:115-139"""
    if not isinstance(act_mode, (DynamicAct, StaticAct, FullAct)):
        raise UsageError(f"unknown activation mode {act_mode!r}")
    return _host(_dev.quantized_linear(x, _dev_w(w), bias, act_mode))


def layer_norm_quantize(x, gamma, beta, bits: int, eps: float = 1e-5) -> QuantizedActivation:
    """igemm.py:150-157"""
    return QuantizedActivation.from_device(_dev.layer_norm_quantize(x, gamma, beta, bits, eps))


def gelu_quantize(x, bits: int) -> QuantizedActivation:
    """igemm.py:160-161"""
    return QuantizedActivation.from_device(_dev.gelu_quantize(x, bits))
