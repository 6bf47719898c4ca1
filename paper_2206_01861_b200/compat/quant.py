"""numpy mirror of `lowbit.quant` (pkg/src/lowbit/quant.py) over the B200
kernels.  Same names, fields, arguments and errors; arrays in and out are
numpy; the arithmetic runs on device (paper_2206_01861_b200.quant)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .. import quant as _dev
from ..errors import UsageError
from ..quant import (  # noqa: F401  (host logic, identical to the reference)
    SUPPORTED_BITS,
    Granularity,
    Mode,
    QuantSpec,
    _check_bits,
    group_layout_for,
    qmax,
)

F32 = np.float32


def _host(t: torch.Tensor) -> np.ndarray:
    return np.ascontiguousarray(t.detach().cpu().numpy())


def _zeros_int8(rows: int, cols: int, align: int) -> torch.Tensor:
    ld = max(align, _dev.round_up(cols, align))
    return torch.zeros((rows, ld), dtype=torch.int8, device="cuda")[:, :cols]


def compute_scale(values, bits: int) -> float:
    """quant.py:80-95"""
    return _dev.compute_scale(values, bits)


def quantize_array(x, scale: float, bits: int) -> np.ndarray:
    """quant.py:103-113"""
    return _host(_dev.quantize_array(x, scale, bits))


def quantize_value(x: float, scale: float, bits: int) -> int:
    """quant.py:116-118"""
    return _dev.quantize_value(x, scale, bits)


def dequantize_array(q, scale: float) -> np.ndarray:
    """quant.py:121-122"""
    return _host(_dev.dequantize_array(np.asarray(q, dtype=F32), scale))


def dequantize_value(q: int, scale: float) -> float:
    """quant.py:125-126"""
    return float(dequantize_array(np.asarray([q]), scale)[0])


@dataclass
class QuantizedMatrix:
    """quant.py:134-181 (numpy fields).  `device()` is the HBM-resident copy the
    kernels read (padded int8 / packed INT4 payload + per-row scales), built on
    first use and rebuilt if the numpy payload is replaced."""

    values: np.ndarray
    bits: int
    group_scales: np.ndarray
    group_layout: list[tuple[int, int]]

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def cols(self) -> int:
        return self.values.shape[1]

    @property
    def num_groups(self) -> int:
        return len(self.group_layout)

    def logical_bits(self) -> int:
        return self.rows * self.cols * self.bits + 32 * self.num_groups

    def row_scales(self) -> np.ndarray:
        """quant.py:165-170"""
        out = np.empty(self.rows, dtype=F32)
        for (start, count), s in zip(self.group_layout, self.group_scales):
            out[start: start + count] = s
        return out

    def dequantize(self) -> np.ndarray:
        """quant.py:172-174 (reference / Full path only)."""
        return _host(self.device().dequantize())

    def group_of_row(self, row: int) -> int:
        for gi, (start, count) in enumerate(self.group_layout):
            if start <= row < start + count:
                return gi
        raise UsageError(f"row {row} outside group layout of {self.rows} rows")

    def device(self) -> _dev.QuantizedMatrix:
        key = (id(self.values), self.values.shape, self.bits, tuple(map(tuple, self.group_layout)),
               np.asarray(self.group_scales, F32).tobytes())
        cached = getattr(self, "_dev_cache", None)
        if cached is not None and cached[0] == key:
            return cached[1]
        v = np.asarray(self.values, dtype=np.int8)
        store = _zeros_int8(self.rows, self.cols, 32)
        store.copy_(torch.from_numpy(np.ascontiguousarray(v)).to(store.device))
        m = _dev.QuantizedMatrix(values=store, bits=self.bits,
                                 group_scales=torch.from_numpy(np.asarray(self.group_scales, F32).copy()).cuda(),
                                 group_layout=list(self.group_layout),
                                 row_scale_vec=torch.from_numpy(self.row_scales()).cuda())
        object.__setattr__(self, "_dev_cache", (key, m))
        return m

    @classmethod
    def from_device(cls, m: _dev.QuantizedMatrix) -> "QuantizedMatrix":
        out = cls(values=_host(m.values), bits=m.bits, group_scales=_host(m.group_scales),
                  group_layout=list(m.group_layout))
        key = (id(out.values), out.values.shape, out.bits, tuple(map(tuple, out.group_layout)),
               np.asarray(out.group_scales, F32).tobytes())
        object.__setattr__(out, "_dev_cache", (key, m))
        return out


@dataclass
class QuantizedActivation:
    """quant.py:183-208 (numpy fields)."""

    values: np.ndarray
    bits: int
    token_scales: np.ndarray | None = None
    static_scale: float | None = None

    def __post_init__(self):
        if (self.token_scales is None) == (self.static_scale is None):
            raise UsageError("exactly one of token_scales / static_scale must be populated")

    @property
    def tokens(self) -> int:
        return self.values.shape[0]

    def scales_per_token(self) -> np.ndarray:
        if self.token_scales is not None:
            return self.token_scales
        return np.full(self.tokens, F32(self.static_scale), dtype=F32)

    def dequantize(self) -> np.ndarray:
        return _host(self.device().dequantize())

    def device(self) -> _dev.QuantizedActivation:
        v = np.asarray(self.values, dtype=np.int8)
        store = _zeros_int8(v.shape[0], v.shape[1], 16)
        store.copy_(torch.from_numpy(np.ascontiguousarray(v)).to(store.device))
        if self.token_scales is not None:
            return _dev.QuantizedActivation(values=store, bits=self.bits,
                                            token_scales=torch.from_numpy(np.asarray(self.token_scales, F32).copy()).cuda())
        return _dev.QuantizedActivation(values=store, bits=self.bits, static_scale=float(self.static_scale))

    @classmethod
    def from_device(cls, a: _dev.QuantizedActivation) -> "QuantizedActivation":
        if a.token_scales is not None:
            return cls(values=_host(a.values), bits=a.bits, token_scales=_host(a.token_scales))
        return cls(values=_host(a.values), bits=a.bits, static_scale=a.static_scale)


def quantize_weight_groupwise(w, groups: int, bits: int) -> QuantizedMatrix:
    """quant.py:236-255"""
    return QuantizedMatrix.from_device(_dev.quantize_weight_groupwise(w, groups, bits))


def quantize_activation_tokenwise(x, bits: int) -> QuantizedActivation:
    """quant.py:258-269"""
    return QuantizedActivation.from_device(_dev.quantize_activation_tokenwise(x, bits))


def quantize_activation_static(x, calibrated_scale: float, bits: int) -> QuantizedActivation:
    """quant.py:272-281"""
    return QuantizedActivation.from_device(_dev.quantize_activation_static(x, calibrated_scale, bits))


class Calibrator(_dev.Calibrator):
    """quant.py:289-330 (extrema reduced on device)."""
