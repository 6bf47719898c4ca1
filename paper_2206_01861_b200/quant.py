"""Drop-in mirror of `lowbit.quant` (pkg/src/lowbit/quant.py) on B200.

Same names, argument meaning and error behaviour as the reference; tensors live
in HBM (torch CUDA tensors; numpy inputs are uploaded) and every quantization
runs in the sm_100a kernels of libzq_b200.so.  Results are bit-identical to the
reference on identical float32 inputs.

Device layout additions (not in the reference, needed by the tensor-core path):
* int8 payloads are views into row-padded storage (row stride a multiple of 16
  for activations, 32 for weights) whose padding is zero, so TMA tiles and MMA
  K-steps can run past the logical width;
* `QuantizedMatrix` keeps the expanded per-row scale vector on device
  (the reference rebuilds it with a Python loop on every epilogue,
  quant.py:165-170) and, for 4-bit weights, the packed INT4 payload.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .errors import UsageError

SUPPORTED_BITS = (4, 8)
F32 = np.float32


def qmax(bits: int) -> int:
    """quant.py:26-28"""
    return (1 << (bits - 1)) - 1


def _check_bits(bits: int) -> None:
    """quant.py:31-33"""
    if bits not in SUPPORTED_BITS:
        raise UsageError(f"unsupported bit width {bits}, expected one of {SUPPORTED_BITS}")


class Granularity(Enum):
    """quant.py:41-44"""

    PER_TENSOR = "per_tensor"
    PER_GROUP = "per_group"
    PER_TOKEN = "per_token"


class Mode(Enum):
    """quant.py:47-49"""

    DYNAMIC = "dynamic"
    STATIC = "static"


@dataclass(frozen=True)
class QuantSpec:
    """quant.py:52-72 (host-side validation only)."""

    bits: int
    granularity: Granularity = Granularity.PER_TENSOR
    mode: Mode = Mode.DYNAMIC
    group_count: int = 1
    for_weights: bool = True

    def __post_init__(self):
        _check_bits(self.bits)
        if self.granularity is Granularity.PER_GROUP:
            if not self.for_weights:
                raise UsageError("per-group quantization is only valid for weights")
            if self.group_count < 1:
                raise UsageError(f"group count must be >= 1, got {self.group_count}")
        if self.granularity is Granularity.PER_TOKEN and self.for_weights:
            raise UsageError("per-token quantization is only valid for activations")
        if self.mode is Mode.STATIC and self.granularity is not Granularity.PER_TENSOR:
            raise UsageError("static mode uses a single calibrated per-tensor scale")


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def as_device_f32(x) -> torch.Tensor:
    """Accept numpy / torch input; return a contiguous float32 CUDA tensor.

    The reference coerces its inputs with `as_f32` (tensor.py:24-29: a numpy
    float32 cast, round-to-nearest) before quantizing weights and activations
    (quant.py:242, :261, :279); float64 input is cast the same way here."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=F32))
    if t.device.type != "cuda":
        t = t.to(_device(), non_blocking=False)
    if t.dtype != torch.float32:
        t = t.float()
    return t.contiguous()


def _as_device_f64_or_f32(x) -> torch.Tensor:
    """compute_scale / quantize_array read their input as float64 without an
    f32 round trip (quant.py:90-93, :106-112): float32 input stays float32 (the
    f64 widening is exact), anything else is widened to float64 on device."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        a = np.asarray(x)
        t = torch.from_numpy(np.ascontiguousarray(a if a.dtype in (np.float32, np.float64) else
                                                  a.astype(np.float64)))
    if t.device.type != "cuda":
        t = t.to(_device(), non_blocking=False)
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    return t.contiguous()


def round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def padded_int8(rows: int, cols: int, align: int = 16) -> torch.Tensor:
    """[rows, cols] int8 view of zero-padded storage with an `align`-multiple stride."""
    ld = max(align, round_up(cols, align))
    return torch.empty((rows, ld), dtype=torch.int8, device=_device())[:, :cols]


class FiniteFlag:
    """Device-side non-finite detector (one int32).  `check()` syncs and raises
    ValueError like the reference's eager np.isfinite checks."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=_device())

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def check(self, what: str) -> None:
        if int(self.t.item()) != 0:
            raise ValueError(f"cannot quantize non-finite {what}")

    def reset(self) -> None:
        self.t.zero_()


# ---------------------------------------------------------------------------
# Scalar / array primitives (quant.py:80-126)
# ---------------------------------------------------------------------------


def compute_scale(values, bits: int) -> float:
    """quant.py:80-95: f32(max|x| / qmax); 1.0 for an all-zero slice.  The max
    runs on device over the input's own precision (float64 stays float64)."""
    _check_bits(bits)
    v = _as_device_f64_or_f32(values).reshape(1, -1)
    if v.numel() == 0:
        raise UsageError("compute_scale called on an empty slice")
    flag = FiniteFlag()
    if v.dtype == torch.float64:
        amax = torch.empty(1, dtype=torch.float64, device=v.device)
        N.call("zq_row_absmax_f64", v.data_ptr(), 1, v.shape[1], v.shape[1], amax.data_ptr(), flag.ptr,
               N.stream_ptr())
    else:
        amax = torch.empty(1, dtype=torch.float32, device=v.device)
        N.call("zq_row_absmax", v.data_ptr(), 1, v.shape[1], v.shape[1], amax.data_ptr(), flag.ptr,
               N.stream_ptr())
    if int(flag.t.item()) != 0:
        raise ValueError("compute_scale called on non-finite values")
    m = float(amax.item())
    if m == 0.0:
        return 1.0
    return float(F32(m / qmax(bits)))


def quantize_array(x, scale: float, bits: int) -> torch.Tensor:
    """quant.py:103-113: RHAFZ(f64(x) / scale), clamped.  Returns int8 (same shape)."""
    _check_bits(bits)
    if not scale > 0:
        raise UsageError(f"quantization scale must be > 0, got {scale}")
    xt = _as_device_f64_or_f32(x)
    shape = xt.shape
    flag = FiniteFlag()
    if xt.dtype == torch.float64:
        out = torch.empty(shape, dtype=torch.int8, device=xt.device)
        N.call("zq_quantize_array_f64", xt.data_ptr(), xt.numel(), float(scale), bits, out.data_ptr(), flag.ptr,
               N.stream_ptr())
        flag.check("values")
        return out
    x2 = xt.reshape(1, -1) if xt.dim() != 2 else xt
    rows, cols = x2.shape
    out = padded_int8(rows, cols)
    if x2.numel():
        N.call("zq_quantize_static", x2.data_ptr(), rows, cols, cols, float(scale), bits,
               out.data_ptr(), out.stride(0), flag.ptr, N.stream_ptr())
        flag.check("values")
    return out.reshape(shape) if xt.dim() != 2 else out


def quantize_value(x: float, scale: float, bits: int) -> int:
    """quant.py:116-118 (a Python float is a float64, as in the reference)."""
    return int(quantize_array(np.asarray([x]), scale, bits)[0].item())


def dequantize_array(q, scale: float) -> torch.Tensor:
    """quant.py:121-122 (reference / FullAct utility; never on the fused path)."""
    qt = q if isinstance(q, torch.Tensor) else torch.as_tensor(np.asarray(q))
    return qt.to(_device()).float() * torch.tensor(F32(scale), device=_device())


def dequantize_value(q: int, scale: float) -> float:
    """quant.py:125-126"""
    return float(F32(F32(q) * F32(scale)))


# ---------------------------------------------------------------------------
# Containers (quant.py:134-208)
# ---------------------------------------------------------------------------


@dataclass
class QuantizedMatrix:
    """quant.py:134-181.  `values` is int8 [rows, cols] (a view into 32-byte
    padded storage); INT4 payloads keep one value per byte in `values` (as the
    reference does) plus the packed nibbles in `packed4` for the W4A8 kernel."""

    values: torch.Tensor
    bits: int
    group_scales: torch.Tensor  # float32 [g] on device
    group_layout: list[tuple[int, int]]
    row_scale_vec: torch.Tensor | None = None  # float32 [rows] on device
    packed4: torch.Tensor | None = None         # uint8 [rows, ld/2]

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def cols(self) -> int:
        return self.values.shape[1]

    @property
    def num_groups(self) -> int:
        return len(self.group_layout)

    @property
    def ld(self) -> int:
        return self.values.stride(0)

    def logical_bits(self) -> int:
        """quant.py:161-163"""
        return self.rows * self.cols * self.bits + 32 * self.num_groups

    def row_scales(self) -> torch.Tensor:
        """quant.py:165-170 (cached on device)."""
        if self.row_scale_vec is None:
            gs = self.group_scales.to(_device())
            counts = torch.tensor([c for _, c in self.group_layout], device=gs.device)
            self.row_scale_vec = torch.repeat_interleave(gs, counts).contiguous()
        return self.row_scale_vec

    def dequantize(self) -> torch.Tensor:
        """quant.py:172-174 (reference / Full path only)."""
        return self.values.float() * self.row_scales()[:, None]

    def group_of_row(self, row: int) -> int:
        """quant.py:176-180"""
        for gi, (start, count) in enumerate(self.group_layout):
            if start <= row < start + count:
                return gi
        raise UsageError(f"row {row} outside group layout of {self.rows} rows")

    def weight_operand(self) -> tuple[int, int, int]:
        """(device pointer, row stride in elements, bits) for the GEMM kernels."""
        if self.bits == 4:
            if self.packed4 is None:
                self.packed4 = pack_int4(self.values)
            return self.packed4.data_ptr(), self.ld, 4
        return self.values.data_ptr(), self.ld, 8


@dataclass
class QuantizedActivation:
    """quant.py:183-208: int8 payload with per-token scales XOR one static scale."""

    values: torch.Tensor
    bits: int
    token_scales: torch.Tensor | None = None
    static_scale: float | None = None

    def __post_init__(self):
        if (self.token_scales is None) == (self.static_scale is None):
            raise UsageError("exactly one of token_scales / static_scale must be populated")

    @property
    def tokens(self) -> int:
        return self.values.shape[0]

    def scales_per_token(self) -> torch.Tensor:
        if self.token_scales is not None:
            return self.token_scales
        return torch.full((self.tokens,), float(F32(self.static_scale)), dtype=torch.float32,
                          device=self.values.device)

    def dequantize(self) -> torch.Tensor:
        return self.values.float() * self.scales_per_token()[:, None]

    def gemm_operand(self) -> torch.Tensor:
        """int8 payload with a 16-byte-multiple row stride (copy only if needed)."""
        v = self.values
        if v.stride(1) == 1 and v.stride(0) % 16 == 0 and v.data_ptr() % 16 == 0:
            return v
        ld = max(16, round_up(v.shape[1], 16))
        store = torch.zeros((v.shape[0], ld), dtype=torch.int8, device=v.device)
        store[:, : v.shape[1]].copy_(v)
        return store[:, : v.shape[1]]


def group_layout_for(rows: int, groups: int) -> list[tuple[int, int]]:
    """quant.py:211-219"""
    if groups < 1 or groups > rows:
        raise UsageError(f"group count {groups} invalid for {rows} rows")
    base = rows // groups
    layout = [(g * base, base) for g in range(groups)]
    start, count = layout[-1]
    layout[-1] = (start, count + rows - groups * base)
    return layout


def pack_int4(values: torch.Tensor) -> torch.Tensor:
    """Packed two's-complement nibbles (element 2k low nibble of byte k)."""
    rows = values.shape[0]
    ld = values.stride(0)
    if ld % 32:
        raise UsageError("int4 packing needs a 32-byte multiple row stride")
    out = torch.empty((rows, ld // 2), dtype=torch.uint8, device=values.device)
    N.call("zq_pack_int4", values.data_ptr(), rows, ld, out.data_ptr(), N.stream_ptr())
    return out


def quantize_weight_groupwise(w, groups: int, bits: int) -> QuantizedMatrix:
    """quant.py:236-255, on device.  groups == 1 is per-tensor quantization."""
    _check_bits(bits)
    wt = as_device_f32(w)
    if wt.dim() != 2:
        raise UsageError(f"weight matrix must be 2-d, got shape {tuple(wt.shape)}")
    rows, cols = wt.shape
    layout = group_layout_for(rows, groups)
    values = padded_int8(rows, cols, align=32)
    gs = torch.empty(groups, dtype=torch.float32, device=wt.device)
    rs = torch.empty(rows, dtype=torch.float32, device=wt.device)
    packed = None
    if bits == 4:
        packed = torch.empty((rows, values.stride(0) // 2), dtype=torch.uint8, device=wt.device)
    flag = FiniteFlag()
    N.call("zq_quantize_weight_groupwise", wt.data_ptr(), rows, cols, groups, bits,
           values.data_ptr(), values.stride(0), gs.data_ptr(), rs.data_ptr(),
           N.ptr(packed), flag.ptr, N.stream_ptr())
    if int(flag.t.item()) != 0:
        raise ValueError("cannot quantize non-finite weights")
    return QuantizedMatrix(values=values, bits=bits, group_scales=gs, group_layout=layout,
                           row_scale_vec=rs, packed4=packed)


def quantize_activation_tokenwise(x, bits: int, *, check_finite: bool = True,
                                  flag: FiniteFlag | None = None) -> QuantizedActivation:
    """quant.py:258-269: one scale per token row, computed on the fly (K1)."""
    _check_bits(bits)
    xt = as_device_f32(x)
    if xt.dim() != 2 or xt.shape[0] < 1:
        raise UsageError(f"activations must be (tokens x dim), got shape {tuple(xt.shape)}")
    rows, cols = xt.shape
    if cols == 0:
        raise ValueError("zero-size array to reduction operation maximum which has no identity")
    q = padded_int8(rows, cols)
    s = torch.empty(rows, dtype=torch.float32, device=xt.device)
    fl = flag or FiniteFlag()
    N.call("zq_quantize_tokenwise", xt.data_ptr(), rows, cols, cols, bits, q.data_ptr(),
           q.stride(0), s.data_ptr(), fl.ptr, N.stream_ptr())
    if check_finite:
        fl.check("activations")
    return QuantizedActivation(values=q, bits=bits, token_scales=s)


def quantize_activation_static(x, calibrated_scale: float, bits: int, *,
                               check_finite: bool = True) -> QuantizedActivation:
    """quant.py:272-281: one calibrated scale; out-of-range values clamp (K2)."""
    _check_bits(bits)
    if not calibrated_scale > 0:
        raise UsageError(f"calibrated scale must be > 0, got {calibrated_scale}")
    xt = as_device_f32(x)
    if xt.dim() != 2:
        raise UsageError(f"activations must be (tokens x dim), got shape {tuple(xt.shape)}")
    rows, cols = xt.shape
    q = padded_int8(rows, cols)
    flag = FiniteFlag()
    N.call("zq_quantize_static", xt.data_ptr(), rows, cols, cols, float(calibrated_scale), bits,
           q.data_ptr(), q.stride(0), flag.ptr, N.stream_ptr())
    if check_finite:
        flag.check("values")
    return QuantizedActivation(values=q, bits=bits, static_scale=float(calibrated_scale))


@dataclass
class Calibrator:
    """quant.py:289-330: momentum min/max tracker (extrema reduced on device)."""

    momentum: float = 0.95
    x_max: float = field(default=0.0, init=False)
    x_min: float = field(default=0.0, init=False)
    observed_batches: int = field(default=0, init=False)

    def __post_init__(self):
        if not 0.0 < self.momentum < 1.0:
            raise UsageError(f"momentum must be in (0, 1), got {self.momentum}")

    def observe(self, x) -> None:
        """quant.py:305-317: batch max / min reduced on device (zq_minmax_f32)."""
        xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        xt = xt.to(_device()).contiguous()
        if xt.dtype != torch.float32:  # the reference reduces the input's own dtype
            xt = xt.double()
            if not bool(torch.isfinite(xt).all()):
                raise ValueError("calibrator observed non-finite values")
            hm = torch.stack([xt.max(), xt.min()]).cpu()
        else:
            mm = torch.empty(2, dtype=torch.float32, device=xt.device)
            flag = FiniteFlag()
            N.call("zq_minmax_f32", xt.data_ptr(), xt.numel(), mm.data_ptr(), flag.ptr, N.stream_ptr())
            hm = mm.cpu()
            if int(flag.t.item()) != 0:
                raise ValueError("calibrator observed non-finite values")
        bmax = float(hm[0])
        bmin = float(hm[1])
        if self.observed_batches == 0:
            self.x_max, self.x_min = bmax, bmin
        else:
            m = self.momentum
            self.x_max = m * self.x_max + (1.0 - m) * bmax
            self.x_min = m * self.x_min + (1.0 - m) * bmin
        self.observed_batches += 1

    def finalize(self, bits: int) -> float:
        _check_bits(bits)
        if self.observed_batches == 0:
            raise UsageError("calibrator finalized before any observation")
        reach = max(abs(self.x_max), abs(self.x_min))
        if reach == 0.0:
            return 1.0
        return float(F32(reach / qmax(bits)))
