"""Caller of the hot path: ZeroQuant post-LN blocks on B200
(mirror of pkg/src/lowbit/transformer.py:26-532).

* `PrecisionConfig` / `default_group_count` / `hw_aligned` are host logic,
  identical to the reference (transformer.py:43-143).
* `quantize_block` quantizes the six weight GEMMs group-wise on device
  (transformer.py:333-361) and additionally keeps q/k/v fused into one
  [3d x d] matrix: the three reference GEMMs consume the same quantized x
  (transformer.py:470-472), so one tcgen05 GEMM with concatenated output
  channels is bit-identical to three.
* `block_forward` keeps the reference's signature and per-site activation
  dispatch (`_act_mode_for`, transformer.py:386-402); LayerNorm+quantize and
  GeLU+quantize run fused, with the residual add folded into the LN kernel.
* `EncoderEngine` is the batched, CUDA-graph-captured forward used for the
  BERT-base / GPT benchmarks (batch x seq tokens per step).

Attention (QK^T, softmax, PV) is float in the reference (transformer.py:413-440)
and stays float here (fp32); it is outside the bit-exact contract, so block
outputs are compared with a tolerance (tests/test_transformer_gpu.py).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N
from . import igemm, quant
from .errors import ShapeError, UsageError
from .igemm import DynamicAct, FullAct, StaticAct
from .quant import QuantizedMatrix, as_device_f32

GEMM_SITES = ("attn_in", "attn_proj_in", "ffc_in", "ffc_mid")
WEIGHT_NAMES = ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh")
BIAS_NAMES = ("b_q", "b_k", "b_v", "b_o", "b_h4h", "b_4hh")
MHSA_WEIGHTS = ("w_q", "w_k", "w_v", "w_o")
FFC_WEIGHTS = ("w_h4h", "w_4hh")
LN_EPS = 1e-5
INIT_STD = 0.02


class ActivationMode(Enum):
    """transformer.py:36-40"""

    FULL = "full"
    INT8 = "int8"
    INT8_ATTN_FULL = "int8_attn_full"


@dataclass(frozen=True)
class PrecisionConfig:
    """transformer.py:43-126 (verbatim semantics)."""

    mhsa_weight_bits: int | None
    ffc_weight_bits: int | None
    activation_mode: ActivationMode = ActivationMode.FULL
    activation_static: bool = False
    group_count: int = 16

    def __post_init__(self):
        for bits in (self.mhsa_weight_bits, self.ffc_weight_bits):
            if bits is not None and bits not in quant.SUPPORTED_BITS:
                raise UsageError(f"weight bits must be 4, 8 or full, got {bits}")
        if (self.mhsa_weight_bits is None) != (self.ffc_weight_bits is None):
            raise UsageError("mixed full/quantized sublayers are not supported: quantize both or neither")
        if self.activation_static and self.activation_mode is ActivationMode.FULL:
            raise UsageError("static activation quantization requires an A8-style mode")

    @property
    def quantizes_weights(self) -> bool:
        return self.mhsa_weight_bits is not None

    @classmethod
    def full(cls) -> "PrecisionConfig":
        return cls(mhsa_weight_bits=None, ffc_weight_bits=None)

    @classmethod
    def from_scheme(cls, scheme: str, group_count: int | None = None,
                    activation_static: bool = False, hidden_dim: int | None = None) -> "PrecisionConfig":
        label = scheme.strip().upper()
        if not label.startswith("W") or "A" not in label:
            raise UsageError(f"malformed scheme {scheme!r}; expected WxAy like W8A8 or W4/8A16")
        w_part, a_part = label[1:].split("A", 1)
        weight_map = {"16": (None, None), "8": (8, 8), "4/8": (8, 4)}
        act_map = {"16": ActivationMode.FULL, "8": ActivationMode.INT8, "8/16": ActivationMode.INT8_ATTN_FULL}
        if w_part not in weight_map or a_part not in act_map:
            raise UsageError(
                f"malformed scheme {scheme!r}; valid schemes: "
                "W16A16, W8A16, W8A8, W8A8/16, W4/8A16, W4/8A8, W4/8A8/16")
        mhsa, ffc = weight_map[w_part]
        mode = act_map[a_part]
        if activation_static and mode is ActivationMode.FULL:
            raise UsageError(f"scheme {scheme!r} has no activations to calibrate")
        g = group_count if group_count is not None else default_group_count(hidden_dim or 0)
        return cls(mhsa_weight_bits=mhsa, ffc_weight_bits=ffc, activation_mode=mode,
                   activation_static=activation_static, group_count=g)

    def label(self) -> str:
        w = {(None, None): "16", (8, 8): "8", (8, 4): "4/8"}[(self.mhsa_weight_bits, self.ffc_weight_bits)]
        a = {ActivationMode.FULL: "16", ActivationMode.INT8: "8", ActivationMode.INT8_ATTN_FULL: "8/16"}[
            self.activation_mode]
        return f"W{w}A{a}"


def default_group_count(hidden_dim: int) -> int:
    """transformer.py:129-137"""
    if hidden_dim >= 2048:
        return 128
    if hidden_dim >= 1024:
        return 64
    if hidden_dim >= 512:
        return 48
    return 16


def hw_aligned(rows: int, groups: int) -> bool:
    """transformer.py:140-143"""
    return all(count % 16 == 0 for _, count in quant.group_layout_for(rows, groups))


# ---------------------------------------------------------------------------
# quantized block on device
# ---------------------------------------------------------------------------


def concat_quantized(mats: list[QuantizedMatrix]) -> QuantizedMatrix:
    """Stack output channels of separately quantized matrices (same bits/cols).
    Each keeps its own groups; the result is what three separate GEMMs see."""
    bits = {m.bits for m in mats}
    cols = {m.cols for m in mats}
    if len(bits) != 1 or len(cols) != 1:
        raise UsageError("concatenated matrices must share bit width and column count")
    ld = mats[0].ld
    rows = sum(m.rows for m in mats)
    store = torch.zeros((rows, ld), dtype=torch.int8, device=mats[0].values.device)
    layout, gs, rs = [], [], []
    off = 0
    for m in mats:
        store[off: off + m.rows, : m.cols].copy_(m.values)
        layout += [(s + off, c) for s, c in m.group_layout]
        gs.append(m.group_scales)
        rs.append(m.row_scales())
        off += m.rows
    out = QuantizedMatrix(values=store[:, : mats[0].cols], bits=bits.pop(), group_scales=torch.cat(gs),
                          group_layout=layout, row_scale_vec=torch.cat(rs).contiguous())
    if out.bits == 4:
        out.packed4 = quant.pack_int4(out.values)
    return out


@dataclass
class DeviceBlock:
    """QuantizedBlock (transformer.py:182-208) resident in HBM, plus the fused
    QKV matrix.  Biases / LN parameters stay float32 (transformer.py:350-359)."""

    w_q: QuantizedMatrix
    w_k: QuantizedMatrix
    w_v: QuantizedMatrix
    w_o: QuantizedMatrix
    w_h4h: QuantizedMatrix
    w_4hh: QuantizedMatrix
    b_q: torch.Tensor
    b_k: torch.Tensor
    b_v: torch.Tensor
    b_o: torch.Tensor
    b_h4h: torch.Tensor
    b_4hh: torch.Tensor
    ln1_gamma: torch.Tensor
    ln1_beta: torch.Tensor
    ln2_gamma: torch.Tensor
    ln2_beta: torch.Tensor
    num_heads: int
    w_qkv: QuantizedMatrix | None = None
    b_qkv: torch.Tensor | None = None

    @property
    def dim(self) -> int:
        return self.w_q.rows

    def __post_init__(self):
        mhsa_bits = {getattr(self, n).bits for n in MHSA_WEIGHTS}
        ffc_bits = {getattr(self, n).bits for n in FFC_WEIGHTS}
        if len(mhsa_bits) != 1 or len(ffc_bits) != 1:
            raise UsageError("MHSA matrices must share one bit width, FFC another")
        if self.dim % self.num_heads != 0:
            raise UsageError(f"hidden dim {self.dim} not divisible by {self.num_heads} heads")
        if self.w_qkv is None:
            self.w_qkv = concat_quantized([self.w_q, self.w_k, self.w_v])
            self.b_qkv = torch.cat([self.b_q, self.b_k, self.b_v]).contiguous()


def _get(block, name):
    return block[name] if isinstance(block, dict) else getattr(block, name)


def quantize_block(block, precision: PrecisionConfig) -> DeviceBlock:
    """transformer.py:333-361: group-wise quantization of the six weight GEMMs
    with groups = min(g, rows); `block` is a BlockWeights-like object or dict of
    float32 arrays (numpy or torch)."""
    if not precision.quantizes_weights:
        raise UsageError("the B200 path runs quantized blocks; use a W8/W4 scheme")
    g = precision.group_count

    def qm(name, bits):
        w = as_device_f32(_get(block, name))
        return quant.quantize_weight_groupwise(w, min(g, w.shape[0]), bits)

    mb, fb = precision.mhsa_weight_bits, precision.ffc_weight_bits
    vec = lambda n: as_device_f32(_get(block, n)).reshape(-1).contiguous()  # noqa: E731
    return DeviceBlock(
        w_q=qm("w_q", mb), w_k=qm("w_k", mb), w_v=qm("w_v", mb), w_o=qm("w_o", mb),
        w_h4h=qm("w_h4h", fb), w_4hh=qm("w_4hh", fb),
        b_q=vec("b_q"), b_k=vec("b_k"), b_v=vec("b_v"), b_o=vec("b_o"), b_h4h=vec("b_h4h"),
        b_4hh=vec("b_4hh"), ln1_gamma=vec("ln1_gamma"), ln1_beta=vec("ln1_beta"),
        ln2_gamma=vec("ln2_gamma"), ln2_beta=vec("ln2_beta"), num_heads=int(_get(block, "num_heads")),
    )


def random_block(dim: int, num_heads: int, mhsa_bits: int, ffc_bits: int, groups: int,
                 seed: int = 0, ffn_mult: int = 4, std: float = INIT_STD) -> DeviceBlock:
    """Random-init block generated and quantized on device (Gaussian(0, 0.02)
    weights, zero biases, identity LN — transformer.py:261-297's recipe, with a
    device RNG so GPT-scale layers don't need a host round trip)."""
    gen = torch.Generator(device="cuda").manual_seed(seed)

    def w(r, c):
        return torch.randn((r, c), generator=gen, device="cuda") * std

    def qm(r, c, bits):
        return quant.quantize_weight_groupwise(w(r, c), min(groups, r), bits)

    z = lambda n: torch.zeros(n, device="cuda")  # noqa: E731
    o = lambda n: torch.ones(n, device="cuda")  # noqa: E731
    f = ffn_mult * dim
    return DeviceBlock(
        w_q=qm(dim, dim, mhsa_bits), w_k=qm(dim, dim, mhsa_bits), w_v=qm(dim, dim, mhsa_bits),
        w_o=qm(dim, dim, mhsa_bits), w_h4h=qm(f, dim, ffc_bits), w_4hh=qm(dim, f, ffc_bits),
        b_q=z(dim), b_k=z(dim), b_v=z(dim), b_o=z(dim), b_h4h=z(f), b_4hh=z(dim),
        ln1_gamma=o(dim), ln1_beta=z(dim), ln2_gamma=o(dim), ln2_beta=z(dim), num_heads=num_heads)


# ---------------------------------------------------------------------------
# forward
# ---------------------------------------------------------------------------


def _act_mode_for(precision: PrecisionConfig, site: str, layer: int, static_scales):
    """transformer.py:386-402"""
    mode = precision.activation_mode
    if mode is ActivationMode.FULL:
        return FullAct()
    if mode is ActivationMode.INT8_ATTN_FULL and site == "attn_in":
        return FullAct()
    if precision.activation_static:
        key = f"layer{layer}.{site}"
        if static_scales is None or key not in static_scales:
            raise UsageError(f"static activation quantization needs a calibrated scale for {key}")
        return StaticAct(scale=static_scales[key], bits=8)
    return DynamicAct(bits=8)


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, num_heads: int, causal: bool,
              batch: int = 1, out: torch.Tensor | None = None) -> torch.Tensor:
    """transformer.py:413-440 on device, float, for `batch` sequences packed as
    [batch*t, d] rows (each sequence attends only to itself).

    q, k, v are column views of one [T, 3d] qkv buffer (as produced by the fused
    QKV GEMM; separate tensors are packed first).  head_dim 64: the tcgen05
    kernels (fp16 two-term split for t <= 128, 3xTF32 online softmax beyond);
    other head sizes (multiples of 32 up to 256, e.g. GPT-J 256, NeoX 96): the
    CUDA-core fp32 flash-attention kernel.  Anything else raises."""
    bt, d = q.shape
    t = bt // batch
    dh = d // num_heads
    scale = float(np.float32(1.0 / math.sqrt(dh)))
    packed = (q.stride(1) == 1 and k.data_ptr() == q.data_ptr() + 4 * d
              and v.data_ptr() == q.data_ptr() + 8 * d and q.stride(0) == k.stride(0) == v.stride(0))
    if not packed:
        qkv = torch.cat([q, k, v], dim=1).contiguous()
        q = qkv[:, :d]
    ctx = out if out is not None else torch.empty((bt, d), dtype=torch.float32, device=q.device)
    N.call("zq_attention_f32", q.data_ptr(), q.stride(0), batch, t, num_heads, dh, int(causal), scale,
           ctx.data_ptr(), ctx.stride(0), N.stream_ptr())
    return ctx


def fused_qkv_attention(xq: torch.Tensor, token_scales: torch.Tensor, w: QuantizedMatrix, bias, num_heads: int,
                        causal: bool, batch: int, out: torch.Tensor) -> bool:
    """quantized_linear(x, W_qkv) then attention (transformer.py:395-440) as one
    kernel (zq_qkv_attention) for an int8 x with per-token scales: out (ctx) is
    bit-identical to zq_linear + zq_attention_f32.  False (nothing launched) when
    the shape is outside the kernel (W4 weights, head_dim != 64, seq > 128,
    d % 128 != 0); ZQ_FUSE_QKV=0 disables it."""
    if w.bits != 8 or os.environ.get("ZQ_FUSE_QKV", "1") != "1":
        return False
    t, d = xq.shape[0], w.cols
    if t % batch or d % num_heads:
        return False
    dh = d // num_heads
    wp, ldw, _ = w.weight_operand()
    scale = float(np.float32(1.0 / math.sqrt(dh)))
    rc = N.call_rc("zq_qkv_attention", xq.data_ptr(), xq.stride(0), token_scales.data_ptr(), wp, ldw,
                   w.row_scales().data_ptr(), N.ptr(bias), batch, t // batch, num_heads, dh, int(causal), scale,
                   out.data_ptr(), out.stride(0), N.stream_ptr())
    return rc == N.ZQ_OK


def _linear_site(x, w: QuantizedMatrix, bias, am, full_act: str = "exact"):
    if isinstance(am, FullAct):
        return igemm.full_linear(x, w, bias, precision=full_act)
    return igemm.quantized_linear(x, w, bias, am)


def block_forward(x, block: DeviceBlock, precision: PrecisionConfig, causal: bool, layer: int = 0,
                  static_scales: dict[str, float] | None = None, batch: int = 1,
                  full_act: str = "exact") -> torch.Tensor:
    """transformer.py:443-486: LN2(h + FFC(h)) with h = LN1(x + MHSA(x)).
    Dynamic-activation sites run the fused kernels (LN/GeLU + quantize); the
    result equals the reference up to attention's float rounding.  FullAct sites
    (A16 schemes, e.g. W8A8/16's attn_in) run igemm.full_linear with
    `full_act` precision: "exact" (bit-exact sequential f32, CUDA cores) or the
    tensor-core tolerance modes "f16" / "f16x2"."""
    xt = as_device_f32(x)
    if xt.dim() != 2 or xt.shape[1] != block.dim:
        raise ShapeError(f"block input {tuple(xt.shape)} does not match hidden dim {block.dim}")
    t, d = xt.shape

    def mode(site):
        return _act_mode_for(precision, site, layer, static_scales)

    am = mode("attn_in")
    ctx = None
    if isinstance(am, DynamicAct) and am.bits == 8 and block.w_qkv.bits == 8:
        # W8A8 dynamic: QKV projection + attention in one kernel (bit-identical)
        xq = quant.quantize_activation_tokenwise(xt, 8)
        ctx = torch.empty((t, d), dtype=torch.float32, device=xt.device)
        if not fused_qkv_attention(xq.values, xq.token_scales, block.w_qkv, block.b_qkv, block.num_heads, causal,
                                   batch, ctx):
            qkv = igemm.fused_linear(xq, block.w_qkv, block.b_qkv)
            ctx = attention(qkv[:, :d], qkv[:, d: 2 * d], qkv[:, 2 * d:], block.num_heads, causal, batch)
    if ctx is None:
        qkv = _linear_site(xt, block.w_qkv, block.b_qkv, am, full_act)
        ctx = attention(qkv[:, :d], qkv[:, d: 2 * d], qkv[:, 2 * d:], block.num_heads, causal, batch)
    attn_out = _linear_site(ctx, block.w_o, block.b_o, mode("attn_proj_in"), full_act)
    h = torch.empty_like(xt)
    m_ffc_in = mode("ffc_in")
    if isinstance(m_ffc_in, DynamicAct):
        hq = igemm.layer_norm_quantize(xt, block.ln1_gamma, block.ln1_beta, 8, LN_EPS, residual=attn_out, ln_out=h)
        u = igemm.fused_linear(hq, block.w_h4h, block.b_h4h)
    else:
        igemm.layer_norm_quantize(xt, block.ln1_gamma, block.ln1_beta, 8, LN_EPS, residual=attn_out, ln_out=h)
        u = _linear_site(h, block.w_h4h, block.b_h4h, m_ffc_in, full_act)
    m_mid = mode("ffc_mid")
    if isinstance(m_mid, DynamicAct):
        zq = igemm.gelu_quantize(u, 8)
        f = igemm.fused_linear(zq, block.w_4hh, block.b_4hh)
    else:
        z = torch.empty_like(u)
        igemm.gelu_quantize(u, 8, gelu_out=z)
        f = _linear_site(z, block.w_4hh, block.b_4hh, m_mid, full_act)
    y = torch.empty_like(xt)
    igemm.layer_norm_quantize(h, block.ln2_gamma, block.ln2_beta, 8, LN_EPS, residual=f, ln_out=y)
    return y


def _matmul_seq(x: torch.Tensor, w: torch.Tensor, bias: torch.Tensor | None) -> torch.Tensor:
    """tensor.matmul(x, w.T) (+= bias), transformer.py:405-410, order-exact."""
    m, k = x.shape
    n = w.shape[0]
    out = torch.empty((m, n), dtype=torch.float32, device=x.device)
    N.call("zq_matmul_f32_seq", x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), N.ptr(bias), m, n, k,
           out.data_ptr(), out.stride(0), N.stream_ptr())
    return out


def float_block_forward(x: torch.Tensor, w: dict, num_heads: int, causal: bool, layer: int = 0,
                        tap=None) -> torch.Tensor:
    """transformer.py:443-486 with float weights (PrecisionConfig.full()): the
    calibration forward, bit-identical to the reference's numpy arithmetic
    (csrc/zq_calib.cu: sequential f32 matmuls, the exact float attention with
    numpy's exp and pairwise softmax sum; the exact LN / GeLU kernels' f32
    outputs).  `x` is one sequence [t, d]; `w` holds float32 device tensors
    (w_q .. ln2_beta); `tap(site, layer, x)` sees the float tensor entering
    each weight GEMM."""
    t, d = x.shape
    dh = d // num_heads
    if tap is not None:
        tap("attn_in", layer, x)
    qkv = torch.empty((t, 3 * d), dtype=torch.float32, device=x.device)
    for i, (wn, bn) in enumerate((("w_q", "b_q"), ("w_k", "b_k"), ("w_v", "b_v"))):
        qkv[:, i * d:(i + 1) * d] = _matmul_seq(x, w[wn], w[bn])
    ctx = torch.empty((t, d), dtype=torch.float32, device=x.device)
    scratch = torch.empty(num_heads * t * t, dtype=torch.float32, device=x.device)
    N.call("zq_attention_exact_f32", qkv.data_ptr(), qkv.stride(0), t, num_heads, dh, int(causal),
           float(np.float32(1.0 / math.sqrt(dh))), scratch.data_ptr(), ctx.data_ptr(), ctx.stride(0),
           N.stream_ptr())
    if tap is not None:
        tap("attn_proj_in", layer, ctx)
    attn_out = _matmul_seq(ctx, w["w_o"], w["b_o"])
    h = torch.empty_like(x)
    igemm.layer_norm_quantize(x, w["ln1_gamma"], w["ln1_beta"], 8, LN_EPS, residual=attn_out, ln_out=h,
                              check_finite=False)
    if tap is not None:
        tap("ffc_in", layer, h)
    u = _matmul_seq(h, w["w_h4h"], w["b_h4h"])
    z = torch.empty_like(u)
    igemm.gelu_quantize(u, 8, gelu_out=z, check_finite=False)
    if tap is not None:
        tap("ffc_mid", layer, z)
    f = _matmul_seq(z, w["w_4hh"], w["b_4hh"])
    y = torch.empty_like(x)
    igemm.layer_norm_quantize(h, w["ln2_gamma"], w["ln2_beta"], 8, LN_EPS, residual=f, ln_out=y,
                              check_finite=False)
    return y


@dataclass
class SiteCalibration:
    """evaluate.py:159-163"""

    x_max: float
    x_min: float
    scale: float


def _calibrators(momentum: float):
    cals: dict[str, quant.Calibrator] = {}

    def tap(site, layer, x):
        key = f"layer{layer}.{site}"
        if key not in cals:
            cals[key] = quant.Calibrator(momentum=momentum)
        cals[key].observe(x)

    return cals, tap


def calibrate_model(embedding, float_blocks: list[dict], num_heads: int, causal: bool, batches,
                    momentum: float = 0.95, bits: int = 8) -> dict[str, SiteCalibration]:
    """evaluate.calibrate_model (evaluate.py:168-196) on device: every batch (a
    1-d token-id sequence, consumed in order) runs embed -> the float blocks
    (model_forward with PrecisionConfig.full(), transformer.py:489-532) with one
    momentum Calibrator per GEMM-input site "layer{L}.{site}" (quant.py:289-330).
    The float forward is order-exact, so x_max / x_min / scale are
    bit-identical to the reference's."""
    cals, tap = _calibrators(momentum)
    emb = as_device_f32(embedding)
    dev_blocks = [{k: as_device_f32(v) for k, v in b.items() if k != "num_heads"} for b in float_blocks]
    n = 0
    for ids in batches:
        ids_t = torch.as_tensor(np.asarray(ids, dtype=np.int64)).reshape(-1)
        if ids_t.numel() == 0:
            raise UsageError("empty token sequence")
        if int(ids_t.min()) < 0 or int(ids_t.max()) >= emb.shape[0]:
            raise UsageError(f"token id out of range [0, {emb.shape[0]})")
        x = emb.index_select(0, ids_t.to(emb.device))
        for li, w in enumerate(dev_blocks):
            x = float_block_forward(x, w, num_heads, causal, li, tap)
        n += 1
    if n == 0:
        raise UsageError("calibration needs at least one batch")
    return {k: SiteCalibration(c.x_max, c.x_min, c.finalize(bits)) for k, c in sorted(cals.items())}


def static_scales_from(calibration: dict[str, SiteCalibration]) -> dict[str, float]:
    """evaluate.py:199-200"""
    return {k: sc.scale for k, sc in calibration.items()}


def calibrate_static_scales(float_blocks: list[dict], batches, num_heads: int, causal: bool,
                            momentum: float = 0.95, bits: int = 8) -> dict[str, float]:
    """Calibration from block-0 inputs: every batch (float32 [tokens, d], one
    sequence) runs through the float blocks (the order-exact forward above)
    with one Calibrator per site; returns the finalized static scales for
    `block_forward(..., static_scales=...)` under activation_static=True."""
    cals, tap = _calibrators(momentum)
    dev_blocks = [{k: as_device_f32(v) for k, v in b.items() if k != "num_heads"} for b in float_blocks]
    n = 0
    for xb in batches:
        x = as_device_f32(xb)
        for li, w in enumerate(dev_blocks):
            x = float_block_forward(x, w, num_heads, causal, li, tap)
        n += 1
    if n == 0:
        raise UsageError("calibration needs at least one batch")
    return {k: c.finalize(bits) for k, c in sorted(cals.items())}


# ---------------------------------------------------------------------------
# Batched encoder / decoder-prefill engine (the benchmark caller)
# ---------------------------------------------------------------------------


@dataclass
class EncoderEngine:
    """Embedding -> L ZeroQuant blocks (W8A8 / W4/8A8, dynamic token-wise
    activations) -> final LN, for `batch` sequences of `seq` tokens.

    All intermediates are preallocated; `forward()` is a fixed launch sequence
    that is captured once into a CUDA graph.  Per block:
      QKV GEMM -> attention -> ctx quantize -> O GEMM -> (x+attn) LN1+quant ->
      h4h GEMM -> GeLU+quant -> 4hh GEMM -> (h+f) LN2+quant (next block's input).
    """

    blocks: list[DeviceBlock]
    embedding: torch.Tensor        # [V, d] float32
    final_gamma: torch.Tensor
    final_beta: torch.Tensor
    batch: int
    seq: int
    causal: bool = False
    use_graph: bool = True
    lanes: int = 1
    _bufs: dict = field(default_factory=dict, init=False)
    _graph: object = field(default=None, init=False)
    _sub: list = field(default_factory=list, init=False)
    _streams: list = field(default_factory=list, init=False)
    _hot: object = field(default=None, init=False)

    def __post_init__(self):
        if self.lanes > 1:
            # `lanes` independent sub-batches on their own streams: the kernels of
            # one lane fill the SMs the other lane's latency-bound phases leave idle
            if self.batch % self.lanes:
                raise UsageError(f"batch {self.batch} not divisible into {self.lanes} lanes")
            d = self.embedding.shape[1]
            sb = self.batch // self.lanes
            dev = self.embedding.device
            self._bufs = dict(ids=torch.zeros(self.tokens, dtype=torch.int64, device=dev),
                              out=torch.empty((self.tokens, d), dtype=torch.float32, device=dev),
                              flag=torch.zeros(1, dtype=torch.int32, device=dev))
            for i in range(self.lanes):
                sub = EncoderEngine(blocks=self.blocks, embedding=self.embedding, final_gamma=self.final_gamma,
                                    final_beta=self.final_beta, batch=sb, seq=self.seq, causal=self.causal,
                                    use_graph=False)
                r0, r1 = i * sb * self.seq, (i + 1) * sb * self.seq
                sub._bufs["ids"] = self._bufs["ids"][r0:r1]
                sub._bufs["out"] = self._bufs["out"][r0:r1]
                sub._bufs["flag"] = self._bufs["flag"]
                self._sub.append(sub)
                self._streams.append(torch.cuda.Stream())
            return
        d = self.embedding.shape[1]
        t = self.batch * self.seq
        f = self.blocks[0].w_h4h.rows
        dev = self.embedding.device
        e = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
        # the [t, d] f32 activations each kernel hands to the next (attn, f, ctx,
        # h, x) share one pool kept L2-resident (zq_l2_persist, 63 MB at BERT-base
        # batch 32); the streamed ones (qkv, u: read once) stay outside it.
        # Adding the int8 operands (72 MB) starved the rest of L2: 6% slower
        self._hot = e(5, t, d)  # attn, f, ctx, h, x
        self._bufs = dict(
            ids=torch.zeros(t, dtype=torch.int64, device=dev),
            attn=self._hot[0], f=self._hot[1], ctx=self._hot[2], h=self._hot[3], x=self._hot[4],
            qkv=e(t, 3 * d), u=e(t, f), out=e(t, d),
            xq=quant.padded_int8(t, d), cq=quant.padded_int8(t, d), hq=quant.padded_int8(t, d),
            zq=quant.padded_int8(t, f), sx=e(t), sc=e(t), sh=e(t), sz=e(t),
            flag=torch.zeros(1, dtype=torch.int32, device=dev),
            # fused linear + LN exchange workspaces (one per call site, zeroed once)
            ws_o=torch.zeros(4 * ((t + 255) // 256) + 16 + 12 * t * 64, dtype=torch.uint8, device=dev),
            ws_f=torch.zeros(4 * ((t + 255) // 256) + 16 + 12 * t * 64, dtype=torch.uint8, device=dev),
        )
        # fused linear + LN measured slower than linear then LN at BERT shapes (the
        # LN work runs on the GEMM's 8 epilogue warps per SM instead of a full-occupancy
        # row kernel): opt-in with ZQ_FUSE_LN=1
        self._fuse_ln = os.environ.get("ZQ_FUSE_LN", "0") == "1"
        # QKV GEMM + attention in one kernel (zq_qkv_attention): the [t, 3d] f32
        # QKV activation stays in the SM; ZQ_FUSE_QKV=0 runs the two kernels
        self._fuse_qkv = os.environ.get("ZQ_FUSE_QKV", "1") == "1"

    @property
    def tokens(self) -> int:
        return self.batch * self.seq

    # -- raw launches (no allocation, no host sync) --------------------------
    def _linear(self, q, s, w: QuantizedMatrix, bias, out):
        t, k = q.shape
        wp, ldw, wb = w.weight_operand()
        N.call("zq_linear", q.data_ptr(), q.stride(0), s.data_ptr(), 0.0, wp, ldw, wb,
               w.row_scales().data_ptr(), bias.data_ptr(), t, w.rows, k, out.data_ptr(), out.stride(0),
               N.OUT_F32, N.stream_ptr())

    def _linear_ln(self, q, s, w: QuantizedMatrix, bias, res, g, b, ln_out, qo, so, ws) -> bool:
        """linear + residual + LN + quantize in one kernel (zq_linear_ln_quantize);
        False when the shape is not fusable (the caller runs the two kernels)."""
        if not self._fuse_ln:
            return False
        t, k = q.shape
        wp, ldw, wb = w.weight_operand()
        rc = N.load().zq_linear_ln_quantize(
            q.data_ptr(), q.stride(0), s.data_ptr(), wp, ldw, wb, w.row_scales().data_ptr(), bias.data_ptr(), t,
            w.rows, k, res.data_ptr(), g.data_ptr(), b.data_ptr(), float(np.float32(LN_EPS)), 8, ln_out.data_ptr(),
            qo.data_ptr(), qo.stride(0), so.data_ptr(), ws.data_ptr(), ws.numel(), self._bufs["flag"].data_ptr(),
            N.stream_ptr())
        if rc == N.ZQ_ERR_UNSUPPORTED:
            self._fuse_ln = False
            return False
        N.check(rc)
        return True

    def _qkv_attention(self, q, s, blk: DeviceBlock, ctx) -> bool:
        """QKV linear + attention fused (zq_qkv_attention, bit-identical to the
        two kernels); False when the shape is not fusable."""
        if not self._fuse_qkv:
            return False
        if not fused_qkv_attention(q, s, blk.w_qkv, blk.b_qkv, blk.num_heads, self.causal, self.batch, ctx):
            self._fuse_qkv = False
            return False
        return True

    def _ln_quant(self, x, res, g, b, ln_out, q, s):
        t, d = x.shape
        N.call("zq_layer_norm_quantize", x.data_ptr(), N.ptr(res), g.data_ptr(), b.data_ptr(), t, d,
               float(np.float32(LN_EPS)), 8, ln_out.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(),
               self._bufs["flag"].data_ptr(), N.stream_ptr())

    def _tok_quant(self, x, q, s):
        t, d = x.shape
        N.call("zq_quantize_tokenwise", x.data_ptr(), t, d, d, 8, q.data_ptr(), q.stride(0), s.data_ptr(),
               self._bufs["flag"].data_ptr(), N.stream_ptr())

    def _gelu_quant(self, u, q, s):
        t, f = u.shape
        N.call("zq_gelu_quantize", u.data_ptr(), t, f, f, 8, None, q.data_ptr(), q.stride(0), s.data_ptr(),
               self._bufs["flag"].data_ptr(), N.stream_ptr())

    def _run(self):
        if self._sub:
            main = torch.cuda.current_stream()
            for sub, st in zip(self._sub, self._streams):
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    sub._run()
            for st in self._streams:
                main.wait_stream(st)
            return
        B = self._bufs
        d = self.embedding.shape[1]
        torch.index_select(self.embedding, 0, B["ids"], out=B["x"])
        self._tok_quant(B["x"], B["xq"], B["sx"])
        x, xq, sx = B["x"], B["xq"], B["sx"]
        for blk in self.blocks:
            if not self._qkv_attention(xq, sx, blk, B["ctx"]):
                self._linear(xq, sx, blk.w_qkv, blk.b_qkv, B["qkv"])
                qkv = B["qkv"]
                attention(qkv[:, :d], qkv[:, d: 2 * d], qkv[:, 2 * d:], blk.num_heads, self.causal,
                          self.batch, out=B["ctx"])
            self._tok_quant(B["ctx"], B["cq"], B["sc"])
            # h = LN1(x + O-proj) and its quantization, fused into the O GEMM when possible
            if not self._linear_ln(B["cq"], B["sc"], blk.w_o, blk.b_o, x, blk.ln1_gamma, blk.ln1_beta, B["h"],
                                   B["hq"], B["sh"], B["ws_o"]):
                self._linear(B["cq"], B["sc"], blk.w_o, blk.b_o, B["attn"])
                self._ln_quant(x, B["attn"], blk.ln1_gamma, blk.ln1_beta, B["h"], B["hq"], B["sh"])
            self._linear(B["hq"], B["sh"], blk.w_h4h, blk.b_h4h, B["u"])
            self._gelu_quant(B["u"], B["zq"], B["sz"])
            # y = LN2(h + f) is the next block's input; its quantization is fused
            if not self._linear_ln(B["zq"], B["sz"], blk.w_4hh, blk.b_4hh, B["h"], blk.ln2_gamma, blk.ln2_beta, x,
                                   xq, sx, B["ws_f"]):
                self._linear(B["zq"], B["sz"], blk.w_4hh, blk.b_4hh, B["f"])
                self._ln_quant(B["h"], B["f"], blk.ln2_gamma, blk.ln2_beta, x, xq, sx)
        self._ln_quant(x, None, self.final_gamma, self.final_beta, B["out"], B["cq"], B["sc"])

    def capture(self):
        """Warm up and capture the whole forward into one CUDA graph."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                self._run()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        if self._hot is not None and os.environ.get("ZQ_L2_PERSIST", "1") == "1":
            # access-policy window on the capture stream: every captured kernel node
            # keeps the hot activation pool L2-resident (set outside the capture)
            k = int(os.environ.get("ZQ_L2_HOT", "5"))  # leading pool tensors in the window
            N.call("zq_l2_persist", cs.cuda_stream, self._hot.data_ptr(), self._hot[0].numel() * 4 * k, None)
        with torch.cuda.graph(g, stream=cs):
            self._run()
        self._graph = g
        return g

    def launch(self):
        """Enqueue one forward on the current stream (ids already in _bufs['ids'])."""
        if self.use_graph:
            if self._graph is None:
                self.capture()
            self._graph.replay()
        else:
            self._run()

    def forward(self, token_ids) -> torch.Tensor:
        """token ids [batch, seq] (host or device) -> final hidden [batch*seq, d]
        on device.  Raises ValueError if any activation went non-finite."""
        ids = token_ids if isinstance(token_ids, torch.Tensor) else torch.as_tensor(np.asarray(token_ids))
        if tuple(ids.shape) != (self.batch, self.seq):
            raise ShapeError(f"expected token ids of shape {(self.batch, self.seq)}, got {tuple(ids.shape)}")
        self._bufs["ids"].copy_(ids.reshape(-1), non_blocking=True)
        self._bufs["flag"].zero_()
        self.launch()
        return self._bufs["out"]

    def check_finite(self):
        if int(self._bufs["flag"].item()) != 0:
            raise ValueError("non-finite activations encountered in the forward")
