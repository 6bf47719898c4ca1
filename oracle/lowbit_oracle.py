"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

Every function cites the reference line it restates (paths relative to
`/root/reference/`).  Nothing in the product package imports this module; it
is the checker for the CUDA path (tests, smoke, bench cpu_baseline).

Conventions follow the reference exactly:
* activations / weights are float32, int payloads int8, scales float32;
* division for quantization happens in float64 and ties round half away from
  zero (pkg/src/lowbit/quant.py:98-113, :229-233);
* float32 reductions use numpy's pairwise summation; `pairwise_sum_f32` below
  restates that order explicitly so the GPU kernel can be checked against a
  written-down algorithm, not just against numpy.
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
INT32_LIMIT = 1 << 31
SUPPORTED_BITS = (4, 8)
LN_EPS = 1e-5
_INV_SQRT2 = 1.0 / math.sqrt(2.0)


class ShapeError(ValueError):
    """pkg/src/lowbit/errors.py:8"""


class UsageError(ValueError):
    """pkg/src/lowbit/errors.py:12"""


# ---------------------------------------------------------------------------
# quant.py
# ---------------------------------------------------------------------------


def qmax(bits: int) -> int:
    """pkg/src/lowbit/quant.py:26-28"""
    return (1 << (bits - 1)) - 1


def check_bits(bits: int) -> None:
    """pkg/src/lowbit/quant.py:31-33"""
    if bits not in SUPPORTED_BITS:
        raise UsageError(f"unsupported bit width {bits}")


def compute_scale(values, bits: int) -> float:
    """pkg/src/lowbit/quant.py:80-95: f32(max|x| (f64) / qmax); 0 -> 1.0."""
    check_bits(bits)
    v = np.asarray(values)
    if v.size == 0:
        raise UsageError("compute_scale called on an empty slice")
    if not np.all(np.isfinite(v)):
        raise ValueError("compute_scale called on non-finite values")
    m = float(np.max(np.abs(v.astype(np.float64))))
    if m == 0.0:
        return 1.0
    return float(F32(m / qmax(bits)))


def round_half_away(v: np.ndarray) -> np.ndarray:
    """pkg/src/lowbit/quant.py:98-100"""
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


def quantize_array(x, scale: float, bits: int) -> np.ndarray:
    """pkg/src/lowbit/quant.py:103-113: RHAFZ(x64 / f64(scale)), clip to +-qmax."""
    check_bits(bits)
    if not scale > 0:
        raise UsageError(f"quantization scale must be > 0, got {scale}")
    x64 = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(x64)):
        raise ValueError("cannot quantize non-finite values")
    m = qmax(bits)
    return np.clip(round_half_away(x64 / float(scale)), -m, m).astype(np.int8)


def dequantize_array(q, scale: float) -> np.ndarray:
    """pkg/src/lowbit/quant.py:121-122"""
    return (np.asarray(q, dtype=F32) * F32(scale)).astype(F32)


def group_layout_for(rows: int, groups: int) -> list[tuple[int, int]]:
    """pkg/src/lowbit/quant.py:211-219: equal groups, remainder joins the last."""
    if groups < 1 or groups > rows:
        raise UsageError(f"group count {groups} invalid for {rows} rows")
    base = rows // groups
    layout = [(g * base, base) for g in range(groups)]
    s, c = layout[-1]
    layout[-1] = (s, c + rows - groups * base)
    return layout


def rowwise_scales(maxabs: np.ndarray, bits: int) -> np.ndarray:
    """pkg/src/lowbit/quant.py:222-226"""
    s = (maxabs / qmax(bits)).astype(F32)
    s[maxabs == 0.0] = F32(1.0)
    return s


def quantize_rows(x64: np.ndarray, row_scales: np.ndarray, bits: int) -> np.ndarray:
    """pkg/src/lowbit/quant.py:229-233"""
    m = qmax(bits)
    q = round_half_away(x64 / row_scales.astype(np.float64)[:, None])
    return np.clip(q, -m, m).astype(np.int8)


def quantize_weight_groupwise(w, groups: int, bits: int):
    """pkg/src/lowbit/quant.py:236-255 -> (values int8[n,m], group_scales f32[g], layout)."""
    check_bits(bits)
    w = np.ascontiguousarray(w, dtype=F32)
    if w.ndim != 2:
        raise UsageError(f"weight matrix must be 2-d, got {w.shape}")
    layout = group_layout_for(w.shape[0], groups)
    w64 = w.astype(np.float64)
    if not np.all(np.isfinite(w64)):
        raise ValueError("cannot quantize non-finite weights")
    row_max = np.abs(w64).max(axis=1)
    gmax = np.maximum.reduceat(row_max, np.asarray([s for s, _ in layout]))
    scales = rowwise_scales(gmax, bits)
    counts = np.asarray([c for _, c in layout])
    values = quantize_rows(w64, np.repeat(scales, counts), bits)
    return values, scales, layout


def expand_row_scales(group_scales: np.ndarray, layout) -> np.ndarray:
    """pkg/src/lowbit/quant.py:165-170 (QuantizedMatrix.row_scales)."""
    rows = sum(c for _, c in layout)
    out = np.empty(rows, dtype=F32)
    for (s, c), sc in zip(layout, group_scales):
        out[s : s + c] = sc
    return out


def quantize_activation_tokenwise(x, bits: int):
    """pkg/src/lowbit/quant.py:258-269 -> (values int8[t,d], token_scales f32[t])."""
    check_bits(bits)
    x = np.ascontiguousarray(x, dtype=F32)
    if x.ndim != 2 or x.shape[0] < 1:
        raise UsageError(f"activations must be (tokens x dim), got {x.shape}")
    x64 = x.astype(np.float64)
    if not np.all(np.isfinite(x64)):
        raise ValueError("cannot quantize non-finite activations")
    scales = rowwise_scales(np.abs(x64).max(axis=1), bits)
    return quantize_rows(x64, scales, bits), scales


def quantize_activation_static(x, scale: float, bits: int) -> np.ndarray:
    """pkg/src/lowbit/quant.py:272-281 (values only; the scale is the input)."""
    check_bits(bits)
    if not scale > 0:
        raise UsageError(f"calibrated scale must be > 0, got {scale}")
    return quantize_array(np.ascontiguousarray(x, dtype=F32), scale, bits)


class Calibrator:
    """pkg/src/lowbit/quant.py:289-330 (momentum min/max tracker)."""

    def __init__(self, momentum: float = 0.95):
        if not 0.0 < momentum < 1.0:
            raise UsageError("momentum must be in (0, 1)")
        self.momentum = momentum
        self.x_max = 0.0
        self.x_min = 0.0
        self.observed = 0

    def observe(self, x) -> None:
        x = np.asarray(x)
        if not np.all(np.isfinite(x)):
            raise ValueError("calibrator observed non-finite values")
        bmax, bmin = float(x.max()), float(x.min())
        if self.observed == 0:
            self.x_max, self.x_min = bmax, bmin
        else:
            m = self.momentum
            self.x_max = m * self.x_max + (1.0 - m) * bmax
            self.x_min = m * self.x_min + (1.0 - m) * bmin
        self.observed += 1

    def finalize(self, bits: int) -> float:
        check_bits(bits)
        if self.observed == 0:
            raise UsageError("calibrator finalized before any observation")
        reach = max(abs(self.x_max), abs(self.x_min))
        return 1.0 if reach == 0.0 else float(F32(reach / qmax(bits)))


# ---------------------------------------------------------------------------
# igemm.py
# ---------------------------------------------------------------------------


def check_overflow_guard(inner: int, act_bits: int, w_bits: int) -> None:
    """pkg/src/lowbit/igemm.py:52-63"""
    if inner * qmax(act_bits) * qmax(w_bits) >= INT32_LIMIT:
        raise UsageError("igemm overflow guard")


def igemm(xv: np.ndarray, wv: np.ndarray) -> np.ndarray:
    """pkg/src/lowbit/igemm.py:66-80: exact int32 acc = xv @ wv.T.

    Restated as a float64 BLAS product of the int8 payloads: every partial sum
    is an integer of magnitude < 2^31 << 2^53, so the f64 result is exact and
    bit-identical to the reference's int64 matmul."""
    if xv.shape[1] != wv.shape[1]:
        raise ShapeError("igemm inner dimensions differ")
    return (xv.astype(np.float64) @ wv.astype(np.float64).T).astype(np.int32)


def igemm_int64(xv: np.ndarray, wv: np.ndarray) -> np.ndarray:
    """pkg/src/lowbit/igemm.py:79 verbatim arithmetic (slow, single-threaded);
    used as the reference-cost CPU baseline."""
    return (xv.astype(np.int64) @ wv.astype(np.int64).T).astype(np.int32)


def dequant_epilogue(acc: np.ndarray, act_scales, w_row_scales: np.ndarray, bias=None):
    """pkg/src/lowbit/igemm.py:83-112: ((f32(acc) * s_tok) * s_w) + bias, strict f32 order."""
    if np.isscalar(act_scales):
        rs = np.full(acc.shape[0], F32(act_scales), dtype=F32)
    else:
        rs = np.asarray(act_scales, dtype=F32)
    out = acc.astype(F32)
    out *= rs[:, None]
    out *= np.asarray(w_row_scales, dtype=F32)[None, :]
    if bias is not None:
        out += np.asarray(bias, dtype=F32)[None, :]
    return out


def matmul_f32(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """pkg/src/lowbit/tensor.py:37-56: sequential (p-ascending) f32 sum of rounded products."""
    a = np.ascontiguousarray(a, dtype=F32)
    b = np.ascontiguousarray(b, dtype=F32)
    return np.einsum("ip,pj->ij", a, b, optimize=False)


# Integer GEMM used by quantized_linear: the exact f64-BLAS restatement by
# default; `use_reference_cost_igemm(True)` switches to igemm.py:79's int64
# matmul (single-threaded numpy) so CPU-baseline timings carry the reference's cost.
_IGEMM = [igemm]


def use_reference_cost_igemm(flag: bool) -> None:
    _IGEMM[0] = igemm_int64 if flag else igemm


def quantized_linear(x, wv, w_row_scales, bias, mode: str, static_scale=None, act_bits=8, w_bits=8):
    """pkg/src/lowbit/igemm.py:115-139.  mode in {"dynamic", "static", "full"}."""
    x = np.ascontiguousarray(x, dtype=F32)
    if mode == "full":
        wdq = (wv.astype(F32) * np.asarray(w_row_scales, F32)[:, None]).astype(F32)
        out = matmul_f32(x, wdq.T)
        return out + (np.asarray(bias, F32)[None, :] if bias is not None else F32(0.0))
    if mode == "dynamic":
        xv, s = quantize_activation_tokenwise(x, act_bits)
        check_overflow_guard(wv.shape[1], act_bits, w_bits)
        return dequant_epilogue(_IGEMM[0](xv, wv), s, w_row_scales, bias)
    if mode == "static":
        xv = quantize_activation_static(x, static_scale, act_bits)
        check_overflow_guard(wv.shape[1], act_bits, w_bits)
        return dequant_epilogue(_IGEMM[0](xv, wv), float(static_scale), w_row_scales, bias)
    raise UsageError(mode)


# ---------------------------------------------------------------------------
# tensor.py (the float producers fused into the quantizers)
# ---------------------------------------------------------------------------


def pairwise_sum_f32(a: np.ndarray) -> np.float32:
    """numpy's float32 pairwise summation (the order behind `x.mean(dtype=f32)`
    in pkg/src/lowbit/tensor.py:70-71), restated:

    * n < 8: sequential from 0;
    * 8 <= n <= 128: 8 interleaved accumulators r[j] += a[8i+j], combined as
      ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail sequentially;
    * n > 128: split at n2 = (n//2) rounded down to a multiple of 8, recurse.
    """
    n = len(a)
    if n < 8:
        r = F32(0.0)
        for v in a:
            r = F32(r + v)
        return r
    if n <= 128:
        m = n - n % 8
        r = a[:m].reshape(-1, 8).astype(F32)
        acc = r[0].copy()
        for i in range(1, r.shape[0]):
            acc = (acc + r[i]).astype(F32)
        res = F32(F32(F32(acc[0] + acc[1]) + F32(acc[2] + acc[3]))
                  + F32(F32(acc[4] + acc[5]) + F32(acc[6] + acc[7])))
        for v in a[m:]:
            res = F32(res + v)
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return F32(pairwise_sum_f32(a[:n2]) + pairwise_sum_f32(a[n2:]))


def layer_norm(x, gamma, beta, eps: float = LN_EPS) -> np.ndarray:
    """pkg/src/lowbit/tensor.py:59-73 with the reductions written out
    (pairwise mean / population variance, separate f32 ops, no FMA)."""
    x = np.ascontiguousarray(x, dtype=F32)
    d = x.shape[-1]
    out = np.empty_like(x)
    e = F32(eps)
    g = np.asarray(gamma, F32)
    b = np.asarray(beta, F32)
    for i in range(x.shape[0]):
        row = x[i]
        mean = F32(pairwise_sum_f32(row) / F32(d))
        diff = (row - mean).astype(F32)
        var = F32(pairwise_sum_f32((diff * diff).astype(F32)) / F32(d))
        den = np.sqrt(F32(var + e), dtype=F32)
        out[i] = ((diff / den).astype(F32) * g).astype(F32) + b
    return out


def layer_norm_numpy(x, gamma, beta, eps: float = LN_EPS) -> np.ndarray:
    """pkg/src/lowbit/tensor.py:70-73 verbatim numpy (fast path of the oracle)."""
    x = np.ascontiguousarray(x, dtype=F32)
    mean = x.mean(axis=-1, keepdims=True, dtype=F32)
    var = np.square(x - mean).mean(axis=-1, keepdims=True, dtype=F32)
    norm = (x - mean) / np.sqrt(var + F32(eps))
    return (norm * np.asarray(gamma, F32) + np.asarray(beta, F32)).astype(F32)


def gelu(x) -> np.ndarray:
    """pkg/src/lowbit/tensor.py:76-83: exact-erf GeLU in f64, rounded once to f32."""
    from scipy.special import erf

    x64 = np.asarray(x, dtype=np.float64)
    return (x64 * 0.5 * (1.0 + erf(x64 * _INV_SQRT2))).astype(F32)


def softmax(x) -> np.ndarray:
    """pkg/src/lowbit/tensor.py:94-99"""
    x = np.asarray(x, dtype=F32)
    e = np.exp(x - x.max(axis=-1, keepdims=True), dtype=F32)
    return (e / e.sum(axis=-1, keepdims=True, dtype=F32)).astype(F32)


def layer_norm_quantize(x, gamma, beta, bits: int, eps: float = LN_EPS):
    """pkg/src/lowbit/igemm.py:150-157"""
    return quantize_activation_tokenwise(layer_norm_numpy(x, gamma, beta, eps), bits)


def gelu_quantize(x, bits: int):
    """pkg/src/lowbit/igemm.py:160-161"""
    return quantize_activation_tokenwise(gelu(x), bits)


# ---------------------------------------------------------------------------
# transformer.py (block forward, the caller of the hot path)
# ---------------------------------------------------------------------------


def default_group_count(hidden_dim: int) -> int:
    """pkg/src/lowbit/transformer.py:129-137"""
    if hidden_dim >= 2048:
        return 128
    if hidden_dim >= 1024:
        return 64
    if hidden_dim >= 512:
        return 48
    return 16


def attention(q, k, v, num_heads: int, causal: bool) -> np.ndarray:
    """pkg/src/lowbit/transformer.py:413-440 (always float)."""
    t, d = q.shape
    dh = d // num_heads
    inv = F32(1.0 / math.sqrt(dh))
    out = np.empty((t, d), dtype=F32)
    for h in range(num_heads):
        c = slice(h * dh, (h + 1) * dh)
        s = matmul_f32(q[:, c], np.ascontiguousarray(k[:, c].T))
        s *= inv
        if causal:
            s[np.triu_indices(t, k=1)] = -np.inf
        out[:, c] = matmul_f32(softmax(s), v[:, c])
    return out


def quantize_block(weights: dict, mhsa_bits: int, ffc_bits: int, groups: int) -> dict:
    """pkg/src/lowbit/transformer.py:333-361: groups = min(g, rows) per matrix."""
    qb = {}
    for name, bits in (("w_q", mhsa_bits), ("w_k", mhsa_bits), ("w_v", mhsa_bits),
                       ("w_o", mhsa_bits), ("w_h4h", ffc_bits), ("w_4hh", ffc_bits)):
        w = weights[name]
        vals, sc, lay = quantize_weight_groupwise(w, min(groups, w.shape[0]), bits)
        qb[name] = (vals, expand_row_scales(sc, lay), bits)
    for k, v in weights.items():
        if not k.startswith("w_"):
            qb[k] = v
    return qb


def block_forward(x, qb: dict, num_heads: int, causal: bool, act_mode: str = "int8") -> np.ndarray:
    """pkg/src/lowbit/transformer.py:443-486 for a QuantizedBlock with dynamic
    activations.  act_mode: "int8" (A8) or "int8_attn_full" (A8/16: q/k/v full)."""
    x = np.ascontiguousarray(x, dtype=F32)

    def lin(inp, name, bname, mode):
        vals, rs, bits = qb[name]
        return quantized_linear(inp, vals, rs, qb[bname], mode, w_bits=bits)

    am = "full" if act_mode == "int8_attn_full" else "dynamic"
    q = lin(x, "w_q", "b_q", am)
    k = lin(x, "w_k", "b_k", am)
    v = lin(x, "w_v", "b_v", am)
    ctx = attention(q, k, v, num_heads, causal)
    attn_out = lin(ctx, "w_o", "b_o", "dynamic")
    h = layer_norm_numpy(x + attn_out, qb["ln1_gamma"], qb["ln1_beta"], LN_EPS)
    u = lin(h, "w_h4h", "b_h4h", "dynamic")
    z = gelu(u)
    f = lin(z, "w_4hh", "b_4hh", "dynamic")
    return layer_norm_numpy(h + f, qb["ln2_gamma"], qb["ln2_beta"], LN_EPS)


def block_forward_static(x, qb: dict, num_heads: int, causal: bool, layer: int,
                         static_scales: dict) -> np.ndarray:
    """pkg/src/lowbit/transformer.py:443-486 with activation_static=True: every
    GEMM-input site quantizes with its calibrated scale (_act_mode_for,
    transformer.py:386-402 -> StaticAct; igemm.py:131-134)."""
    x = np.ascontiguousarray(x, dtype=F32)

    def lin(inp, name, bname, site):
        vals, rs, bits = qb[name]
        return quantized_linear(inp, vals, rs, qb[bname], "static",
                                static_scale=static_scales[f"layer{layer}.{site}"], w_bits=bits)

    q = lin(x, "w_q", "b_q", "attn_in")
    k = lin(x, "w_k", "b_k", "attn_in")
    v = lin(x, "w_v", "b_v", "attn_in")
    ctx = attention(q, k, v, num_heads, causal)
    attn_out = lin(ctx, "w_o", "b_o", "attn_proj_in")
    h = layer_norm_numpy(x + attn_out, qb["ln1_gamma"], qb["ln1_beta"], LN_EPS)
    u = lin(h, "w_h4h", "b_h4h", "ffc_in")
    z = gelu(u)
    f = lin(z, "w_4hh", "b_4hh", "ffc_mid")
    return layer_norm_numpy(h + f, qb["ln2_gamma"], qb["ln2_beta"], LN_EPS)


# ---------------------------------------------------------------------------
# Deterministic synthetic inputs: pkg/src/lowbit/tensor.py:113-164
# ---------------------------------------------------------------------------

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


class Rng:
    """Counter-based splitmix64 (pkg/src/lowbit/tensor.py:119-164)."""

    def __init__(self, seed: int):
        self._seed = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self._counter = 0

    def _raw(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(self._counter + 1, self._counter + n + 1, dtype=np.uint64)
            z = self._seed + idx * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _MIX1
            z = (z ^ (z >> np.uint64(27))) * _MIX2
            z = z ^ (z >> np.uint64(31))
        self._counter += n
        return z

    def uniform(self, n: int) -> np.ndarray:
        return (self._raw(n) >> np.uint64(11)).astype(np.float64) * (1.0 / float(1 << 53))

    def gaussian(self, shape, std: float = 1.0) -> np.ndarray:
        n = int(np.prod(shape)) if not isinstance(shape, int) else shape
        pairs = (n + 1) // 2
        u1 = 1.0 - self.uniform(pairs)
        u2 = self.uniform(pairs)
        r = np.sqrt(-2.0 * np.log(u1))
        th = 2.0 * math.pi * u2
        z = np.concatenate([r * np.cos(th), r * np.sin(th)])[:n]
        return (z * std).astype(F32).reshape(shape)

    def integers(self, upper: int, n: int) -> np.ndarray:
        return (self._raw(n) % np.uint64(upper)).astype(np.int64)


# ---------------------------------------------------------------------------
# INT4 packing used by the B200 W4A8 path (new format; no reference analogue:
# the reference stores INT4 one value per byte, pkg/src/lowbit/quant.py:138-141)
# ---------------------------------------------------------------------------


def pack_int4(values: np.ndarray) -> np.ndarray:
    """Two's-complement nibbles, element 2k in the low nibble of byte k (per row)."""
    v = np.asarray(values, dtype=np.int8)
    if v.shape[-1] % 2:
        raise UsageError("int4 packing needs an even number of columns")
    lo = (v[..., 0::2].astype(np.uint8) & 0xF)
    hi = (v[..., 1::2].astype(np.uint8) & 0xF) << 4
    return (lo | hi).astype(np.uint8)


def unpack_int4(packed: np.ndarray) -> np.ndarray:
    p = np.asarray(packed, dtype=np.uint8)
    lo = (p & 0xF).astype(np.int8)
    hi = (p >> 4).astype(np.int8)
    lo = np.where(lo > 7, lo - 16, lo).astype(np.int8)
    hi = np.where(hi > 7, hi - 16, hi).astype(np.int8)
    out = np.empty(p.shape[:-1] + (p.shape[-1] * 2,), dtype=np.int8)
    out[..., 0::2] = lo
    out[..., 1::2] = hi
    return out


# ---------------------------------------------------------------------------
# scipy.special.erf provenance (the f64 erf inside tensor.gelu, tensor.py:15,83)
# ---------------------------------------------------------------------------
# scipy 1.18's real erf is the Cephes ndtr.c algorithm; restated here (and in
# the GPU kernel, csrc/zq_quant.cu cephes_erf) so that the GeLU's f64 value —
# whose low bits survive the 1 + erf(x) cancellation for x << 0 — is pinned to
# a written-down algorithm.  tests/test_oracle_golden.py checks it equals scipy.
_ERF_T = [9.60497373987051638749E0, 9.00260197203842689217E1, 2.23200534594684319226E3,
          7.00332514112805075473E3, 5.55923013010394962768E4]
_ERF_U = [3.35617141647503099647E1, 5.21357949780152679795E2, 4.59432382970980127987E3,
          2.26290000613890934246E4, 4.92673942608635921086E4]
_ERF_P = [2.46196981473530512524E-10, 5.64189564831068821977E-1, 7.46321056442269912687E0,
          4.86371970985681366614E1, 1.96520832956077098242E2, 5.26445194995477358631E2,
          9.34528527171957607540E2, 1.02755188689515710272E3, 5.57535335369399327526E2]
_ERF_Q = [1.32281951154744992508E1, 8.67072140885989742329E1, 3.54937778887819891062E2,
          9.75708501743205489753E2, 1.82390916687909736289E3, 2.24633760818710981792E3,
          1.65666309194161350182E3, 5.57535340817727675546E2]
_ERF_R = [5.64189583547755073984E-1, 1.27536670759978104416E0, 5.01905042251180477414E0,
          6.16021097993053585195E0, 7.40974269950448939160E0, 2.97886665372100240670E0]
_ERF_S = [2.26052863220117276590E0, 9.39603524938001434673E0, 1.20489539808096656605E1,
          1.70814450747565897222E1, 9.60896809063285878198E0, 3.36907645100081516050E0]
_MAXLOG = 7.09782712893383996843E2


def _polevl(x, c, n):
    a = c[0]
    for i in range(1, n + 1):
        a = a * x + c[i]
    return a


def _p1evl(x, c, n):
    a = x + c[0]
    for i in range(1, n):
        a = a * x + c[i]
    return a


def cephes_erf(x: float) -> float:
    """Scalar Cephes erf in IEEE double (Python floats), op order as ndtr.c."""
    if x < 0.0:
        return -cephes_erf(-x)
    if x <= 1.0:
        z = x * x
        return x * _polevl(z, _ERF_T, 4) / _p1evl(z, _ERF_U, 5)
    z = -x * x
    if z < -_MAXLOG:
        return 1.0
    e = math.exp(z)
    if x < 8.0:
        p, q = _polevl(x, _ERF_P, 8), _p1evl(x, _ERF_Q, 8)
    else:
        p, q = _polevl(x, _ERF_R, 5), _p1evl(x, _ERF_S, 6)
    return 1.0 - (e * p) / q


# ---------------------------------------------------------------------------
# Static calibration on the float model (evaluate.py:168-196)
# ---------------------------------------------------------------------------


def numpy_expf(x) -> np.ndarray:
    """numpy 2.x's float32 exp (simd_exp_f32, the kernel behind np.exp on
    float32 arrays in tensor.softmax, tensor.py:94-99), restated: Cody-Waite
    range reduction with FMA, a [5/2] rational minimax, scaling by 2^k.  FMA is
    emulated in float64 (a*b is exact there); pinned against np.exp in
    tests/test_oracle_golden.py.  The GPU restates it as np_expf
    (csrc/zq_calib.cu)."""
    x = np.asarray(x, dtype=F32)
    d = np.float64

    def fma(a, b, c):  # f32(a*b + c), one rounding (a*b exact in f64)
        return (np.asarray(a, d) * np.asarray(b, d) + np.asarray(c, d)).astype(F32)

    P = [F32(c) for c in (9.999999999980870924916e-01, 7.257664613233124478488e-01, 2.473615434895520810817e-01,
                          5.114512081637298353406e-02, 6.757896990527504603057e-03, 5.082762527590693718096e-04)]
    Q1, Q2 = F32(-2.742335390411667452936e-01), F32(2.159509375685829852307e-02)
    with np.errstate(all="ignore"):
        quad = (x * F32(1.442695040888963407359924681001892137)).astype(F32)
        quad = ((quad + F32(12582912.0)).astype(F32) - F32(12582912.0)).astype(F32)
        r = fma(quad, F32(-6.93145752e-1), x)
        r = fma(quad, F32(-1.42860677e-6), r)
        num = fma(P[5], r, P[4])
        for c in (P[3], P[2], P[1], P[0]):
            num = fma(num, r, c)
        den = fma(fma(Q2, r, Q1), r, F32(1.0))
        v = (num / den).astype(F32)
        out = (v.astype(d) * np.exp2(quad.astype(d))).astype(F32)
    out = np.where(x >= F32(88.72283935546875), F32(np.inf), out)
    out = np.where(x <= F32(-103.97208404541015625), F32(0.0), out)
    return np.where(np.isnan(x), x, out).astype(F32)


def float_block_forward(x, w: dict, num_heads: int, causal: bool, layer: int = 0, tap=None) -> np.ndarray:
    """pkg/src/lowbit/transformer.py:443-486 for float weights (FullAct
    everywhere, _linear = tensor.matmul + bias, transformer.py:405-410)."""
    x = np.ascontiguousarray(x, dtype=F32)

    def lin(inp, a, b):
        out = matmul_f32(inp, np.ascontiguousarray(w[a].T))
        out += np.asarray(w[b], F32)[None, :]
        return out

    if tap is not None:
        tap("attn_in", layer, x)
    ctx = attention(lin(x, "w_q", "b_q"), lin(x, "w_k", "b_k"), lin(x, "w_v", "b_v"), num_heads, causal)
    if tap is not None:
        tap("attn_proj_in", layer, ctx)
    h = layer_norm_numpy(x + lin(ctx, "w_o", "b_o"), w["ln1_gamma"], w["ln1_beta"])
    if tap is not None:
        tap("ffc_in", layer, h)
    z = gelu(lin(h, "w_h4h", "b_h4h"))
    if tap is not None:
        tap("ffc_mid", layer, z)
    return layer_norm_numpy(h + lin(z, "w_4hh", "b_4hh"), w["ln2_gamma"], w["ln2_beta"])


def calibrate_model(embedding, blocks: list, num_heads: int, causal: bool, batches, momentum: float = 0.95,
                    bits: int = 8) -> dict:
    """pkg/src/lowbit/evaluate.py:168-196: {key: (x_max, x_min, scale)}."""
    cals: dict = {}

    def tap(site, layer, x):
        cals.setdefault(f"layer{layer}.{site}", Calibrator(momentum)).observe(x)

    for ids in batches:
        x = np.asarray(embedding, F32)[np.asarray(ids, np.int64)]
        for li, w in enumerate(blocks):
            x = float_block_forward(x, w, num_heads, causal, li, tap)
    return {k: (c.x_max, c.x_min, c.finalize(bits)) for k, c in sorted(cals.items())}
