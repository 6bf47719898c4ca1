"""GPU parity of the converted-weight CTA-pair GEMMs (csrc/zq_gemm_conv.cu):

* W4A8 on CTA pairs (INT4 -> int8 in shared memory, kind::i8): bit-exact vs the
  oracle's quantized_linear (pkg/src/lowbit/igemm.py:115-139).
* FullAct tolerance modes (igemm.py:127-130): int8 / INT4 weights -> f16 in
  shared memory, activations as 1 ("f16") or 2 ("f16x2") power-of-two-scaled f16
  terms, tcgen05 kind::f16.  Stated tolerances, max|out - ref| / max|ref|:
  f16 <= 2e-3, f16x2 <= 5e-5 (ref = the oracle's sequential f32 FullAct, and a
  float64 evaluation of the same dequantized product; f16x2's split error is
  ~2^-22, the rest is f32 accumulation order, which the reference's own
  sequential sum shares at K = 6144)."""

import numpy as np
import pytest
import torch

from oracle import lowbit_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32
TOL = {"f16": 2e-3, "f16x2": 5e-5}


@pytest.fixture(scope="module")
def zq():
    from paper_2206_01861_b200 import igemm, quant

    return quant, igemm


def h(t):
    return t.detach().float().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def bits_eq(a, b):
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _case(quant, shape, wbits, seed, xscale=1.0):
    t, d, n, g = shape
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((t, d)) * xscale).astype(F32)
    w = (rng.standard_normal((n, d)) * 0.02).astype(F32)
    bias = (rng.standard_normal(n) * 0.1).astype(F32)
    wq = quant.quantize_weight_groupwise(w, g, wbits)
    wv, gs, lay = O.quantize_weight_groupwise(w, g, wbits)
    rs = O.expand_row_scales(gs, lay)
    return x, bias, wq, wv, rs


def _ref64(x, wv, rs, bias):
    wdq = (wv.astype(F32) * rs[:, None]).astype(F32).astype(np.float64)
    return x.astype(np.float64) @ wdq.T + bias.astype(np.float64)[None, :]


@pytest.mark.parametrize("wbits", [8, 4])
@pytest.mark.parametrize("shape", [(4096, 768, 3072, 48), (1000, 1000, 3000, 30), (600, 3072, 768, 48),
                                   (8192, 1024, 4096, 64)])
def test_w4a8_pair_bit_exact(zq, shape, wbits):
    """Shapes large enough for the CTA-pair path (W8 already had it; W4 now runs
    the converted-weight pair kernel)."""
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, shape, wbits, sum(shape) + wbits)
    out = h(igemm.quantized_linear(x, wq, bias, igemm.DynamicAct(8)))
    ref = O.quantized_linear(x, wv, rs, bias, "dynamic", w_bits=wbits)
    assert bits_eq(out, ref), shape


@pytest.mark.parametrize("wbits", [8, 4])
def test_w4a8_pair_f16_out_is_rn_cast(zq, wbits):
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, (2048, 768, 3072, 48), wbits, 5)
    ref = O.quantized_linear(x, wv, rs, bias, "dynamic", w_bits=wbits)
    xq = quant.quantize_activation_tokenwise(x, 8)
    for dt in (torch.float16, torch.bfloat16):
        out = igemm.fused_linear(xq, wq, bias, out_dtype=dt)
        assert torch.equal(out.cpu(), torch.from_numpy(ref).to(dt)), dt


@pytest.mark.parametrize("precision", ["f16", "f16x2"])
@pytest.mark.parametrize("wbits", [8, 4])
@pytest.mark.parametrize("shape", [(256, 768, 512, 8), (300, 1000, 700, 7), (33, 200, 130, 1)])
def test_full_tc_vs_oracle(zq, shape, wbits, precision):
    """Small shapes (ragged M / N / K, K not a multiple of 64): the oracle's
    sequential f32 FullAct and a float64 evaluation."""
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, shape, wbits, 7 * sum(shape) + wbits)
    out = h(igemm.full_linear(x, wq, bias, precision=precision))
    ref = O.quantized_linear(x, wv, rs, bias, "full", w_bits=wbits)
    r64 = _ref64(x, wv, rs, bias)
    scale = np.abs(r64).max()
    assert np.abs(out - ref).max() <= TOL[precision] * scale, (shape, precision)
    assert np.abs(out - r64).max() <= TOL[precision] * scale, (shape, precision)


@pytest.mark.parametrize("precision", ["f16", "f16x2"])
@pytest.mark.parametrize("wbits", [8, 4])
def test_full_tc_large_vs_float64(zq, wbits, precision):
    """A NeoX-width slice (K = 6144) against float64 on the device: the
    row-wise error bound of the split, independent of the f32 order."""
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, (512, 6144, 2304, 48), wbits, 11 + wbits)
    out = igemm.full_linear(x, wq, bias, precision=precision).double()
    wdq = torch.from_numpy((wv.astype(F32) * rs[:, None]).astype(F32)).cuda().double()
    r64 = torch.from_numpy(x).cuda().double() @ wdq.T + torch.from_numpy(bias).cuda().double()[None, :]
    assert ((out - r64).abs().max() / r64.abs().max()).item() <= TOL[precision]


def test_full_tc_activation_range(zq):
    """Power-of-two row scaling: rows far outside the fp16 range (1e6, 1e-6)
    keep their relative precision; a zero row gives zeros."""
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, (64, 512, 256, 4), 8, 3)
    x[0] *= F32(1e6)
    x[1] *= F32(1e-6)
    x[2] = 0
    r64 = _ref64(x, wv, rs, np.zeros_like(bias))
    for precision in ("f16", "f16x2"):
        out = h(igemm.full_linear(x, wq, None, precision=precision))
        assert np.isfinite(out).all()
        for i in (0, 1, 3):
            assert np.abs(out[i] - r64[i]).max() <= 2 * TOL[precision] * np.abs(r64[i]).max(), (precision, i)
        assert not out[2].any()


def test_full_tc_half_outputs(zq):
    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, (300, 768, 1000, 8), 8, 9)
    r64 = _ref64(x, wv, rs, bias)
    for dt, tol in ((torch.float16, 3e-3), (torch.bfloat16, 1e-2)):
        out = h(igemm.full_linear(x, wq, bias, precision="f16x2", out_dtype=dt))
        assert np.abs(out - r64).max() <= tol * np.abs(r64).max(), dt


def test_full_precision_validation(zq):
    from paper_2206_01861_b200.errors import UsageError

    quant, igemm = zq
    x, bias, wq, wv, rs = _case(quant, (4, 64, 32, 1), 8, 1)
    with pytest.raises(UsageError):
        igemm.full_linear(x, wq, bias, precision="tf32")
    with pytest.raises(UsageError):
        igemm.full_linear(x, wq, bias, precision="exact", out_dtype=torch.float16)


@pytest.mark.parametrize("full_act", ["f16", "f16x2"])
@pytest.mark.parametrize("causal", [False, True])
def test_block_forward_a16_site_tensor_core(golden, full_act, causal):
    """W8A8/16 (attn_in is FullAct, transformer.py:395) with the QKV projection on
    the tensor-core weight-only path: the block output stays within the block
    tolerance of the reference's golden output (relative L2 2e-3, as the exact
    path in tests/test_transformer_gpu.py)."""
    from paper_2206_01861_b200 import transformer as T

    blk = {k[len("block_"):]: v for k, v in golden.items()
           if k.startswith("block_") and not k.startswith("block_W") and k != "block_x"}
    blk["num_heads"] = 4
    prec = T.PrecisionConfig.from_scheme("W8A8/16", hidden_dim=64)
    db = T.quantize_block(blk, prec)
    y = T.block_forward(golden["block_x"], db, prec, causal, full_act=full_act).cpu().numpy().astype(np.float64)
    ref = golden[f"block_W8A8_16_c{int(causal)}_y"].astype(np.float64)
    assert np.linalg.norm(y - ref) / np.linalg.norm(ref) < 2e-3
