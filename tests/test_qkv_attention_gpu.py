"""Fused QKV projection + attention (zq_qkv_attention, csrc/zq_attention.cu):
ctx must be bit-identical to the two-kernel path it replaces (zq_linear with f32
output -> zq_attention_f32), i.e. to the reference's quantized_linear on the
concatenated QKV weight followed by attention (pkg/src/lowbit/transformer.py:
395-440).  Covers BERT-base / BERT-large widths, ragged sequences (128-row GEMM
tiles that straddle sequences and run past the last token), causal masking, no
bias, and the engine with the fusion on and off."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zq():
    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import quant, transformer

    return N, quant, transformer


def _unfused(N, xq, w, bias, batch, seq, heads, causal):
    t, d = xq.values.shape[0], w.cols
    qkv = torch.empty((t, 3 * d), dtype=torch.float32, device="cuda")
    wp, ldw, wb = w.weight_operand()
    N.call("zq_linear", xq.values.data_ptr(), xq.values.stride(0), xq.token_scales.data_ptr(), 0.0, wp, ldw, wb,
           w.row_scales().data_ptr(), N.ptr(bias), t, 3 * d, d, qkv.data_ptr(), qkv.stride(0), N.OUT_F32,
           N.stream_ptr())
    ctx = torch.full((t, d), float("nan"), device="cuda")
    scale = float(np.float32(1.0 / math.sqrt(d // heads)))
    N.call("zq_attention_f32", qkv.data_ptr(), qkv.stride(0), batch, seq, heads, d // heads, int(causal), scale,
           ctx.data_ptr(), ctx.stride(0), N.stream_ptr())
    return ctx


def _fused(N, xq, w, bias, batch, seq, heads, causal):
    t, d = xq.values.shape[0], w.cols
    ctx = torch.full((t, d), float("nan"), device="cuda")
    wp, ldw, _ = w.weight_operand()
    scale = float(np.float32(1.0 / math.sqrt(d // heads)))
    rc = N.call_rc("zq_qkv_attention", xq.values.data_ptr(), xq.values.stride(0), xq.token_scales.data_ptr(), wp,
                   ldw, w.row_scales().data_ptr(), N.ptr(bias), batch, seq, heads, d // heads, int(causal), scale,
                   ctx.data_ptr(), ctx.stride(0), N.stream_ptr())
    return rc, ctx


def _case(quant, batch, seq, d, groups, seed, with_bias=True, xscale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((batch * seq, d), device="cuda", generator=g) * xscale
    w = torch.randn((3 * d, d), device="cuda", generator=g) * 0.05
    bias = torch.randn(3 * d, device="cuda", generator=g) * 0.1 if with_bias else None
    return quant.quantize_activation_tokenwise(x, 8), quant.quantize_weight_groupwise(w, groups, 8), bias


@pytest.mark.parametrize("batch,seq,heads,groups,causal,with_bias", [
    (32, 128, 12, 48, False, True),    # BERT-base bench shape
    (4, 128, 16, 64, False, True),     # BERT-large width (d = 1024)
    (5, 100, 12, 48, False, True),     # tiles straddle sequences and run past the last token
    (3, 77, 2, 1, True, True),         # causal, d = 128, per-tensor weight scale
    (7, 128, 4, 8, True, False),       # no bias
    (1, 1, 12, 48, False, True),       # one token
    (200, 64, 12, 48, False, True),    # more units than SMs, several per CTA
])
def test_fused_qkv_attention_bit_identical(zq, batch, seq, heads, groups, causal, with_bias):
    N, quant, _ = zq
    d = 64 * heads
    xq, w, bias = _case(quant, batch, seq, d, groups, seed=batch * 1000 + seq + heads, with_bias=with_bias)
    ref = _unfused(N, xq, w, bias, batch, seq, heads, causal)
    rc, out = _fused(N, xq, w, bias, batch, seq, heads, causal)
    assert rc == N.ZQ_OK
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))


def test_fused_qkv_attention_extreme_scales(zq):
    """Large and tiny activations (the per-tile power-of-two scales of the
    attention split see the projected values exactly as the unfused path)."""
    N, quant, _ = zq
    batch, seq, heads = 6, 128, 12
    d = 64 * heads
    for xs in (1e4, 1e-4):
        xq, w, bias = _case(quant, batch, seq, d, 48, seed=int(xs * 7) % 97 + 5, xscale=xs)
        ref = _unfused(N, xq, w, bias, batch, seq, heads, False)
        rc, out = _fused(N, xq, w, bias, batch, seq, heads, False)
        assert rc == N.ZQ_OK
        assert torch.equal(out.view(torch.int32), ref.view(torch.int32)), xs


def test_fused_qkv_attention_unsupported(zq):
    N, quant, _ = zq
    xq, w, bias = _case(quant, 2, 16, 96, 1, seed=3)  # head_dim 32
    rc, _ = _fused(N, xq, w, bias, 2, 16, 3, False)
    assert rc == N.ZQ_ERR_UNSUPPORTED
    xq, w, bias = _case(quant, 2, 160, 128, 1, seed=4)  # seq > 128
    rc, _ = _fused(N, xq, w, bias, 2, 160, 2, False)
    assert rc == N.ZQ_ERR_UNSUPPORTED


@pytest.mark.parametrize("causal", [False, True])
def test_engine_fused_qkv_bit_identical(zq, causal):
    """EncoderEngine (CUDA graph) with the fused QKV + attention kernel against
    the same engine running the two kernels."""
    N, quant, T = zq
    d, heads, layers, batch, seq = 768, 12, 2, 8, 128
    blocks = [T.random_block(d, heads, 8, 8, 48, seed=10 + i) for i in range(layers)]
    emb = torch.randn((500, d), device="cuda") * 0.5
    ids = torch.randint(0, 500, (batch, seq))
    outs = []
    for fuse in (True, False):
        eng = T.EncoderEngine(blocks=blocks, embedding=emb, final_gamma=torch.ones(d, device="cuda"),
                              final_beta=torch.zeros(d, device="cuda"), batch=batch, seq=seq, causal=causal)
        eng._fuse_qkv = fuse
        outs.append(eng.forward(ids).clone())
        eng.check_finite()
        assert eng._fuse_qkv == fuse  # the fused shape was accepted
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))


_VARIANT_CHECK = r"""
import math, sys, numpy as np, torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import test_qkv_attention_gpu as Tq
from paper_2206_01861_b200 import _native as N, quant
for batch, seq, heads, causal in ((32, 128, 12, False), (5, 100, 12, False), (7, 128, 4, True)):
    xq, w, bias = Tq._case(quant, batch, seq, 64 * heads, 48 if heads == 12 else 8, seed=batch + seq)
    ref = Tq._unfused(N, xq, w, bias, batch, seq, heads, causal)
    rc, out = Tq._fused(N, xq, w, bias, batch, seq, heads, causal)
    assert rc == N.ZQ_OK and torch.equal(out.view(torch.int32), ref.view(torch.int32)), (batch, seq, heads)
    for _ in range(3):  # back-to-back launches (programmatic dependent launch between them)
        Tq._fused(N, xq, w, bias, batch, seq, heads, causal)
    torch.cuda.synchronize()
print("ok")
"""


@pytest.mark.parametrize("variant", ["8", "0"])
def test_fused_qkv_attention_variants(variant):
    """The selectable kernel variants (ZQ_QA_CW=8: 8 compute warps; 0: split
    convert / attention roles) are bit-identical too; the variant is chosen once
    per process, so each runs in its own interpreter (timeout: a hang fails)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _VARIANT_CHECK.format(root=root, tests=os.path.join(root, "tests"))
    env = dict(os.environ, ZQ_QA_CW=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
