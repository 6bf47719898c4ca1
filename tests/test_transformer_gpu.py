"""GPU: block forward / encoder engine vs the reference block (golden vectors
from lowbit.transformer.block_forward, and the oracle).  Attention is float in
the reference and on B200 (different summation order), so block outputs are
compared with a relative-L2 tolerance; the quantized sub-steps are bit-exact
(tests/test_quant_gpu.py, tests/test_igemm_gpu.py)."""

import numpy as np
import pytest
import torch

from oracle import lowbit_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32
TOL = 2e-3  # relative L2 after LN (attention rounding can flip rare int8 codes)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def golden_block(golden):
    return {k[len("block_"):]: v for k, v in golden.items()
            if k.startswith("block_") and not k.startswith("block_W") and k != "block_x"}


@pytest.mark.parametrize("scheme", ["W8A8", "W4/8A8", "W8A8/16"])
@pytest.mark.parametrize("causal", [False, True])
def test_block_forward_golden(golden, scheme, causal):
    from paper_2206_01861_b200 import transformer as T

    blk = golden_block(golden)
    blk["num_heads"] = 4
    prec = T.PrecisionConfig.from_scheme(scheme, hidden_dim=64)
    db = T.quantize_block(blk, prec)
    y = T.block_forward(golden["block_x"], db, prec, causal).cpu().numpy()
    ref = golden[f"block_{scheme.replace('/', '_')}_c{int(causal)}_y"]
    assert rel(y, ref) < TOL, rel(y, ref)


def test_quantize_block_matches_reference_payloads(golden):
    from paper_2206_01861_b200 import transformer as T

    blk = golden_block(golden)
    blk["num_heads"] = 4
    prec = T.PrecisionConfig.from_scheme("W4/8A8", hidden_dim=64)
    db = T.quantize_block(blk, prec)
    qb = O.quantize_block(blk, 8, 4, 16)
    for name in ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh"):
        m = getattr(db, name)
        assert np.array_equal(m.values.cpu().numpy(), qb[name][0]), name
        assert np.array_equal(m.row_scales().cpu().numpy(), qb[name][1]), name
    # fused QKV = the three matrices stacked
    assert np.array_equal(db.w_qkv.values.cpu().numpy(),
                          np.concatenate([qb["w_q"][0], qb["w_k"][0], qb["w_v"][0]]))


def test_bert_shaped_block_vs_oracle():
    """One BERT-base-shaped block (d=768, 12 heads, FFN 3072, g=48) on 2 x 128
    tokens vs the oracle's reference block forward."""
    from paper_2206_01861_b200 import transformer as T

    d, f, seq = 768, 3072, 128
    rng = O.Rng(5)
    w = {n: rng.gaussian(s, std=0.02) for n, s in (
        ("w_q", (d, d)), ("w_k", (d, d)), ("w_v", (d, d)), ("w_o", (d, d)), ("w_h4h", (f, d)), ("w_4hh", (d, f)))}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d),
                 ("ln1_beta", d), ("ln2_beta", d)):
        w[n] = (0.01 * np.arange(s) / s).astype(F32)
    w["ln1_gamma"] = np.ones(d, F32)
    w["ln2_gamma"] = np.ones(d, F32)
    w["num_heads"] = 12
    prec = T.PrecisionConfig.from_scheme("W8A8", hidden_dim=d)
    db = T.quantize_block(w, prec)
    qb = O.quantize_block(w, 8, 8, 48)
    xs = [O.Rng(10 + i).gaussian((seq, d), std=0.5) for i in range(2)]
    y = T.block_forward(np.concatenate(xs), db, prec, causal=False, batch=2).cpu().numpy()
    for i, x in enumerate(xs):
        ref = O.block_forward(x, qb, 12, False, "int8")
        assert rel(y[i * seq:(i + 1) * seq], ref) < TOL


def test_encoder_engine_matches_block_forward():
    from paper_2206_01861_b200 import transformer as T

    d, heads, layers, batch, seq = 256, 4, 3, 2, 64
    blocks = [T.random_block(d, heads, 8, 8, 16, seed=i) for i in range(layers)]
    emb = torch.randn((100, d), device="cuda") * 0.02
    eng = T.EncoderEngine(blocks=blocks, embedding=emb, final_gamma=torch.ones(d, device="cuda"),
                          final_beta=torch.zeros(d, device="cuda"), batch=batch, seq=seq, causal=True)
    ids = torch.randint(0, 100, (batch, seq))
    out = eng.forward(ids).clone()
    eng.check_finite()
    prec = T.PrecisionConfig.from_scheme("W8A8", group_count=16)
    x = emb[ids.reshape(-1).cuda()]
    for blk in blocks:
        x = T.block_forward(x, blk, prec, causal=True, batch=batch)
    from paper_2206_01861_b200 import igemm

    ref = torch.empty_like(x)
    igemm.layer_norm_quantize(x, torch.ones(d, device="cuda"), torch.zeros(d, device="cuda"), 8, ln_out=ref)
    assert rel(out.cpu().numpy(), ref.cpu().numpy()) < 1e-6
    # graph replay is deterministic
    out2 = eng.forward(ids).clone()
    assert torch.equal(out, out2)


def _float_weights(rng, d, f):
    w = {n: rng.gaussian(s, std=0.05) for n, s in (
        ("w_q", (d, d)), ("w_k", (d, d)), ("w_v", (d, d)), ("w_o", (d, d)),
        ("w_h4h", (f, d)), ("w_4hh", (d, f)))}
    for n, s in (("b_q", d), ("b_k", d), ("b_v", d), ("b_o", d), ("b_h4h", f), ("b_4hh", d)):
        w[n] = rng.gaussian((s,), std=0.02)
    for n in ("ln1", "ln2"):
        w[f"{n}_gamma"] = (1.0 + rng.gaussian((d,), std=0.1)).astype(F32)
        w[f"{n}_beta"] = rng.gaussian((d,), std=0.1)
    return w


def _oracle_float_block(x, w, heads, causal, layer, tap):
    """transformer.py:443-486 with float weights (the calibration forward)."""
    lin = lambda inp, a, b: O.matmul_f32(inp, w[a].T) + w[b]  # noqa: E731
    tap("attn_in", layer, x)
    ctx = O.attention(lin(x, "w_q", "b_q"), lin(x, "w_k", "b_k"), lin(x, "w_v", "b_v"), heads, causal)
    tap("attn_proj_in", layer, ctx)
    h = O.layer_norm_numpy(x + lin(ctx, "w_o", "b_o"), w["ln1_gamma"], w["ln1_beta"])
    tap("ffc_in", layer, h)
    z = O.gelu(lin(h, "w_h4h", "b_h4h"))
    tap("ffc_mid", layer, z)
    return O.layer_norm_numpy(h + lin(z, "w_4hh", "b_4hh"), w["ln2_gamma"], w["ln2_beta"])


def test_static_calibration_and_static_forward():
    """§8f row 3: calibration on device (evaluate.py:168-200 over the float blocks,
    one momentum Calibrator per GEMM-input site) reproduces the reference's
    calibrated scales, and the static-activation block forward (StaticAct at every
    site, transformer.py:386-402) matches the reference block with those scales."""
    from paper_2206_01861_b200 import transformer as T

    d, heads, f, L = 128, 4, 512, 2
    rng = O.Rng(11)
    ws = [_float_weights(rng, d, f) for _ in range(L)]
    batches = [rng.gaussian((48, d), std=0.5) for _ in range(3)]
    scales = T.calibrate_static_scales(ws, batches, heads, causal=True)
    cals = {}

    def tap(site, layer, x):
        cals.setdefault(f"layer{layer}.{site}", O.Calibrator()).observe(x)

    for xb in batches:
        x = xb
        for li, w in enumerate(ws):
            x = _oracle_float_block(x, w, heads, True, li, tap)
    ref_scales = {k: c.finalize(8) for k, c in cals.items()}
    assert sorted(scales) == sorted(ref_scales)
    for k in ref_scales:  # the float forward is order-exact: identical scales
        assert scales[k] == ref_scales[k], (k, scales[k], ref_scales[k])
    prec = T.PrecisionConfig.from_scheme("W8A8", group_count=16, activation_static=True)
    x = batches[0]
    for li, w in enumerate(ws):
        db = T.quantize_block(dict(w, num_heads=heads), prec)
        y = T.block_forward(x, db, prec, True, layer=li, static_scales=scales).cpu().numpy()
        ref = O.block_forward_static(x, O.quantize_block(w, 8, 8, 16), heads, True, li, ref_scales)
        assert rel(y, ref) < TOL, (li, rel(y, ref))
        x = ref


def test_calibrate_model_bit_exact_vs_reference_then_static_forward():
    """§8f row 3 end to end against the REAL reference (tests/golden/calibration.npz,
    oracle/make_calibration_golden.py): lowbit.evaluate.calibrate_model over three
    token sequences of the fixture model; the device calibration (order-exact
    float forward, csrc/zq_calib.cu) must give the same x_max / x_min / scale per
    site bit for bit.  The W8A8 static model built from those scales then runs on
    device and is compared with the reference's static model_forward logits."""
    import os

    from paper_2206_01861_b200 import igemm
    from paper_2206_01861_b200 import transformer as T

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "calibration.npz"))
    L, heads = int(g["layers"]), int(g["num_heads"])
    blocks = [{n[3:]: g[n] for n in g.files if n.startswith(f"l{li}_")} for li in range(L)]
    batches = [g[f"batch{i}"] for i in range(3)]
    cal = T.calibrate_model(g["embedding"], blocks, heads, True, batches)
    assert list(cal) == list(g["site_keys"])
    for k, xm, xn, sc in zip(g["site_keys"], g["site_xmax"], g["site_xmin"], g["site_scale"]):
        assert (cal[k].x_max, cal[k].x_min, cal[k].scale) == (xm, xn, sc), (k, cal[k], (xm, xn, sc))
    scales = T.static_scales_from(cal)
    prec = T.PrecisionConfig.from_scheme("W8A8", group_count=16, activation_static=True)
    emb = torch.from_numpy(g["embedding"]).cuda()
    x = emb[torch.from_numpy(batches[0]).cuda()]
    for li, w in enumerate(blocks):
        db = T.quantize_block(dict(w, num_heads=heads), prec)
        x = T.block_forward(x, db, prec, True, layer=li, static_scales=scales)
    hf = torch.empty_like(x)
    igemm.layer_norm_quantize(x, torch.from_numpy(g["final_gamma"]).cuda(), torch.from_numpy(g["final_beta"]).cuda(),
                              8, ln_out=hf)
    logits = T._matmul_seq(hf, emb, None).cpu().numpy()
    assert rel(logits, g["static_logits_b0"]) < TOL, rel(logits, g["static_logits_b0"])


def test_numpy_exp_on_device_is_np_exp():
    from paper_2206_01861_b200 import _native as N

    rng = np.random.default_rng(1)
    xs = np.concatenate([-rng.random(1 << 20) * 40, rng.uniform(-110, 90, 1 << 18),
                         [-np.inf, np.inf, -0.0, 88.72283935546875, -103.97208404541015625]]).astype(F32)
    xt = torch.from_numpy(xs).cuda()
    y = torch.empty_like(xt)
    N.call("zq_np_expf", xt.data_ptr(), xt.numel(), y.data_ptr(), N.stream_ptr())
    with np.errstate(all="ignore"):
        ref = np.exp(xs)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), ref.view(np.uint32))
