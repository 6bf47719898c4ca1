"""CPU: pin the numpy oracle (oracle/lowbit_oracle.py) against the golden
vectors produced by the real reference (oracle/make_golden.py)."""

import hashlib

import numpy as np
import pytest

from oracle import lowbit_oracle as O

F32 = np.float32


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_rng_stream(golden):
    r = O.Rng(1234)
    assert np.array_equal(r._raw(4), golden["rng_u64"])
    assert np.array_equal(O.Rng(7).gaussian((3, 5), std=0.5), golden["rng_gauss"])
    assert np.array_equal(O.Rng(9).integers(1000, 16), golden["rng_ints"])


def test_tokenwise(golden, golden_meta):
    for name in golden_meta["cases"]["tok"] + ["tok_kat"]:
        bits = 4 if name.endswith("_b4") else 8
        q, s = O.quantize_activation_tokenwise(golden[name + "_x"], bits)
        assert np.array_equal(q, golden[name + "_q"]), name
        assert np.array_equal(s.view(np.uint32), golden[name + "_s"].view(np.uint32)), name


def test_tokenwise_kat():
    x = np.zeros((2, 4), dtype=F32)
    x[0, 0] = 35.0
    x[1, 2] = -8.0
    _, s = O.quantize_activation_tokenwise(x, 8)
    assert s[0] == F32(35.0 / 127.0) and s[1] == F32(8.0 / 127.0)  # test_quant.py:206-212
    assert O.quantize_array(np.array([1.0]), 2.0 / 127.0, 8)[0] == 64  # tie, test_quant.py:86-88
    assert O.quantize_array(np.array([-2.0]), 2.0 / 127.0, 8)[0] == -127
    assert O.quantize_array(np.array([100.0]), 0.01, 4)[0] == 7


def test_static(golden, golden_meta):
    for name in golden_meta["cases"]["static"]:
        bits = 4 if name.endswith("_b4") else 8
        q = O.quantize_activation_static(golden[name + "_x"], float(golden[name + "_scale"][0]), bits)
        assert np.array_equal(q, golden[name + "_q"]), name


def test_groupwise(golden, golden_meta):
    for name in golden_meta["cases"]["wq"]:
        g = int(name.split("_g")[1].split("_")[0])
        bits = 4 if name.endswith("_b4") else 8
        q, gs, lay = O.quantize_weight_groupwise(golden[name + "_w"], g, bits)
        assert np.array_equal(q, golden[name + "_q"]), name
        assert np.array_equal(gs, golden[name + "_gs"]), name
        assert np.array_equal(np.asarray(lay), golden[name + "_layout"]), name
        assert np.array_equal(O.expand_row_scales(gs, lay), golden[name + "_rs"]), name
    q, gs, lay = O.quantize_weight_groupwise(golden["wq_kat_w"], 2, 8)
    assert lay == [(0, 2), (2, 2)] and gs[0] == F32(10 / 127) and gs[1] == F32(0.1 / 127)


def test_linear(golden, golden_meta):
    for name in golden_meta["cases"]["lin"]:
        t, d, n, g, wbits = (int(v) for v in golden[name + "_meta"])
        x, w = golden[name + "_x"], golden[name + "_w"]
        bias = golden.get(name + "_bias")
        wv, gs, lay = O.quantize_weight_groupwise(w, g, wbits)
        rs = O.expand_row_scales(gs, lay)
        xv, s = O.quantize_activation_tokenwise(x, 8)
        assert np.array_equal(O.igemm(xv, wv), golden[name + "_acc"]), name
        assert np.array_equal(O.igemm_int64(xv, wv), golden[name + "_acc"]), name
        dyn = O.quantized_linear(x, wv, rs, bias, "dynamic", w_bits=wbits)
        assert np.array_equal(dyn.view(np.uint32), golden[name + "_dyn"].view(np.uint32)), name
        sta = O.quantized_linear(x, wv, rs, bias, "static", float(golden[name + "_sscale"][0]), w_bits=wbits)
        assert np.array_equal(sta.view(np.uint32), golden[name + "_sta"].view(np.uint32)), name
        if name + "_full" in golden:
            full = O.quantized_linear(x, wv, rs, bias, "full")
            assert np.array_equal(full, golden[name + "_full"]), name


def test_fused_ln_gelu(golden, golden_meta):
    for name in golden_meta["cases"]["fused"]:
        x, g, b = golden[name + "_x"], golden[name + "_gamma"], golden[name + "_beta"]
        ln = O.layer_norm(x, g, b)  # explicit pairwise restatement
        assert np.array_equal(ln.view(np.uint32), golden[name + "_ln"].view(np.uint32)), name
        q, s = O.quantize_activation_tokenwise(ln, 8)
        assert np.array_equal(q, golden[name + "_lnq"]) and np.array_equal(s, golden[name + "_lns"]), name
        ge = O.gelu(x)
        assert np.array_equal(ge.view(np.uint32), golden[name + "_gelu"].view(np.uint32)), name
        q, s = O.gelu_quantize(x, 8)
        assert np.array_equal(q, golden[name + "_geq"]) and np.array_equal(s, golden[name + "_ges"]), name


@pytest.mark.parametrize("d", [1, 7, 8, 12, 96, 128, 130, 300, 768, 1024, 4096, 6144, 24576])
def test_pairwise_restatement_matches_numpy(d, np_rng):
    for _ in range(5):
        x = (np_rng.standard_normal(d) * np_rng.uniform(0.1, 100)).astype(F32)
        assert O.pairwise_sum_f32(x) == x.sum(dtype=F32)


def test_block_forward(golden):
    names = ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh")
    blk = {k[len("block_"):]: v for k, v in golden.items() if k.startswith("block_") and
           not k.startswith("block_W") and k != "block_x"}
    for scheme, (mb, fb, am) in {"W8A8": (8, 8, "int8"), "W4_8A8": (8, 4, "int8"),
                                 "W8A8_16": (8, 8, "int8_attn_full")}.items():
        qb = O.quantize_block(blk, mb, fb, O.default_group_count(64))
        for causal in (0, 1):
            y = O.block_forward(golden["block_x"], qb, 4, bool(causal), am)
            ref = golden[f"block_{scheme}_c{causal}_y"]
            assert np.array_equal(y, ref), (scheme, causal)
    assert set(names) <= set(blk)


def test_c1_digests(golden_meta):
    h = golden_meta["hashes"]["c1"]
    w = O.Rng(0).gaussian((3072, 768), std=0.02)
    x = O.Rng(1).gaussian((4096, 768), std=1.0)
    assert sha(w) == h["w"] and sha(x) == h["x"]
    wv, gs, lay = O.quantize_weight_groupwise(w, 48, 8)
    assert sha(wv) == h["wq_values"] and sha(gs) == h["wq_scales"]
    xv, s = O.quantize_activation_tokenwise(x, 8)
    assert sha(xv) == h["xq_values"] and sha(s) == h["xq_scales"]
    acc = O.igemm(xv, wv)
    assert sha(acc) == h["acc"]
    assert sha(O.dequant_epilogue(acc, s, O.expand_row_scales(gs, lay))) == h["out_f32"]


def test_fused_digests(golden_meta):
    h = golden_meta["hashes"]
    xl = O.Rng(2).gaussian((512, 768), std=1.0)
    q, s = O.layer_norm_quantize(xl, np.ones(768, F32), np.zeros(768, F32), 8)
    assert sha(xl) == h["ln_512x768"]["x"] and sha(q) == h["ln_512x768"]["q"] and sha(s) == h["ln_512x768"]["s"]
    xg = O.Rng(3).gaussian((256, 3072), std=1.0)
    q, s = O.gelu_quantize(xg, 8)
    assert sha(q) == h["gelu_256x3072"]["q"] and sha(s) == h["gelu_256x3072"]["s"]


def test_int4_pack_roundtrip(np_rng):
    v = np_rng.integers(-7, 8, (5, 64)).astype(np.int8)
    assert np.array_equal(O.unpack_int4(O.pack_int4(v)), v)


def test_error_taxonomy():
    with pytest.raises(O.UsageError):
        O.quantize_activation_tokenwise(np.ones((2, 2), F32), 16)
    with pytest.raises(ValueError):
        O.quantize_activation_tokenwise(np.array([[1.0, np.nan]], F32), 8)
    with pytest.raises(O.UsageError):
        O.check_overflow_guard(140000, 8, 8)
    O.check_overflow_guard(133000, 8, 8)
    with pytest.raises(O.UsageError):
        O.group_layout_for(4, 5)


def test_cephes_erf_is_scipy_erf():
    """Pins the f64 erf the GPU GeLU restates (csrc/zq_quant.cu cephes_erf)."""
    from scipy.special import erf

    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.standard_normal(20000) * 3, rng.uniform(-8, 8, 20000),
                         rng.uniform(-1, 1, 5000), rng.uniform(-30, 30, 2000), [0.0, 1.0, -1.0, 8.0]])
    ref = erf(xs)
    mine = np.asarray([O.cephes_erf(float(v)) for v in xs])
    assert np.array_equal(mine, ref)


def test_numpy_expf_restatement_is_np_exp():
    """Pins the float32 exp the calibration forward restates (numpy's SIMD
    simd_exp_f32; csrc/zq_calib.cu np_expf): identical to np.exp on float32,
    although 39% of np.exp's results are not the correctly rounded exp."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([-rng.random(400000) * 30, rng.uniform(-104, -80, 100000), rng.uniform(-5, 5, 100000),
                         [-np.inf, -200.0, -103.97208404541015625, -87.3, -0.0, 0.0, 88.72283935546875, 50.0]])
    xs = xs.astype(F32)
    with np.errstate(all="ignore"):
        ref = np.exp(xs)
    assert np.array_equal(O.numpy_expf(xs), ref)
    assert (O.numpy_expf(xs[:1000]) != np.exp(xs[:1000].astype(np.float64)).astype(F32)).any()


def test_oracle_calibration_matches_reference_golden():
    """oracle.calibrate_model (evaluate.py:168-196 restated) reproduces the
    reference's own calibration of the fixture model bit for bit."""
    import os

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "calibration.npz"))
    blocks = [{n[3:]: g[n] for n in g.files if n.startswith(f"l{li}_")} for li in range(int(g["layers"]))]
    batches = [g[f"batch{i}"] for i in range(3)]
    cal = O.calibrate_model(g["embedding"], blocks, int(g["num_heads"]), True, batches)
    assert list(cal) == list(g["site_keys"])
    for k, xm, xn, sc in zip(g["site_keys"], g["site_xmax"], g["site_xmin"], g["site_scale"]):
        assert cal[k] == (xm, xn, sc), (k, cal[k], (xm, xn, sc))
