"""GPU parity: quantizers (K1 token-wise, K2 static, K3 group-wise, K4 LN+quant,
K5 GeLU+quant) vs the reference golden vectors and the numpy oracle.
Bar: bit-exact int8 payloads and float32 scales."""

import hashlib

import numpy as np
import pytest
import torch

from oracle import lowbit_oracle as O

pytestmark = pytest.mark.gpu
F32 = np.float32


@pytest.fixture(scope="module")
def zq():
    from paper_2206_01861_b200 import igemm, quant

    return quant, igemm


def h(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype == np.float32:
        return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.astype(np.float32).view(np.uint32))
    return a.shape == b.shape and np.array_equal(a, b)


def sha(*arrays):
    hh = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        hh.update(str(a.dtype).encode())
        hh.update(str(a.shape).encode())
        hh.update(a.tobytes())
    return hh.hexdigest()


def test_tokenwise_golden(zq, golden, golden_meta):
    quant, _ = zq
    for name in golden_meta["cases"]["tok"] + ["tok_kat"]:
        bits = 4 if name.endswith("_b4") else 8
        qa = quant.quantize_activation_tokenwise(golden[name + "_x"], bits)
        assert same_bits(h(qa.values), golden[name + "_q"]), name
        assert same_bits(h(qa.token_scales), golden[name + "_s"]), name


def test_tokenwise_padding_is_zero(zq):
    quant, _ = zq
    x = np.random.default_rng(0).standard_normal((5, 37)).astype(F32)
    qa = quant.quantize_activation_tokenwise(x, 8)
    store = qa.values.as_strided((5, qa.values.stride(0)), (qa.values.stride(0), 1))
    assert not h(store)[:, 37:].any()


def test_tokenwise_random_shapes_and_ties(zq):
    quant, _ = zq
    rng = np.random.default_rng(7)
    for i in range(60):
        t = int(rng.integers(1, 65))
        d = int(rng.integers(1, 4097))
        x = (rng.standard_normal((t, d)) * rng.uniform(0.01, 50)).astype(F32)
        if i % 3 == 0:
            x[0] = 0.0
        if i % 4 == 1:  # plant exact ties k+0.5 at the row's own scale
            s = np.asarray([O.compute_scale(r, 8) for r in x], np.float64)
            k = rng.integers(0, 127, (t, d)) + 0.5
            cand = (k * s[:, None]).astype(F32)
            ok = (cand.astype(np.float64) == k * s[:, None]) & (np.abs(cand) < np.abs(x).max(1, keepdims=True))
            x = np.where(ok & (rng.uniform(size=(t, d)) < 0.3), cand, x).astype(F32)
        bits = 4 if i % 5 == 0 else 8
        qa = quant.quantize_activation_tokenwise(x, bits)
        q_ref, s_ref = O.quantize_activation_tokenwise(x, bits)
        assert same_bits(h(qa.values), q_ref), (t, d, bits)
        assert same_bits(h(qa.token_scales), s_ref), (t, d, bits)


def test_tokenwise_c1_digest(zq, golden_meta):
    quant, _ = zq
    hh = golden_meta["hashes"]["c1"]
    x = O.Rng(1).gaussian((4096, 768), std=1.0)
    qa = quant.quantize_activation_tokenwise(x, 8)
    assert sha(h(qa.values)) == hh["xq_values"]
    assert sha(h(qa.token_scales)) == hh["xq_scales"]


def test_tokenwise_errors(zq):
    from paper_2206_01861_b200.errors import UsageError

    quant, _ = zq
    with pytest.raises(UsageError):
        quant.quantize_activation_tokenwise(np.ones((2, 3), F32), 16)
    with pytest.raises(ValueError):
        quant.quantize_activation_tokenwise(np.array([[1.0, np.nan]], F32), 8)
    with pytest.raises(ValueError):
        quant.quantize_activation_tokenwise(np.array([[1.0], [np.inf]], F32), 8)
    with pytest.raises(UsageError):
        quant.quantize_activation_tokenwise(np.ones((3,), F32), 8)


def test_static_golden(zq, golden, golden_meta):
    quant, _ = zq
    for name in golden_meta["cases"]["static"]:
        bits = 4 if name.endswith("_b4") else 8
        qa = quant.quantize_activation_static(golden[name + "_x"], float(golden[name + "_scale"][0]), bits)
        assert same_bits(h(qa.values), golden[name + "_q"]), name


def test_scalar_kats(zq):
    from paper_2206_01861_b200.errors import UsageError

    quant, _ = zq
    assert quant.quantize_value(1.0, 2.0 / 127.0, 8) == 64  # test_quant.py:86-88
    assert quant.quantize_value(-2.0, 2.0 / 127.0, 8) == -127
    assert quant.quantize_value(0.0, 0.37, 4) == 0
    assert quant.quantize_value(100.0, 0.01, 4) == 7 and quant.quantize_value(-100.0, 0.01, 4) == -7
    assert quant.compute_scale(np.array([0.5, -2.0, 1.0], F32), 8) == float(F32(2.0 / 127.0))
    assert quant.compute_scale(np.zeros(3, F32), 4) == 1.0
    with pytest.raises(ValueError):
        quant.quantize_value(float("inf"), 1.0, 8)
    with pytest.raises(UsageError):
        quant.quantize_value(1.0, 0.0, 8)
    with pytest.raises(UsageError):
        quant.compute_scale(np.array([], F32), 8)
    with pytest.raises(ValueError):
        quant.compute_scale(np.array([1.0, np.nan], F32), 8)


def test_negation_symmetry_and_monotone(zq):
    quant, _ = zq
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(5000) * 10).astype(F32)
    for bits in (4, 8):
        s = quant.compute_scale(x, bits)
        qp = h(quant.quantize_array(x, s, bits))
        qn = h(quant.quantize_array(-x, s, bits))
        assert np.array_equal(qn, -qp)
        xs = np.sort(x)
        q = h(quant.quantize_array(xs, 0.07, bits)).astype(np.int32)
        assert np.all(np.diff(q) >= 0)


def test_groupwise_golden(zq, golden, golden_meta):
    quant, _ = zq
    for name in golden_meta["cases"]["wq"]:
        g = int(name.split("_g")[1].split("_")[0])
        bits = 4 if name.endswith("_b4") else 8
        qm = quant.quantize_weight_groupwise(golden[name + "_w"], g, bits)
        assert same_bits(h(qm.values), golden[name + "_q"]), name
        assert same_bits(h(qm.group_scales), golden[name + "_gs"]), name
        assert same_bits(h(qm.row_scales()), golden[name + "_rs"]), name
        assert qm.group_layout == [tuple(v) for v in golden[name + "_layout"].tolist()], name
        if bits == 4:
            packed = h(qm.packed4)[:, : (qm.cols + 1) // 2]
            assert np.array_equal(O.unpack_int4(packed)[:, : qm.cols], golden[name + "_q"]), name


def test_groupwise_errors_and_c1(zq, golden_meta):
    from paper_2206_01861_b200.errors import UsageError

    quant, _ = zq
    with pytest.raises(UsageError):
        quant.quantize_weight_groupwise(np.ones((4, 2), F32), 5, 8)
    with pytest.raises(UsageError):
        quant.quantize_weight_groupwise(np.ones((4, 2), F32), 0, 8)
    with pytest.raises(ValueError):
        quant.quantize_weight_groupwise(np.array([[1.0, np.inf]], F32), 1, 8)
    hh = golden_meta["hashes"]["c1"]
    w = O.Rng(0).gaussian((3072, 768), std=0.02)
    qm = quant.quantize_weight_groupwise(w, 48, 8)
    assert sha(h(qm.values)) == hh["wq_values"] and sha(h(qm.group_scales)) == hh["wq_scales"]


def test_layer_norm_quantize_golden(zq, golden, golden_meta):
    _, igemm = zq
    for name in golden_meta["cases"]["fused"]:
        x, g, b = golden[name + "_x"], golden[name + "_gamma"], golden[name + "_beta"]
        ln = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        qa = igemm.layer_norm_quantize(x, g, b, 8, ln_out=ln)
        assert same_bits(h(ln), golden[name + "_ln"]), name
        assert same_bits(h(qa.values), golden[name + "_lnq"]), name
        assert same_bits(h(qa.token_scales), golden[name + "_lns"]), name


def test_layer_norm_residual_and_widths(zq):
    _, igemm = zq
    rng = np.random.default_rng(11)
    for d in (1, 5, 8, 64, 96, 100, 129, 300, 768, 1000, 1024, 3072, 4096, 6144, 8192):
        x = (rng.standard_normal((6, d)) * rng.uniform(0.2, 5)).astype(F32)
        r = (rng.standard_normal((6, d)) * 0.5).astype(F32)
        g = (1 + 0.1 * rng.standard_normal(d)).astype(F32)
        b = (0.1 * rng.standard_normal(d)).astype(F32)
        ln = torch.empty((6, d), dtype=torch.float32, device="cuda")
        qa = igemm.layer_norm_quantize(x, g, b, 8, residual=r, ln_out=ln)
        ref = O.layer_norm_numpy((x + r).astype(F32), g, b)
        assert same_bits(h(ln), ref), d
        q_ref, s_ref = O.quantize_activation_tokenwise(ref, 8)
        assert same_bits(h(qa.values), q_ref) and same_bits(h(qa.token_scales), s_ref), d


def test_ln_digest(zq, golden_meta):
    _, igemm = zq
    hh = golden_meta["hashes"]["ln_512x768"]
    xl = O.Rng(2).gaussian((512, 768), std=1.0)
    qa = igemm.layer_norm_quantize(xl, np.ones(768, F32), np.zeros(768, F32), 8)
    assert sha(h(qa.values)) == hh["q"] and sha(h(qa.token_scales)) == hh["s"]


def test_gelu_quantize_golden(zq, golden, golden_meta):
    _, igemm = zq
    for name in golden_meta["cases"]["fused"]:
        x = golden[name + "_x"]
        ge = torch.empty(x.shape, dtype=torch.float32, device="cuda")
        qa = igemm.gelu_quantize(x, 8, gelu_out=ge)
        assert same_bits(h(ge), golden[name + "_gelu"]), name
        assert same_bits(h(qa.values), golden[name + "_geq"]), name
        assert same_bits(h(qa.token_scales), golden[name + "_ges"]), name


def test_gelu_digest_and_large(zq, golden_meta):
    _, igemm = zq
    hh = golden_meta["hashes"]["gelu_256x3072"]
    xg = O.Rng(3).gaussian((256, 3072), std=1.0)
    ge = torch.empty(xg.shape, dtype=torch.float32, device="cuda")
    qa = igemm.gelu_quantize(xg, 8, gelu_out=ge)
    assert sha(h(ge)) == hh["gelu"]
    assert sha(h(qa.values)) == hh["q"] and sha(h(qa.token_scales)) == hh["s"]
    # NeoX FFN width, decode-sized batch
    x = (np.random.default_rng(5).standard_normal((16, 24576)) * 2).astype(F32)
    qa = igemm.gelu_quantize(x, 8)
    q_ref, s_ref = O.gelu_quantize(x, 8)
    assert same_bits(h(qa.values), q_ref) and same_bits(h(qa.token_scales), s_ref)


@pytest.mark.parametrize("std", [0.3, 1.0, 3.0, 10.0])
def test_gelu_quantize_fast_path_exact(zq, std):
    """The q/scale-only GeLU path (fp32 bracket + exact f64 fallback) must equal
    quantize(gelu_f64(x)) bit for bit, including heavy negative tails (< -3,
    where the reference's 1 + erf cancellation rules) and zero rows."""
    _, igemm = zq
    rng = np.random.default_rng(int(std * 10))
    for (t, d) in [(512, 3072), (64, 4096), (16, 24576), (300, 1024), (3, 16384), (1, 4096), (5, 6004)]:
        x = (rng.standard_normal((t, d)) * std).astype(F32)
        if t >= 3:
            x[0] = 0.0
            x[1, : d // 2] = -abs(x[1, : d // 2]) - 3.0
            x[2] = -np.abs(x[2])
        qa = igemm.gelu_quantize(x, 8)
        q_ref, s_ref = O.gelu_quantize(x, 8)
        assert same_bits(h(qa.token_scales), s_ref), (t, d, std)
        assert same_bits(h(qa.values), q_ref), (t, d, std)


def test_gelu_quantize_wide_rows(zq):
    """Rows wider than 8 chunks x 128 threads with too many rows for a cluster split
    (NeoX FFN prefill: 24576 columns, one CTA of 768 threads per row)."""
    _, igemm = zq
    x = (np.random.default_rng(41).standard_normal((320, 24576)) * 1.5).astype(F32)
    qa = igemm.gelu_quantize(x, 8)
    q_ref, s_ref = O.gelu_quantize(x, 8)
    assert same_bits(h(qa.token_scales), s_ref)
    assert same_bits(h(qa.values), q_ref)


def test_ln_uniform_and_generic_paths_agree(zq):
    """Balanced-tree (uniform) and generic plan LN kernels vs numpy for widths
    around the uniform/non-uniform boundary."""
    _, igemm = zq
    rng = np.random.default_rng(21)
    for d in (256, 512, 768, 1024, 2048, 3072, 4096, 6144, 640, 1000, 1536, 2304):
        x = (rng.standard_normal((37, d)) * 2 + 0.5).astype(F32)
        g = (1 + 0.1 * rng.standard_normal(d)).astype(F32)
        b = (0.1 * rng.standard_normal(d)).astype(F32)
        ln = torch.empty((37, d), dtype=torch.float32, device="cuda")
        qa = igemm.layer_norm_quantize(x, g, b, 8, ln_out=ln)
        ref = O.layer_norm_numpy(x, g, b)
        assert same_bits(h(ln), ref), d
        q_ref, s_ref = O.quantize_activation_tokenwise(ref, 8)
        assert same_bits(h(qa.values), q_ref) and same_bits(h(qa.token_scales), s_ref), d


def test_gelu_estimate_within_its_bracket(zq):
    """The bracket the fast GeLU quantizer relies on: |est - gelu_ref| <= bound * |gelu_ref|
    on a dense grid over [-5.5, 12] (gelu_ref = the exact f32 restatement of
    tensor.py:76-83, pinned to scipy in tests/test_oracle_golden.py)."""
    from paper_2206_01861_b200 import _native as N

    x = np.concatenate([np.linspace(-5.5, 12.0, 400_001), np.linspace(-0.01, 0.01, 20_001),
                        np.linspace(-5.5, -3.0, 50_001)]).astype(F32)
    xt = torch.from_numpy(x).cuda()
    est = torch.empty_like(xt)
    bnd = torch.empty_like(xt)
    N.call("zq_gelu_estimate", xt.data_ptr(), x.size, est.data_ptr(), bnd.data_ptr(), N.stream_ptr())
    ref = O.gelu(x).astype(np.float64)
    e = h(est).astype(np.float64)
    b = h(bnd).astype(np.float64)
    nz = ref != 0
    rel = np.abs(e[nz] - ref[nz]) / np.abs(ref[nz])
    assert np.all(rel <= b[nz]), (rel.max(), x[nz][np.argmax(rel - b[nz])])
    assert rel.max() <= 2.0 ** -17, rel.max()  # the bracket gelu_quant_kernel assumes
    assert np.all(e[~nz] == 0.0)


def test_float64_inputs_follow_the_reference(zq):
    """compute_scale / quantize_array / quantize_value read float64 input in
    float64 (quant.py:80-118); the other quantizers cast to float32 first
    (as_f32, quant.py:242, :261, :279) instead of rejecting it."""
    from paper_2206_01861_b200 import quant

    assert quant.quantize_value(0.1, 0.01, 8) == 10           # 0.1 / 0.01 in f64 = 10.000000000000002
    assert quant.quantize_value(1.0, 2.0 / 127.0, 8) == 64    # exact f64 tie 63.5 -> away from zero
    assert quant.quantize_value(-1.0, 2.0 / 127.0, 8) == -64
    x = np.array([0.1, -0.25000000000000006, 1e-300, 3.0, -1e300, 0.0])
    ref = O.quantize_array(x, 0.05, 8)
    assert np.array_equal(h(quant.quantize_array(x, 0.05, 8)), ref)
    v = np.array([0.30000000000000004, -0.1, 1e-320])
    assert quant.compute_scale(v, 8) == O.compute_scale(v, 8) == float(np.float32(0.30000000000000004 / 127))
    assert quant.compute_scale(np.array([1, -254, 3]), 8) == 2.0       # integer input -> exact f64
    rng = np.random.default_rng(0)
    w64 = rng.standard_normal((64, 48)) * 0.02
    qm = quant.quantize_weight_groupwise(w64, 4, 8)
    vals, gs, _ = O.quantize_weight_groupwise(w64.astype(np.float32), 4, 8)
    assert np.array_equal(h(qm.values), vals) and np.array_equal(h(qm.group_scales), gs)
    x64 = rng.standard_normal((7, 33))
    qa = quant.quantize_activation_tokenwise(x64, 8)
    q_ref, s_ref = O.quantize_activation_tokenwise(x64.astype(np.float32), 8)
    assert np.array_equal(h(qa.values), q_ref) and np.array_equal(h(qa.token_scales), s_ref)
    with pytest.raises(ValueError):
        quant.quantize_array(np.array([1.0, np.inf]), 0.1, 8)
    with pytest.raises(ValueError):
        quant.compute_scale(np.array([np.nan]), 8)


@pytest.mark.parametrize("shape", [(16, 6144), (2048, 768), (33, 1000), (5, 3), (7, 4096)])
def test_quantize_with_absmax_matches_tokenwise(shape):
    """zq_quantize_with_absmax (the TP row-parallel quantizer, given the all-reduced
    row max) == the token-wise quantizer when given the local max, and == the
    oracle's RHAFZ with the scale of a larger (other-rank) max; planted ties."""
    from paper_2206_01861_b200 import _native as N
    from paper_2206_01861_b200 import quant

    rows, cols = shape
    rng = np.random.default_rng(rows * 7 + cols)
    x = rng.standard_normal((rows, cols)).astype(np.float32)
    x[:, 0] = 127.0 / 2 * np.float32(0.03)  # candidates for exact half-way cases
    xt = torch.from_numpy(x).cuda()
    ld = (cols + 15) // 16 * 16
    amax = torch.from_numpy(np.abs(x).max(axis=1).astype(np.float32)).cuda()
    for mult in (1.0, 1.7):
        am = amax * mult
        q = torch.empty(rows, ld, dtype=torch.int8, device="cuda")
        s = torch.empty(rows, device="cuda")
        N.call("zq_quantize_with_absmax", xt.data_ptr(), rows, cols, cols, am.data_ptr(), 8, q.data_ptr(), ld,
               s.data_ptr(), N.stream_ptr())
        sref = np.array([np.float32(np.float64(v) / 127.0) for v in am.cpu().numpy()], dtype=np.float32)
        assert np.array_equal(s.cpu().numpy().view(np.uint32), sref.view(np.uint32)), (shape, mult)
        qref = np.stack([O.quantize_array(x[i], float(sref[i]), 8) for i in range(rows)])
        assert np.array_equal(q[:, :cols].cpu().numpy(), qref), (shape, mult)
        assert not q[:, cols:].any()
        if mult == 1.0:
            qa = quant.quantize_activation_tokenwise(xt, 8)
            assert torch.equal(qa.values, q[:, :cols]) and torch.equal(qa.token_scales, s)


@pytest.mark.parametrize("t", [300, 16])
def test_gelu_quantize_far_negative_tail_small_rows(zq, t):
    """Elements below -5.5 take the estimate at -5.5 (~ -1.04e-7; the reference
    has |g| <= 1.1e-7 there): they must still quantize to 0, and never decide the
    row max, for row maxima around the 1e-5 candidate and 3e-5 degenerate-row
    thresholds; elements just above -5.5 go through the bracket as usual.  300
    rows: one CTA per row; 16 rows: rows split over a CTA cluster."""
    _, igemm = zq
    rng = np.random.default_rng(7 + t)
    d = 3072
    x = rng.uniform(-12.0, -5.5, (t, d)).astype(F32)
    x[:, 7] = -5.5
    x[:, 8] = np.nextafter(F32(-5.5), F32(0))
    x[:, 9] = np.nextafter(F32(-5.5), F32(-10))
    x[:, 10:40] = rng.uniform(-5.5, -4.0, (t, 30)).astype(F32)
    # the row's only positive element sets the row max: ~GeLU(x) = x / 2 for tiny x
    peaks = np.array([6.2e-5, 6.0e-5, 5.0e-5, 2.4e-5, 1.0e-5, 2e-6, 1e-3, 0.5], dtype=F32)
    x[:, 100] = peaks[np.arange(t) % len(peaks)]
    qa = igemm.gelu_quantize(x, 8)
    q_ref, s_ref = O.gelu_quantize(x, 8)
    assert same_bits(h(qa.token_scales), s_ref)
    assert same_bits(h(qa.values), q_ref)
