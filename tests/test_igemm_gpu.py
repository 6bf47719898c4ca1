"""GPU parity: tcgen05 kind::i8 igemm (bit-exact int32), fused dequant epilogue
(bit-exact float32; fp16/bf16 = RN cast of the exact f32, checked exactly and
against a 1e-3 relative tolerance), W4A8, FullAct, and the reference KATs
(pkg/tests/test_igemm.py)."""

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


def bits_eq(a, b):
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def make_qmat(quant, values, scales=(1.0,), layout=None, bits=8):
    v = np.asarray(values, dtype=np.int8)
    n, m = v.shape
    full = torch.zeros((n, quant.round_up(max(m, 1), 32)), dtype=torch.int8, device="cuda")
    full[:, :m] = torch.from_numpy(v).cuda()
    gs = torch.tensor(np.asarray(scales, F32), device="cuda")
    layout = layout or [(0, n)]
    return quant.QuantizedMatrix(values=full[:, :m], bits=bits, group_scales=gs, group_layout=layout)


def make_qact(quant, values, scales=None, static=None, bits=8):
    v = torch.from_numpy(np.asarray(values, dtype=np.int8)).cuda()
    if static is not None:
        return quant.QuantizedActivation(values=v, bits=bits, static_scale=static)
    if scales is None:
        scales = np.ones(v.shape[0], F32)
    return quant.QuantizedActivation(values=v, bits=bits, token_scales=torch.tensor(np.asarray(scales, F32)).cuda())


def test_forced_arithmetic(zq):
    quant, igemm = zq
    acc = igemm.igemm(make_qact(quant, [[1, 2]]), make_qmat(quant, [[3, 4]]))
    assert acc.acc.dtype == torch.int32 and h(acc.acc).tolist() == [[11]]


def test_zero_activation(zq):
    quant, igemm = zq
    acc = igemm.igemm(make_qact(quant, np.zeros((3, 5))), make_qmat(quant, np.arange(10).reshape(2, 5) - 5))
    assert not h(acc.acc).any()


@pytest.mark.parametrize("seed", range(4))
def test_igemm_random_shapes(zq, seed):
    quant, igemm = zq
    rng = np.random.default_rng(100 + seed)
    for _ in range(12):
        t, d, n = int(rng.integers(1, 300)), int(rng.integers(1, 700)), int(rng.integers(1, 600))
        xv = rng.integers(-127, 128, (t, d))
        wv = rng.integers(-127, 128, (n, d))
        acc = igemm.igemm(make_qact(quant, xv), make_qmat(quant, wv))
        assert np.array_equal(h(acc.acc), O.igemm(xv.astype(np.int8), wv.astype(np.int8))), (t, d, n)


@pytest.mark.parametrize("shape", [(128, 128, 256), (4096, 768, 3072), (256, 3072, 768),
                                   (16, 6144, 6144), (300, 24576, 128), (1000, 4096, 640)])
def test_igemm_large_exact(zq, shape):
    quant, igemm = zq
    t, d, n = shape
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    xv = torch.randint(-127, 128, (t, d), dtype=torch.int8, device="cuda", generator=g)
    wv = torch.randint(-127, 128, (n, d), dtype=torch.int8, device="cuda", generator=g)
    xq = quant.QuantizedActivation(values=xv, bits=8, token_scales=torch.ones(t, device="cuda"))
    wq = make_qmat(quant, h(wv))
    acc = h(igemm.igemm(xq, wq).acc)
    ref = O.igemm(h(xv), h(wv))
    assert np.array_equal(acc, ref)


def test_bit_identical_across_runs(zq):
    quant, igemm = zq
    rng = np.random.default_rng(1)
    xv, wv = rng.integers(-127, 128, (160, 640)), rng.integers(-127, 128, (320, 640))
    first = h(igemm.igemm(make_qact(quant, xv), make_qmat(quant, wv)).acc)
    for _ in range(3):
        assert np.array_equal(h(igemm.igemm(make_qact(quant, xv), make_qmat(quant, wv)).acc), first)


def test_shape_mismatch_and_guard(zq):
    from paper_2206_01861_b200.errors import ShapeError, UsageError

    quant, igemm = zq
    with pytest.raises(ShapeError):
        igemm.igemm(make_qact(quant, np.zeros((1, 3))), make_qmat(quant, np.zeros((2, 4))))
    igemm.check_overflow_guard(133000, 8, 8)
    with pytest.raises(UsageError):
        igemm.check_overflow_guard(140000, 8, 8)
    with pytest.raises(UsageError):
        igemm.igemm(make_qact(quant, np.zeros((1, 150000))), make_qmat(quant, np.zeros((1, 150000))))


def test_epilogue_kats(zq):
    quant, igemm = zq
    acc = igemm.IntAccumulator(acc=torch.tensor([[11]], dtype=torch.int32, device="cuda"))
    out = igemm.dequant_epilogue(acc, np.array([0.5], F32), make_qmat(quant, [[1]], scales=[0.25]))
    assert abs(h(out)[0, 0] - 1.375) < 1e-7
    acc = igemm.IntAccumulator(acc=torch.zeros((2, 3), dtype=torch.int32, device="cuda"))
    bias = np.array([1.0, -2.0, 3.0], F32)
    out = igemm.dequant_epilogue(acc, np.ones(2, F32), make_qmat(quant, np.ones((3, 4)), scales=[0.1]), bias)
    assert np.array_equal(h(out), np.tile(bias, (2, 1)))
    acc = igemm.IntAccumulator(acc=torch.tensor([[10, 10]], dtype=torch.int32, device="cuda"))
    w = make_qmat(quant, np.ones((2, 1)), scales=[1.0, 3.0], layout=[(0, 1), (1, 1)])
    assert h(igemm.dequant_epilogue(acc, np.array([2.0], F32), w)).tolist() == [[20.0, 60.0]]


def test_golden_linear(zq, golden, golden_meta):
    """Every golden case: igemm, dynamic and static quantized_linear bit-exact."""
    quant, igemm = zq
    for name in golden_meta["cases"]["lin"]:
        t, d, n, g, wbits = (int(v) for v in golden[name + "_meta"])
        x, w = golden[name + "_x"], golden[name + "_w"]
        bias = golden.get(name + "_bias")
        wq = quant.quantize_weight_groupwise(w, g, wbits)
        xq = quant.quantize_activation_tokenwise(x, 8)
        assert np.array_equal(h(igemm.igemm(xq, wq).acc), golden[name + "_acc"]), name
        dyn = igemm.quantized_linear(x, wq, bias, igemm.DynamicAct(8))
        assert bits_eq(h(dyn), golden[name + "_dyn"]), name
        sta = igemm.quantized_linear(x, wq, bias, igemm.StaticAct(float(golden[name + "_sscale"][0]), 8))
        assert bits_eq(h(sta), golden[name + "_sta"]), name
        if name + "_full" in golden:
            full = igemm.quantized_linear(x, wq, bias, igemm.FullAct())
            assert bits_eq(h(full), golden[name + "_full"]), name


@pytest.mark.parametrize("wbits", [8, 4])
@pytest.mark.parametrize("shape", [(4096, 768, 3072, 48), (1024, 1024, 4096, 64), (16, 4096, 4096, 128),
                                   (200, 3072, 768, 48), (33, 100, 70, 7)])
def test_fused_linear_vs_oracle(zq, shape, wbits):
    quant, igemm = zq
    t, d, n, g = shape
    rng = np.random.default_rng(t + d + n)
    x = (rng.standard_normal((t, d))).astype(F32)
    w = (rng.standard_normal((n, d)) * 0.02).astype(F32)
    bias = (rng.standard_normal(n) * 0.1).astype(F32)
    wq = quant.quantize_weight_groupwise(w, g, wbits)
    out = h(igemm.quantized_linear(x, wq, bias, igemm.DynamicAct(8)))
    wv, gs, lay = O.quantize_weight_groupwise(w, g, wbits)
    ref = O.quantized_linear(x, wv, O.expand_row_scales(gs, lay), bias, "dynamic", w_bits=wbits)
    assert bits_eq(out, ref)
    # half outputs: RN cast of the exact f32 result, and within 1e-3 relative
    for dt in (torch.float16, torch.bfloat16):
        o16 = igemm.quantized_linear(x, wq, bias, igemm.DynamicAct(8), out_dtype=dt)
        exact = torch.from_numpy(ref).to(dt)
        assert torch.equal(o16.cpu(), exact)
        rel = np.linalg.norm(o16.float().cpu().numpy() - ref) / np.linalg.norm(ref)
        assert rel < (1e-3 if dt == torch.float16 else 8e-3)


def test_no_dequant_materialisation(zq, monkeypatch):
    """test_igemm.py:188-199: the fused path never calls dequantize()."""
    quant, igemm = zq
    rng = np.random.default_rng(2)
    x = rng.standard_normal((4, 16)).astype(F32)
    wq = quant.quantize_weight_groupwise(rng.standard_normal((4, 16)).astype(F32), 2, 8)

    def boom(self):
        raise AssertionError("fused path materialized a dequantized matrix")

    monkeypatch.setattr(quant.QuantizedMatrix, "dequantize", boom)
    monkeypatch.setattr(quant.QuantizedActivation, "dequantize", boom)
    igemm.quantized_linear(x, wq, None, igemm.DynamicAct(8))
    igemm.quantized_linear(x, wq, None, igemm.StaticAct(0.05, 8))


def test_scale_linearity_power_of_two(zq):
    quant, igemm = zq
    rng = np.random.default_rng(4)
    xv, wv = rng.integers(-127, 128, (4, 16)), rng.integers(-127, 128, (8, 16))
    w = make_qmat(quant, wv, scales=[0.37])
    acc = igemm.igemm(make_qact(quant, xv), w)
    s = rng.uniform(0.01, 1, 4).astype(F32)
    base = h(igemm.dequant_epilogue(acc, s, w))
    doubled = h(igemm.dequant_epilogue(acc, s * F32(2.0), w))
    assert np.array_equal(doubled, base * F32(2.0))


@pytest.mark.parametrize("shape", [(1, 4096, 4096), (16, 4096, 12288), (33, 16384, 4096), (64, 768, 3072),
                                   (7, 6144, 3000), (16, 24576, 6144), (2, 200, 300)])
def test_skinny_decode_gemm_exact(zq, shape):
    """M <= 64 runs the split-K swap-AB kernel (cluster DSMEM reduction): the int32
    accumulators and the fused f32 epilogue must stay bit-exact."""
    quant, igemm = zq
    t, d, n = shape
    rng = np.random.default_rng(sum(shape))
    xv = rng.integers(-127, 128, (t, d)).astype(np.int8)
    wv = rng.integers(-127, 128, (n, d)).astype(np.int8)
    xa, wm = make_qact(quant, xv, scales=rng.random(t).astype(F32) + 0.01), make_qmat(quant, wv, scales=(0.003,))
    acc = igemm.igemm(xa, wm)
    ref_acc = O.igemm(xv, wv)
    assert np.array_equal(h(acc.acc), ref_acc), shape
    bias = rng.standard_normal(n).astype(F32)
    out = igemm.fused_linear(xa, wm, bias)
    ref = O.dequant_epilogue(ref_acc, h(xa.token_scales), np.full(n, F32(0.003)), bias)
    assert bits_eq(h(out), ref), shape


@pytest.mark.parametrize("shape", [(4096, 768, 768), (4096, 768, 3072), (300, 768, 768), (1000, 1024, 1024),
                                   (600, 3072, 768)])
def test_fused_linear_ln_quantize_matches_unfused(zq, shape):
    """zq_linear_ln_quantize (GEMM + residual + LN + quantize in one kernel, row
    statistics exchanged across CTAs) == zq_linear then zq_layer_norm_quantize,
    bit for bit, over repeated launches sharing one workspace."""
    from paper_2206_01861_b200 import _native as N

    quant, igemm = zq
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    xa = make_qact(quant, rng.integers(-127, 128, (m, k)), scales=(rng.random(m) * 0.05 + 0.01).astype(F32))
    w = quant.quantize_weight_groupwise((rng.standard_normal((n, k)) * 0.02).astype(F32), 16, 8)
    bias = torch.from_numpy((rng.standard_normal(n) * 0.1).astype(F32)).cuda()
    g = torch.from_numpy((1 + 0.1 * rng.standard_normal(n)).astype(F32)).cuda()
    b = torch.from_numpy((0.1 * rng.standard_normal(n)).astype(F32)).cuda()
    leaf = n
    while leaf > 128:
        leaf //= 2
    nt = n // (2 * leaf)
    ws = torch.zeros(4 * ((m + 255) // 256) + 16 + 12 * m * nt + 64, dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = xa.gemm_operand()
    wp, ldw, wb = w.weight_operand()
    for it in range(3):
        res = torch.from_numpy(rng.standard_normal((m, n)).astype(F32)).cuda()
        y = torch.empty(m, n, device="cuda")
        q = quant.padded_int8(m, n)
        s = torch.empty(m, device="cuda")
        N.call("zq_linear_ln_quantize", a.data_ptr(), a.stride(0), xa.token_scales.data_ptr(), wp, ldw, wb,
               w.row_scales().data_ptr(), bias.data_ptr(), m, n, k, res.data_ptr(), g.data_ptr(), b.data_ptr(),
               1e-5, 8, y.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(), ws.data_ptr(), ws.numel(),
               flag.data_ptr(), N.stream_ptr())
        f = igemm.fused_linear(xa, w, bias)
        y_ref = torch.empty(m, n, device="cuda")
        qa = igemm.layer_norm_quantize(res, g, b, 8, residual=f, ln_out=y_ref)
        assert bits_eq(h(y), h(y_ref)), (shape, it)
        assert np.array_equal(h(q), h(qa.values)) and bits_eq(h(s), h(qa.token_scales)), (shape, it)
    assert int(flag.item()) == 0


@pytest.mark.parametrize("shape", [(1, 1024, 4096), (8, 4096, 1024), (16, 4096, 16384), (64, 768, 3072), (5, 160, 200)])
def test_skinny_decode_gemm_w4_exact(zq, shape):
    """W4A8 at decode sizes: packed INT4 tiles unpacked in smem by the skinny kernel."""
    quant, igemm = zq
    t, d, n = shape
    rng = np.random.default_rng(7 * sum(shape))
    xv = rng.integers(-127, 128, (t, d)).astype(np.int8)
    wv = rng.integers(-7, 8, (n, d)).astype(np.int8)
    xa = make_qact(quant, xv, scales=rng.random(t).astype(F32) + 0.01)
    wm = make_qmat(quant, wv, scales=(0.01,), bits=4)
    acc = igemm.igemm(xa, wm)
    ref_acc = O.igemm(xv, wv)
    assert np.array_equal(h(acc.acc), ref_acc), shape
    out = igemm.fused_linear(xa, wm, None)
    assert bits_eq(h(out), O.dequant_epilogue(ref_acc, h(xa.token_scales), np.full(n, F32(0.01)), None)), shape


@pytest.mark.parametrize("shape", [(16, 4096, 12288), (16, 6144, 24576), (16, 24576, 6144), (1, 4096, 4096),
                                   (33, 6144, 3000), (8, 1024, 3072), (64, 768, 768), (3, 200, 300)])
def test_streamk_decode_gemm_exact(zq, shape):
    """zq_linear_ws (M <= 64, int8 weights): the stream-K skinny kernel (k-block
    units split evenly over the SMs, int32 partials added in a workspace, the
    last contributor of a tile dequantizes) is bit-exact, over repeated launches
    on one workspace (each launch must leave it zeroed), for f32 and f16 outputs."""
    from paper_2206_01861_b200 import _native as N

    quant, igemm = zq
    t, d, n = shape
    rng = np.random.default_rng(sum(shape) + 7)
    xv = rng.integers(-127, 128, (t, d)).astype(np.int8)
    wv = rng.integers(-127, 128, (n, d)).astype(np.int8)
    xa, wm = make_qact(quant, xv, scales=rng.random(t).astype(F32) + 0.01), make_qmat(quant, wv, scales=(0.003,))
    bias = torch.from_numpy(rng.standard_normal(n).astype(F32)).cuda()
    ref_acc = O.igemm(xv, wv)
    ref = O.dequant_epilogue(ref_acc, h(xa.token_scales), np.full(n, F32(0.003)), h(bias))
    nbytes = int(N.load().zq_linear_ws_bytes(t, n))
    ws = torch.zeros(nbytes // 4, dtype=torch.int32, device="cuda")
    a = xa.gemm_operand()
    wp, ldw, wb = wm.weight_operand()
    for it in range(3):
        for dt, code in ((torch.float32, N.OUT_F32), (torch.float16, N.OUT_F16)):
            out = torch.empty(t, n, dtype=dt, device="cuda")
            N.call("zq_linear_ws", a.data_ptr(), a.stride(0), xa.token_scales.data_ptr(), 0.0, wp, ldw, wb,
                   wm.row_scales().data_ptr(), bias.data_ptr(), t, n, d, out.data_ptr(), out.stride(0), code,
                   ws.data_ptr(), nbytes, N.stream_ptr())
            if dt == torch.float32:
                assert bits_eq(h(out), ref), (shape, it)
            else:
                assert torch.equal(out.cpu(), torch.from_numpy(ref).half()), (shape, it)
            assert not ws.any(), "workspace must be left zeroed"
