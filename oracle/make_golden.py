"""Generate golden fixtures from the REAL reference (`lowbit`, imported read-only
from /root/reference/pkg/src).  TEST INFRASTRUCTURE ONLY.

Run in the build container (the reference does not exist on the GPU box):

    python oracle/make_golden.py            # writes tests/golden/*.npz + hashes.json

Small cases are stored in full (inputs and outputs).  Cases at BASELINE sizes
store only SHA-256 digests of the reference outputs; their inputs are
regenerated in the tests from the portable splitmix64 `Rng`
(pkg/src/lowbit/tensor.py:119-164), whose stream is itself pinned here.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")
F32 = np.float32


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def planted_ties(rng, t, d, bits):
    """Rows whose entries sit exactly on RHAFZ ties for the row's own scale."""
    from lowbit import quant

    x = (rng.standard_normal((t, d)) * rng.uniform(0.1, 10)).astype(F32)
    s = np.asarray([quant.compute_scale(r, bits) for r in x], dtype=np.float64)
    k = rng.integers(0, quant.qmax(bits), (t, d)).astype(np.float64) + 0.5
    cand = (k * s[:, None]).astype(F32)
    exact = cand.astype(np.float64) == k * s[:, None]
    mask = (rng.uniform(size=(t, d)) < 0.3) & exact
    # keep the row max unchanged so the planted values stay ties
    am = np.abs(x).max(axis=1, keepdims=True)
    ok = mask & (np.abs(cand) < am)
    x = np.where(ok, np.sign(rng.standard_normal((t, d))).astype(F32) * cand, x).astype(F32)
    return x


def main() -> None:
    sys.path.insert(0, REF)
    from lowbit import igemm, quant, tensor, transformer
    from lowbit.igemm import DynamicAct, FullAct, StaticAct
    from lowbit.tensor import Rng

    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20220603)
    arrays: dict[str, np.ndarray] = {}
    hashes: dict[str, dict] = {}

    # -- Rng stream pin (tensor.py:119-164) --------------------------------
    r = Rng(1234)
    arrays["rng_u64"] = np.asarray([r.next_u64() for _ in range(4)], dtype=np.uint64)
    arrays["rng_gauss"] = Rng(7).gaussian((3, 5), std=0.5)
    arrays["rng_ints"] = Rng(9).integers(1000, 16)

    # -- token-wise activation quantization (quant.py:258-269) -------------
    tok_cases = []
    shapes = [(1, 1), (1, 16), (2, 4), (3, 7), (5, 33), (8, 64), (16, 96), (7, 100),
              (4, 768), (3, 1024), (2, 3072), (1, 4096), (2, 6144), (1, 16384), (33, 257)]
    for i, (t, d) in enumerate(shapes):
        for bits in (8, 4):
            kind = i % 3
            if kind == 0:
                x = (rng.standard_normal((t, d)) * rng.uniform(0.01, 50)).astype(F32)
            elif kind == 1:
                x = planted_ties(rng, t, d, bits)
            else:
                x = (rng.standard_normal((t, d)) * 3).astype(F32)
                x[0] = 0.0  # zero row -> scale 1.0
                if t > 1:
                    x[-1, ::3] = -x[-1, ::3]
            qa = quant.quantize_activation_tokenwise(x, bits)
            name = f"tok_{t}x{d}_b{bits}"
            arrays[name + "_x"] = x
            arrays[name + "_q"] = qa.values
            arrays[name + "_s"] = qa.token_scales
            tok_cases.append(name)

    # KAT: quant.py docstring cases (test_quant.py:206-212)
    x = np.zeros((2, 4), dtype=F32)
    x[0, 0] = 35.0
    x[1, 2] = -8.0
    qa = quant.quantize_activation_tokenwise(x, 8)
    arrays["tok_kat_x"], arrays["tok_kat_q"], arrays["tok_kat_s"] = x, qa.values, qa.token_scales

    # -- static quantization (quant.py:272-281, :103-113) ------------------
    static_cases = []
    for j, scale in enumerate([0.05, 1.0 / 127.0, 2.0 / 127.0, float(F32(0.0123)), 0.37, 3.0e-3]):
        for bits in (8, 4):
            x = (rng.standard_normal((9, 70)) * rng.uniform(0.1, 3)).astype(F32)
            if j == 2:
                x[0, :5] = [1.0, -1.0, 2.0, -2.0, 0.0]  # test_quant.py:57-66 ties/extremes
            qa = quant.quantize_activation_static(x, scale, bits)
            name = f"static_{j}_b{bits}"
            arrays[name + "_x"] = x
            arrays[name + "_q"] = qa.values
            arrays[name + "_scale"] = np.asarray([scale], dtype=np.float64)
            static_cases.append(name)

    # -- group-wise weight quantization (quant.py:236-255) -----------------
    wq_cases = []
    for (n, m, g) in [(4, 2, 2), (5, 2, 2), (6, 5, 1), (16, 24, 4), (64, 32, 16), (48, 96, 48),
                      (100, 64, 7), (768, 64, 48), (256, 128, 128), (33, 40, 33)]:
        for bits in (8, 4):
            w = (rng.standard_normal((n, m)) * 0.02).astype(F32)
            hot = rng.choice(n, max(1, n // 4), replace=False)
            w[hot] *= F32(10.0)
            qm = quant.quantize_weight_groupwise(w, g, bits)
            name = f"wq_{n}x{m}_g{g}_b{bits}"
            arrays[name + "_w"] = w
            arrays[name + "_q"] = qm.values
            arrays[name + "_gs"] = qm.group_scales
            arrays[name + "_rs"] = qm.row_scales()
            arrays[name + "_layout"] = np.asarray(qm.group_layout, dtype=np.int64)
            wq_cases.append(name)
    w = np.array([[10.0, -10.0], [8.0, 8.0], [0.1, -0.1], [0.05, 0.1]], dtype=F32)
    qm = quant.quantize_weight_groupwise(w, 2, 8)  # test_quant.py:118-128
    arrays["wq_kat_w"], arrays["wq_kat_q"], arrays["wq_kat_gs"] = w, qm.values, qm.group_scales

    # -- igemm / epilogue / quantized_linear (igemm.py:66-139) -------------
    lin_cases = []
    for i in range(40):
        t = int(rng.integers(1, 65))
        d = int(rng.integers(1, 257))
        n = int(rng.integers(1, 257))
        if i % 5 == 0:
            d = 32 * int(rng.integers(1, 9))  # tensor-core friendly K as well
        x = (rng.standard_normal((t, d)) * rng.uniform(0.1, 8.0)).astype(F32)
        w = (rng.standard_normal((n, d)) * rng.uniform(0.01, 2.0)).astype(F32)
        bias = rng.standard_normal(n).astype(F32) if i % 4 else None
        groups = int(rng.integers(1, min(16, n) + 1))
        wbits = 8 if i % 3 else 4
        wq = quant.quantize_weight_groupwise(w, groups, wbits)
        xq = quant.quantize_activation_tokenwise(x, 8)
        acc = igemm.igemm(xq, wq).acc
        dyn = igemm.quantized_linear(x, wq, bias, DynamicAct(8))
        sscale = float(quant.compute_scale(x, 8)) * 0.9
        sta = igemm.quantized_linear(x, wq, bias, StaticAct(sscale, 8))
        name = f"lin_{i}"
        arrays[name + "_x"] = x
        arrays[name + "_w"] = w
        if bias is not None:
            arrays[name + "_bias"] = bias
        arrays[name + "_meta"] = np.asarray([t, d, n, groups, wbits], dtype=np.int64)
        arrays[name + "_sscale"] = np.asarray([sscale], dtype=np.float64)
        arrays[name + "_acc"] = acc
        arrays[name + "_dyn"] = dyn
        arrays[name + "_sta"] = sta
        if i < 12:
            arrays[name + "_full"] = igemm.quantized_linear(x, wq, bias, FullAct())
        lin_cases.append(name)

    # -- quantize-on-write LN / GeLU (igemm.py:150-161, tensor.py:59-83) ---
    fused_cases = []
    for (t, d) in [(6, 12), (3, 8), (2, 5), (4, 64), (5, 96), (3, 100), (4, 130), (8, 768),
                   (4, 1024), (2, 3072), (2, 4096), (2, 6144), (1, 300)]:
        x = (rng.standard_normal((t, d)) * rng.uniform(0.2, 4)).astype(F32)
        gamma = (1.0 + 0.1 * rng.standard_normal(d)).astype(F32)
        beta = (0.1 * rng.standard_normal(d)).astype(F32)
        ln = tensor.layer_norm(x, gamma, beta)
        lq = igemm.layer_norm_quantize(x, gamma, beta, 8)
        ge = tensor.gelu(x)
        gq = igemm.gelu_quantize(x, 8)
        name = f"fused_{t}x{d}"
        arrays[name + "_x"] = x
        arrays[name + "_gamma"] = gamma
        arrays[name + "_beta"] = beta
        arrays[name + "_ln"] = ln
        arrays[name + "_lnq"] = lq.values
        arrays[name + "_lns"] = lq.token_scales
        arrays[name + "_gelu"] = ge
        arrays[name + "_geq"] = gq.values
        arrays[name + "_ges"] = gq.token_scales
        fused_cases.append(name)

    # -- block forward (transformer.py:443-486), tolerance-only downstream --
    model = transformer.generate_toy_model(dim=64, num_heads=4, num_layers=1, vocab=64, seed=3)
    blk = model.blocks[0]
    xb = Rng(11).gaussian((16, 64), std=0.5)
    for scheme in ("W8A8", "W4/8A8", "W8A8/16"):
        prec = transformer.PrecisionConfig.from_scheme(scheme, hidden_dim=64)
        qb = transformer.quantize_block(blk, prec)
        for causal in (False, True):
            y = transformer.block_forward(xb, qb, prec, causal)
            arrays[f"block_{scheme.replace('/', '_')}_c{int(causal)}_y"] = y
    arrays["block_x"] = xb
    for nm in transformer.WEIGHT_NAMES + transformer.BIAS_NAMES + (
            "ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta"):
        arrays["block_" + nm] = getattr(blk, nm)

    # -- BASELINE-size digests: inputs regenerated from Rng in the tests ----
    # C1: quantized_linear W8A8, 4096 tok, 768 -> 3072, g=48
    w = Rng(0).gaussian((3072, 768), std=0.02)
    x = Rng(1).gaussian((4096, 768), std=1.0)
    wq = quant.quantize_weight_groupwise(w, 48, 8)
    xq = quant.quantize_activation_tokenwise(x, 8)
    acc = (xq.values.astype(np.float64) @ wq.values.astype(np.float64).T).astype(np.int32)
    out = igemm.dequant_epilogue(igemm.IntAccumulator(acc), xq.token_scales, wq, None)
    hashes["c1"] = {
        "w": sha(w), "x": sha(x),
        "wq_values": sha(wq.values), "wq_scales": sha(wq.group_scales),
        "xq_values": sha(xq.values), "xq_scales": sha(xq.token_scales),
        "acc": sha(acc), "out_f32": sha(out),
        "note": "igemm via exact f64 BLAS (bit-identical to igemm.py:79; checked on a slice below)",
    }
    sl = igemm.igemm(quant.QuantizedActivation(xq.values[:64], 8, xq.token_scales[:64]), wq).acc
    assert np.array_equal(sl, acc[:64]), "f64 BLAS igemm restatement disagrees with reference"
    # fused LN / GeLU quantize at a BERT-base shape
    xl = Rng(2).gaussian((512, 768), std=1.0)
    lq = igemm.layer_norm_quantize(xl, np.ones(768, F32), np.zeros(768, F32), 8)
    hashes["ln_512x768"] = {"x": sha(xl), "q": sha(lq.values), "s": sha(lq.token_scales)}
    xg = Rng(3).gaussian((256, 3072), std=1.0)
    gq = igemm.gelu_quantize(xg, 8)
    hashes["gelu_256x3072"] = {"x": sha(xg), "q": sha(gq.values), "s": sha(gq.token_scales),
                               "gelu": sha(tensor.gelu(xg))}

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    meta = {
        "generator": "oracle/make_golden.py",
        "reference": "lowbit 0.1.0 (/root/reference/pkg/src)",
        "numpy": np.__version__,
        "cases": {"tok": tok_cases, "static": static_cases, "wq": wq_cases,
                  "lin": lin_cases, "fused": fused_cases},
        "hashes": hashes,
    }
    import scipy

    meta["scipy"] = scipy.__version__
    with open(os.path.join(OUT, "golden_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    size = os.path.getsize(os.path.join(OUT, "golden.npz"))
    print(f"wrote {len(arrays)} arrays ({size / 1e6:.2f} MB) and {len(hashes)} digest groups")


if __name__ == "__main__":
    main()
