"""Golden fixture for static calibration from the REAL
reference (`lowbit`, imported read-only from /root/reference/pkg/src).
TEST INFRASTRUCTURE ONLY; run in the build container:

    python oracle/make_calibration_golden.py   # writes tests/golden/calibration.npz

Model: lowbit.transformer.generate_toy_model(dim=64, heads=4, layers=2,
vocab=128, seed=3, hetero_knob=True, causal=True) with its biases and
LayerNorm parameters then perturbed from the same splitmix64 Rng (so every
term of the float forward is exercised).  Calibration:
lowbit.evaluate.calibrate_model over three token sequences of lengths 17, 32
and 9 (evaluate.py:168-196).  Static forward: the W8A8 static model
(quantize_model + model_forward with the calibrated scales,
transformer.py:364-378, :522-532) on the first sequence.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "calibration.npz")
F32 = np.float32


def main() -> None:
    sys.path.insert(0, REF)
    from lowbit import evaluate, transformer
    from lowbit.tensor import Rng

    model = transformer.generate_toy_model(dim=64, num_heads=4, num_layers=2, vocab=128, seed=3,
                                           hetero_knob=True, causal=True)
    rng = Rng(77)
    for b in model.blocks:
        for n in ("b_q", "b_k", "b_v", "b_o", "b_h4h", "b_4hh", "ln1_beta", "ln2_beta"):
            v = getattr(b, n)
            setattr(b, n, rng.gaussian(v.shape, std=0.05))
        for n in ("ln1_gamma", "ln2_gamma"):
            setattr(b, n, (1.0 + rng.gaussian((model.dim,), std=0.1)).astype(F32))
    model.final_gamma = (1.0 + rng.gaussian((model.dim,), std=0.1)).astype(F32)
    model.final_beta = rng.gaussian((model.dim,), std=0.05)
    ids_rng = np.random.default_rng(5)
    batches = [ids_rng.integers(0, 128, n).astype(np.int64) for n in (17, 32, 9)]
    cal = evaluate.calibrate_model(model, batches)
    scales = evaluate.static_scales_from(cal)
    prec = transformer.PrecisionConfig.from_scheme("W8A8", group_count=16, activation_static=True)
    qmodel = transformer.quantize_model(model, prec)
    logits = transformer.model_forward(batches[0], qmodel, prec, static_scales=scales)
    out = {"embedding": model.embedding, "final_gamma": model.final_gamma, "final_beta": model.final_beta,
           "num_heads": np.int64(model.num_heads), "layers": np.int64(len(model.blocks)),
           "static_logits_b0": logits}
    for i, n in enumerate((17, 32, 9)):
        out[f"batch{i}"] = batches[i]
    for li, b in enumerate(model.blocks):
        for n in ("w_q", "w_k", "w_v", "w_o", "w_h4h", "w_4hh", "b_q", "b_k", "b_v", "b_o", "b_h4h", "b_4hh",
                  "ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta"):
            out[f"l{li}_{n}"] = getattr(b, n)
    keys = sorted(cal)
    out["site_keys"] = np.array(keys)
    out["site_xmax"] = np.array([cal[k].x_max for k in keys], np.float64)
    out["site_xmin"] = np.array([cal[k].x_min for k in keys], np.float64)
    out["site_scale"] = np.array([cal[k].scale for k in keys], np.float64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(keys)} sites, scales {[round(cal[k].scale, 6) for k in keys]}")


if __name__ == "__main__":
    main()
