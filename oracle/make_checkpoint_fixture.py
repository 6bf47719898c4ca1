"""Generate the ZQCK checkpoint fixture from the REAL reference (read-only import
of /root/reference/pkg/src).  TEST INFRASTRUCTURE ONLY.

    python oracle/make_checkpoint_fixture.py

writes tests/golden/tiny_w48a8.zqck (lowbit.checkpoint.save_model of a
quantized toy model: dim 64, 4 heads, 2 layers, vocab 128, W4/8A8, 16 groups)
and tests/golden/tiny_w48a8_ref.npz (token ids + the reference's
model_forward logits for them), so the device loader can be checked without
the reference on the GPU box.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    sys.path.insert(0, REF)
    from lowbit import checkpoint, transformer

    model = transformer.generate_toy_model(dim=64, num_heads=4, num_layers=2, vocab=128, seed=5, causal=True)
    prec = transformer.PrecisionConfig.from_scheme("W4/8A8", group_count=16)
    qmodel = transformer.quantize_model(model, prec)
    path = os.path.join(OUT, "tiny_w48a8.zqck")
    checkpoint.save_model(qmodel, path)
    ids = np.random.default_rng(9).integers(0, 128, 12)
    logits = transformer.model_forward(ids, qmodel, prec)
    np.savez_compressed(os.path.join(OUT, "tiny_w48a8_ref.npz"), ids=ids, logits=logits)
    print(f"wrote {path} ({os.path.getsize(path)} bytes) and reference logits {logits.shape}")


if __name__ == "__main__":
    main()
