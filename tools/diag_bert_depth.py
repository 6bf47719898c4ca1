"""Diagnose per-layer divergence of the BERT-base encoder vs the oracle:
one-step error (oracle block applied to the device's own layer input) and the
accumulated error, for sequence 0."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lowbit_oracle as O  # noqa: E402
from paper_2206_01861_b200 import transformer as T  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_baseline_shapes_gpu import oracle_qb, rel, h  # noqa: E402

d, heads, L, V = 768, 12, 12, 30522
std = float(sys.argv[1]) if len(sys.argv) > 1 else 0.02
blocks = [T.random_block(d, heads, 8, 8, 48, seed=100 + i, ffn_mult=4, std=std) for i in range(L)]
gen = torch.Generator(device="cuda").manual_seed(7)
emb = torch.randn((V, d), generator=gen, device="cuda") * 0.02
ids = np.random.default_rng(3).integers(0, V, (32, 128))
prec = T.PrecisionConfig.from_scheme("W8A8", group_count=48)
x = emb[torch.from_numpy(ids.reshape(-1)).cuda()]
xo = h(x)[:128]
for li, blk in enumerate(blocks):
    qb = oracle_qb(blk)
    xin = h(x)[:128]
    x = T.block_forward(x, blk, prec, causal=False, batch=32)
    y = h(x)[:128]
    one = O.block_forward(xin, qb, heads, False, "int8")
    xo = O.block_forward(xo, qb, heads, False, "int8")
    # how many int8 codes differ in the first quantization of this layer
    qd, _ = O.quantize_activation_tokenwise(xin, 8)
    print(f"layer {li}: one-step rel {rel(y, one):.2e}  accumulated rel {rel(y, xo):.2e}  |x| {np.linalg.norm(y)/np.sqrt(y.size):.3f}")
