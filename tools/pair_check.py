"""Quick correctness check of the CTA-pair GEMM path on a few shapes (exact int32)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import lowbit_oracle as O  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402

bad = 0
for (t, k, n) in [(4096, 768, 3072), (4000, 768, 3000), (300, 256, 512), (8192, 1024, 2048), (256, 128, 256)]:
    g = torch.Generator(device="cuda").manual_seed(t + n)
    xv = torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda", generator=g)
    wv = torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda", generator=g)
    xq = quant.QuantizedActivation(values=xv, bits=8, token_scales=torch.ones(t, device="cuda"))
    store = torch.zeros((n, quant.round_up(k, 32)), dtype=torch.int8, device="cuda")
    store[:, :k] = wv
    wq = quant.QuantizedMatrix(values=store[:, :k], bits=8, group_scales=torch.ones(1, device="cuda"),
                               group_layout=[(0, n)])
    acc = igemm.igemm(xq, wq).acc.cpu().numpy()
    ref = O.igemm(xv.cpu().numpy(), wv.cpu().numpy())
    ok = np.array_equal(acc, ref)
    bad += not ok
    print((t, k, n), "ok" if ok else f"MISMATCH {np.mean(acc != ref):.4f}", flush=True)
sys.exit(1 if bad else 0)
