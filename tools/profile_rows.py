"""BERT-shape row kernels for ncu: tok quant (4096x768), LN+residual+quant
(4096x768), GeLU+quant (4096x3072), one launch each after a warm-up."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import igemm, quant  # noqa: E402

x = torch.randn(4096, 768, device="cuda")
r = torch.randn(4096, 768, device="cuda")
u = torch.randn(4096, 3072, device="cuda") * 0.7
g, b = torch.ones(768, device="cuda"), torch.zeros(768, device="cuda")
ln = torch.empty_like(x)
for _ in range(3):
    quant.quantize_activation_tokenwise(x, 8, check_finite=False)
    igemm.layer_norm_quantize(x, g, b, 8, residual=r, ln_out=ln, check_finite=False)
    igemm.gelu_quantize(u, 8, check_finite=False)
torch.cuda.synchronize()
