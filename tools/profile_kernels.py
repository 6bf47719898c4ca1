"""One launch each of the north-star kernels at large shapes, for ncu --set full:
W8A8 GEMM 8192^3 (f16 out), 4096x4096x16384, decode 16x6144x24576, token
quantize / LN+quant / GeLU+quant at 4096x3072.  Two warm-up launches each."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def gemm(t, k, n, od=torch.float16):
    xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda"), bits=8,
                                   token_scales=torch.rand(t, device="cuda"))
    w = quant.QuantizedMatrix(values=torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda"), bits=8,
                              group_scales=torch.rand(1, device="cuda"), group_layout=[(0, n)])
    out = torch.empty(t, n, dtype=od, device="cuda")
    for _ in range(3):
        igemm.fused_linear(xq, w, None, out=out)


gemm(8192, 8192, 8192)
gemm(4096, 4096, 16384)
gemm(16, 6144, 24576)
x = torch.randn(4096, 3072, device="cuda")
r = torch.randn(4096, 3072, device="cuda")
g, b = torch.ones(3072, device="cuda"), torch.zeros(3072, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    quant.quantize_activation_tokenwise(x, 8, check_finite=False)
for _ in range(3):
    igemm.layer_norm_quantize(x, g, b, 8, residual=r, ln_out=y, check_finite=False)
for _ in range(3):
    igemm.gelu_quantize(x, 8, check_finite=False)
torch.cuda.synchronize()
