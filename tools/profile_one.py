"""Run one op a few times for ncu capture: python tools/profile_one.py <op>."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def gemm(t, k, n, od=torch.float16, wb=8):
    xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda"),
                                   bits=8, token_scales=torch.rand(t, device="cuda"))
    lo, hi = (-7, 8) if wb == 4 else (-127, 128)
    wq = quant.QuantizedMatrix(values=torch.randint(lo, hi, (n, k), dtype=torch.int8, device="cuda"), bits=wb,
                               group_scales=torch.rand(1, device="cuda"), group_layout=[(0, n)])
    out = torch.empty(t, n, dtype=od, device="cuda")
    for _ in range(3):
        igemm.fused_linear(xq, wq, None, out=out)


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "c1"
    torch.manual_seed(0)
    if op == "c1":
        gemm(4096, 768, 3072)
    elif op == "big":
        gemm(8192, 8192, 8192)
    elif op == "c1f32":
        gemm(4096, 768, 3072, torch.float32)
    elif op == "quant":
        x = torch.randn(4096, 3072, device="cuda")
        for _ in range(3):
            quant.quantize_activation_tokenwise(x, 8, check_finite=False)
            igemm.gelu_quantize(x, 8, check_finite=False)
            igemm.layer_norm_quantize(x, torch.ones(3072, device="cuda"), torch.zeros(3072, device="cuda"), 8,
                                      check_finite=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
