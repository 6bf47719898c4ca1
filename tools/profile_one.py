"""Run one op a few times for ncu capture: python tools/profile_one.py <op>."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def main():
    op = sys.argv[1] if len(sys.argv) > 1 else "c1"
    torch.manual_seed(0)
    if op == "c1":
        x = torch.randn(4096, 768, device="cuda")
        w = torch.randn(3072, 768, device="cuda") * 0.02
        wq = quant.quantize_weight_groupwise(w, 48, 8)
        for _ in range(3):
            xq = quant.quantize_activation_tokenwise(x, 8, check_finite=False)
            igemm.fused_linear(xq, wq, None, out_dtype=torch.float16)
            xg = igemm.gelu_quantize(x, 8, check_finite=False)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
