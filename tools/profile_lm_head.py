"""GPT-J-sized LM head (16 tokens x 50400 x 4096) for ncu / timing."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from tools.timing import graph_time  # noqa: E402

ntok, vocab, dim = 16, 50400, 4096
x = torch.randn(ntok, dim, device="cuda")
embs = [torch.randn(vocab, dim, device="cuda") * 0.02 for _ in range(2)]
scale = math.ldexp(1.0, 15 - math.frexp(float(embs[0].abs().max()))[1])
xh = torch.zeros(16 * dim, dtype=torch.float16, device="cuda")
xl = torch.zeros_like(xh)
xinv = torch.zeros(16, device="cuda")
keys = torch.zeros(16, dtype=torch.int64, device="cuda")
ids = torch.zeros(ntok, dtype=torch.int64, device="cuda")


def run(e):
    N.call("zq_lm_head_argmax", x.data_ptr(), x.stride(0), ntok, e.data_ptr(), vocab, dim, scale, xh.data_ptr(),
           xl.data_ptr(), xinv.data_ptr(), keys.data_ptr(), ids.data_ptr(), N.stream_ptr())


if __name__ == "__main__":
    sec = graph_time([lambda e=e: run(e) for e in embs])
    print(f"lm head {ntok}x{vocab}x{dim}: {sec * 1e6:.1f} us, {vocab * dim * 4 / sec / 1e12:.2f} TB/s")
    lo = torch.empty(ntok, vocab, device="cuda")
    sec2 = graph_time([lambda e=e: (torch.matmul(x, e.t(), out=lo), torch.argmax(lo, 1)) for e in embs])
    print(f"cuBLAS sgemm + argmax: {sec2 * 1e6:.1f} us")
