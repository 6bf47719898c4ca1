"""Fused linear + residual + LN + quantize vs the two-kernel path (BERT shapes)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402
from tools.timing import graph_time  # noqa: E402


def run(m, n, k):
    xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (m, k), dtype=torch.int8, device="cuda"), bits=8,
                                   token_scales=torch.rand(m, device="cuda") * 0.05)
    w = quant.quantize_weight_groupwise(torch.randn(n, k, device="cuda") * 0.02, 16, 8)
    bias, g, b = torch.zeros(n, device="cuda"), torch.ones(n, device="cuda"), torch.zeros(n, device="cuda")
    res = torch.randn(m, n, device="cuda")
    y, f = torch.empty(m, n, device="cuda"), torch.empty(m, n, device="cuda")
    q = quant.padded_int8(m, n)
    s = torch.empty(m, device="cuda")
    ws = torch.zeros(4 * ((m + 255) // 256) + 16 + 12 * m * 64, dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    a = xq.gemm_operand()
    wp, ldw, wb = w.weight_operand()

    def fused():
        N.call("zq_linear_ln_quantize", a.data_ptr(), a.stride(0), xq.token_scales.data_ptr(), wp, ldw, wb,
               w.row_scales().data_ptr(), bias.data_ptr(), m, n, k, res.data_ptr(), g.data_ptr(), b.data_ptr(),
               1e-5, 8, y.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(), ws.data_ptr(), ws.numel(),
               flag.data_ptr(), N.stream_ptr())

    def unfused():
        igemm.fused_linear(xq, w, bias, out=f)
        N.call("zq_layer_norm_quantize", res.data_ptr(), f.data_ptr(), g.data_ptr(), b.data_ptr(), m, n, 1e-5, 8,
               y.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(), flag.data_ptr(), N.stream_ptr())

    print(json.dumps({"shape": [m, n, k], "fused_us": round(graph_time([fused]) * 1e6, 2),
                      "unfused_us": round(graph_time([unfused]) * 1e6, 2)}))


if __name__ == "__main__":
    run(4096, 768, 768)
    run(4096, 768, 3072)
