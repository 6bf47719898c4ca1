"""Row kernels (LN + quant, GeLU + quant, token quant) at BERT-base shapes timed
as 20 back-to-back launches in one CUDA graph (warm instruction cache, inputs
L2-resident after the first) — to compare with their in-graph cost inside the
forward (bench.py row_kernels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402

t, d, f = 4096, 768, 3072


def graph_time(fn, iters=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / iters)
    return best


flag = torch.zeros(1, dtype=torch.int32, device="cuda")
x = torch.randn(t, d, device="cuda")
r = torch.randn(t, d, device="cuda")
g_ = torch.ones(d, device="cuda")
b_ = torch.zeros(d, device="cuda")
lo = torch.empty(t, d, device="cuda")
q = quant.padded_int8(t, d)
sc = torch.empty(t, device="cuda")
u = torch.randn(t, f, device="cuda")
qf = quant.padded_int8(t, f)


def ln():
    N.call("zq_layer_norm_quantize", x.data_ptr(), r.data_ptr(), g_.data_ptr(), b_.data_ptr(), t, d,
           float(np.float32(1e-12)), 8, lo.data_ptr(), q.data_ptr(), q.stride(0), sc.data_ptr(), flag.data_ptr(),
           N.stream_ptr())


def gelu():
    N.call("zq_gelu_quantize", u.data_ptr(), t, f, f, 8, None, qf.data_ptr(), qf.stride(0), sc.data_ptr(),
           flag.data_ptr(), N.stream_ptr())


def tok():
    N.call("zq_quantize_tokenwise", x.data_ptr(), t, d, d, 8, q.data_ptr(), q.stride(0), sc.data_ptr(),
           flag.data_ptr(), N.stream_ptr())


for name, fn in (("ln_quant", ln), ("gelu_quant", gelu), ("tok_quant", tok)):
    print(f"{name}: {graph_time(fn):.2f} us per launch (graph of 20, warm)")
