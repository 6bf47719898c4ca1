"""Decode-sized row kernels (8 / 16 rows) timed as 20 back-to-back launches in one
CUDA graph (warm instruction cache) — against their in-graph cost inside a decode
step (tools/ablate_decode.py).  python tools/row_graph_bench_decode.py [rows d]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402

t = int(sys.argv[1]) if len(sys.argv) > 1 else 8
d = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
f = 4 * d


def graph_time(fn, iters=20, interleave=None):
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
            if interleave is not None:
                interleave()
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
big = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def ln():
    N.call("zq_layer_norm_quantize", x.data_ptr(), r.data_ptr(), g_.data_ptr(), b_.data_ptr(), t, d,
           float(np.float32(1e-5)), 8, lo.data_ptr(), q.data_ptr(), q.stride(0), sc.data_ptr(), flag.data_ptr(),
           N.stream_ptr())


def gelu():
    N.call("zq_gelu_quantize", u.data_ptr(), t, f, f, 8, None, qf.data_ptr(), qf.stride(0), sc.data_ptr(),
           flag.data_ptr(), N.stream_ptr())


def tok():
    N.call("zq_quantize_tokenwise", x.data_ptr(), t, d, d, 8, q.data_ptr(), q.stride(0), sc.data_ptr(),
           flag.data_ptr(), N.stream_ptr())


def evict():  # a 256 MB memset between launches: the kernel's code and data leave L2
    big.zero_()


for name, fn in (("ln_quant", ln), ("gelu_quant", gelu), ("tok_quant", tok)):
    warm = graph_time(fn)
    both = graph_time(fn, interleave=evict)
    alone = graph_time(evict)
    print(f"{name} [{t}x{d}]: warm {warm:.2f} us; after an L2-evicting memset {both - alone:.2f} us")
