"""Fused QKV projection + attention (zq_qkv_attention) against the two kernels it
replaces (zq_linear f32 out -> zq_attention_f32) at the BERT bench shape: CUDA
events around graph replays of 20 back-to-back calls."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402


def timeit(fn, iters=20, reps=5):
    """Per-call time of `iters` calls captured into one CUDA graph (no host launch
    cost in the measurement), best of `reps` replays."""
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
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / iters * 1e3)
    return best


def run(batch, seq, heads):
    d = 64 * heads
    t = batch * seq
    xq = quant.quantize_activation_tokenwise(torch.randn(t, d, device="cuda"), 8)
    w = quant.quantize_weight_groupwise(torch.randn(3 * d, d, device="cuda") * 0.05, 48, 8)
    bias = torch.randn(3 * d, device="cuda") * 0.1
    qkv = torch.empty(t, 3 * d, device="cuda")
    ctx = torch.empty(t, d, device="cuda")
    wp, ldw, wb = w.weight_operand()
    rs = w.row_scales()
    scale = float(np.float32(1 / math.sqrt(64)))
    X, S = xq.values, xq.token_scales

    def lin():
        N.call("zq_linear", X.data_ptr(), X.stride(0), S.data_ptr(), 0.0, wp, ldw, wb, rs.data_ptr(),
               bias.data_ptr(), t, 3 * d, d, qkv.data_ptr(), qkv.stride(0), N.OUT_F32, N.stream_ptr())

    def att():
        N.call("zq_attention_f32", qkv.data_ptr(), qkv.stride(0), batch, seq, heads, 64, 0, scale, ctx.data_ptr(),
               ctx.stride(0), N.stream_ptr())

    def fused():
        N.call("zq_qkv_attention", X.data_ptr(), X.stride(0), S.data_ptr(), wp, ldw, rs.data_ptr(), bias.data_ptr(),
               batch, seq, heads, 64, 0, scale, ctx.data_ptr(), ctx.stride(0), N.stream_ptr())

    tl, ta = timeit(lin), timeit(att)
    tu = timeit(lambda: (lin(), att()))
    tf = timeit(fused)
    return {"shape": [batch, seq, heads], "linear_us": round(tl, 2), "attention_us": round(ta, 2),
            "two_kernels_us": round(tu, 2), "fused_us": round(tf, 2)}


if __name__ == "__main__":
    for shp in [(32, 128, 12), (64, 128, 12), (32, 128, 16), (8, 128, 12)]:
        print(json.dumps(run(*shp)), flush=True)
