"""Decode-shaped (M = 16 tokens) W8A8 linears at GPT-J / NeoX widths: GB/s of
int8 weights streamed, each launch on a different weight copy (> L2), chained
in one CUDA graph with PDL as in the decode step."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402

# ZQ_GEMM_STREAMK_MIN=0 forces stream-K for every shape (with SK=1)
SHAPES = [("gptj qkv", 4096, 12288), ("gptj o", 4096, 4096), ("gptj h4h", 4096, 16384), ("gptj 4hh", 16384, 4096),
          ("neox qkv", 6144, 18432), ("neox o", 6144, 6144), ("neox h4h", 6144, 24576), ("neox 4hh", 24576, 6144)]
M = int(os.environ.get("M", "16"))
for name, k, n in SHAPES:
    copies = max(2, int(600e6 // (n * k)))
    ws = []
    for _ in range(copies):
        w = quant.padded_int8(n, k, align=32)
        w.copy_(torch.randint(-127, 128, (n, k), device="cuda", dtype=torch.int8))
        ws.append(w)
    rs = torch.rand(n, device="cuda") * 1e-3
    xq = quant.padded_int8(M, k)
    xq.copy_(torch.randint(-127, 128, (M, k), device="cuda", dtype=torch.int8))
    ts = torch.rand(M, device="cuda")
    out = torch.empty(M, n, device="cuda")

    nb = int(N.load().zq_linear_ws_bytes(M, n))
    skws = torch.zeros(nb // 4 + 4, dtype=torch.int32, device="cuda")
    use_ws = os.environ.get("SK", "1") == "1"

    def run(i):
        w = ws[i % copies]
        if use_ws:
            N.call("zq_linear_ws", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, w.data_ptr(), w.stride(0), 8,
                   rs.data_ptr(), None, M, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, skws.data_ptr(),
                   4 * skws.numel(), N.stream_ptr())
        else:
            N.call("zq_linear", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, w.data_ptr(), w.stride(0), 8,
                   rs.data_ptr(), None, M, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, N.stream_ptr())

    for i in range(3):
        run(i)
    g = torch.cuda.CUDAGraph()
    reps = 3 * copies
    with torch.cuda.graph(g):
        for i in range(reps):
            run(i)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / reps * 1e3
    print(json.dumps({"shape": name, "streamk": use_ws, "K": k, "N": n, "M": M, "us": round(us, 2),
                      "GBps": round(n * k / us / 1e3, 1)}),
          flush=True)
    del ws
    torch.cuda.empty_cache()
