"""Timing of the converted-weight CTA-pair GEMMs (csrc/zq_gemm_conv.cu):
weight-only f16 / f16x2 at NeoX prefill shapes (TFLOP/s vs the bf16 peak) and
W4A8 pair vs the 1-CTA W4 kernel at GPT-3 350M / C1 shapes.  CUDA events on the
launching stream, graph-free back-to-back launches after warm-up."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def wmat(n, k, bits):
    w = torch.randn(n, k, device="cuda") * 0.02
    return quant.quantize_weight_groupwise(w, 48, bits)


def wo(m, k, n, bits, terms):
    wq = wmat(n, k, bits)
    x = torch.randn(m, k, device="cuda")
    ld_h = (k + 7) // 8 * 8
    hi = torch.empty(m, ld_h, dtype=torch.float16, device="cuda")
    lo = torch.empty(m, ld_h, dtype=torch.float16, device="cuda") if terms == 2 else None
    ri = torch.empty(m, device="cuda")
    out = torch.empty(m, n, dtype=torch.float16, device="cuda")
    wp, ld_w, wb = wq.weight_operand()
    rs = wq.row_scales()

    def split():
        N.call("zq_act_split16", x.data_ptr(), x.stride(0), m, k, terms, hi.data_ptr(), N.ptr(lo), ld_h,
               ri.data_ptr(), None, N.stream_ptr())

    def gemm():
        N.call("zq_linear_wo", hi.data_ptr(), N.ptr(lo), ld_h, ri.data_ptr(), wp, ld_w, wb, rs.data_ptr(), None,
               m, n, k, out.data_ptr(), out.stride(0), N.OUT_F16, N.stream_ptr())

    split()
    tg = timeit(gemm)
    ts = timeit(split)
    tf = 2.0 * m * n * k / (tg * 1e-6) / 1e12
    return {"shape": [m, k, n], "w_bits": bits, "terms": terms, "gemm_us": round(tg, 2), "split_us": round(ts, 2),
            "tflops_gemm": round(tf, 1), "tflops_with_split": round(2.0 * m * n * k / ((tg + ts) * 1e-6) / 1e12, 1)}


def w4a8(m, k, n):
    wq = wmat(n, k, 4)
    xq = quant.quantize_activation_tokenwise(torch.randn(m, k, device="cuda"), 8)
    out = torch.empty(m, n, dtype=torch.float32, device="cuda")
    t = timeit(lambda: igemm.fused_linear(xq, wq, None, out=out))
    return {"shape": [m, k, n], "w4a8_us": round(t, 2), "tops": round(2.0 * m * n * k / (t * 1e-6) / 1e12, 1)}


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "wo"):
        for shp in [(2048, 6144, 18432), (2048, 6144, 6144), (2048, 6144, 24576), (2048, 24576, 6144),
                    (8192, 8192, 8192)]:
            for bits, terms in [(8, 1), (8, 2), (4, 1)]:
                print(json.dumps(wo(*shp, bits, terms)), flush=True)
    if what in ("all", "w4"):
        for shp in [(8192, 1024, 4096), (8192, 4096, 1024), (4096, 768, 3072), (4096, 3072, 768)]:
            print(json.dumps(w4a8(*shp)), flush=True)
