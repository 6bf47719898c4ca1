"""Per-launch cost of the decode-sized row kernels and skinny GEMMs when chained
back to back in one CUDA graph (PDL on), at GPT-3 350M (8 x 1024) and GPT-J
(16 x 4096) decode shapes.  kv_append of 1 row is the near-empty reference."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402


def chain(fn, n=64):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for name, t, d, f in (("gpt3-350m", 8, 1024, 4096), ("gptj-6b", 16, 4096, 16384), ("neox-20b", 16, 6144, 24576)):
    x = torch.randn(t, d, device="cuda")
    res = torch.randn(t, d, device="cuda")
    u = torch.randn(t, f, device="cuda")
    g = torch.ones(d, device="cuda")
    b = torch.zeros(d, device="cuda")
    y = torch.empty(t, d, device="cuda")
    q = quant.padded_int8(t, d)
    qf = quant.padded_int8(t, f)
    s = torch.empty(t, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    kc = torch.zeros(t, 4, 64, device="cuda")
    vc = torch.zeros(t, 4, 64, device="cuda")
    qkv = torch.randn(t, 3 * 64, device="cuda")
    pos = torch.zeros(t, dtype=torch.int32, device="cuda")
    w = quant.quantize_weight_groupwise(torch.randn(d, d, device="cuda") * 0.02, 64, 8)
    w4 = quant.quantize_weight_groupwise(torch.randn(f, d, device="cuda") * 0.02, 64, 4)
    w4b = quant.quantize_weight_groupwise(torch.randn(d, f, device="cuda") * 0.02, 64, 4)
    out = torch.empty(t, f, device="cuda")
    r = {"case": name}
    r["kv_append_1row"] = chain(lambda: N.call("zq_kv_append", qkv.data_ptr(), qkv.stride(0), t, 1, 64, pos.data_ptr(),
                                               kc.data_ptr(), vc.data_ptr(), 4, N.stream_ptr()))
    r["tok_quant"] = chain(lambda: N.call("zq_quantize_tokenwise", x.data_ptr(), t, d, d, 8, q.data_ptr(), q.stride(0),
                                          s.data_ptr(), flag.data_ptr(), N.stream_ptr()))
    r["ln_quant"] = chain(lambda: N.call("zq_layer_norm_quantize", x.data_ptr(), res.data_ptr(), g.data_ptr(),
                                         b.data_ptr(), t, d, 1e-5, 8, y.data_ptr(), q.data_ptr(), q.stride(0),
                                         s.data_ptr(), flag.data_ptr(), N.stream_ptr()))
    r["gelu_quant"] = chain(lambda: N.call("zq_gelu_quantize", u.data_ptr(), t, f, f, 8, None, qf.data_ptr(),
                                           qf.stride(0), s.data_ptr(), flag.data_ptr(), N.stream_ptr()))
    for nm, wm, xq in (("gemm_dxd_w8", w, q), ("gemm_dxf_w4", w4, q), ("gemm_fxd_w4", w4b, qf)):
        wp, ldw, wb = wm.weight_operand()
        r[nm] = chain(lambda: N.call("zq_linear", xq.data_ptr(), xq.stride(0), s.data_ptr(), 0.0, wp, ldw, wb,
                                     wm.row_scales().data_ptr(), None, t, wm.rows, wm.cols, out.data_ptr(),
                                     out.stride(0), N.OUT_F32, N.stream_ptr()))
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
