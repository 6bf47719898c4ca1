"""One profiled launch each of the north-star kernels at large shapes, for
ncu --set full --nvtx --nvtx-include "prof/": W8A8 GEMM 8192^3 (f16 out),
4096x4096x16384, W4A8 CTA pair 8192x4096x1024, weight-only f16 NeoX QKV prefill
(2048x6144x18432), decode 16x6144x24576 (stream-K + sum epilogue), TMA decode
attention (NeoX, 16 x 192 keys), token quantize / LN+quant / GeLU+quant at
4096x3072, the fused QKV + attention kernel at the BERT bench shape.  Two
warm-up launches each, outside the NVTX range."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def prof(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("prof")
    fn()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()


def gemm(t, k, n, od=torch.float16, bits=8):
    xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda"), bits=8,
                                   token_scales=torch.rand(t, device="cuda"))
    w = quant.quantize_weight_groupwise(torch.randn(n, k, device="cuda") * 0.02, 64, bits)
    out = torch.empty(t, n, dtype=od, device="cuda")
    prof(lambda: igemm.fused_linear(xq, w, None, out=out))


def decode_streamk(t, k, n):
    xq = quant.padded_int8(t, k)
    xq.copy_(torch.randint(-127, 128, (t, k), device="cuda", dtype=torch.int8))
    w = quant.quantize_weight_groupwise(torch.randn(n, k, device="cuda") * 0.02, 64, 8)
    ts = torch.rand(t, device="cuda")
    out = torch.empty(t, n, device="cuda")
    nb = int(N.load().zq_linear_ws_bytes(t, n))
    ws = torch.zeros(nb // 4, dtype=torch.int32, device="cuda")
    wp, ldw, wb = w.weight_operand()
    prof(lambda: N.call("zq_linear_ws", xq.data_ptr(), xq.stride(0), ts.data_ptr(), 0.0, wp, ldw, wb,
                        w.row_scales().data_ptr(), None, t, n, k, out.data_ptr(), out.stride(0), N.OUT_F32,
                        ws.data_ptr(), nb, N.stream_ptr()))


gemm(8192, 8192, 8192)
gemm(4096, 4096, 16384)
gemm(8192, 4096, 1024, torch.float32, bits=4)
xw = torch.randn(2048, 6144, device="cuda")
ww = quant.quantize_weight_groupwise(torch.randn(18432, 6144, device="cuda") * 0.02, 128, 8)
prof(lambda: igemm.full_linear(xw, ww, None, precision="f16", out_dtype=torch.float16))
decode_streamk(16, 6144, 24576)
batch, heads, dh, ctx_len, max_ctx = 16, 64, 96, 192, 256
kc = torch.randn(batch, max_ctx, heads * dh, device="cuda")
vc = torch.randn(batch, max_ctx, heads * dh, device="cuda")
q = torch.randn(batch, 3 * heads * dh, device="cuda")
lens = torch.full((batch,), ctx_len, dtype=torch.int32, device="cuda")
ctx = torch.empty(batch, heads * dh, device="cuda")
C = int(N.load().zq_decode_attention_chunks(batch, heads, max_ctx))
prof(lambda: N.call("zq_decode_attention_f32", q.data_ptr(), q.stride(0), kc.data_ptr(), vc.data_ptr(), max_ctx,
                    batch, heads, dh, lens.data_ptr(), dh ** -0.5, ctx.data_ptr(), ctx.stride(0), C, N.stream_ptr()))
x = torch.randn(4096, 3072, device="cuda")
r = torch.randn(4096, 3072, device="cuda")
g, b = torch.ones(3072, device="cuda"), torch.zeros(3072, device="cuda")
y = torch.empty_like(x)
prof(lambda: quant.quantize_activation_tokenwise(x, 8, check_finite=False))
prof(lambda: igemm.layer_norm_quantize(x, g, b, 8, residual=r, ln_out=y, check_finite=False))
prof(lambda: igemm.gelu_quantize(x, 8, check_finite=False))
# fused W8A8 QKV projection + attention at the BERT-base bench shape (32 x 128, 12 heads)
from paper_2206_01861_b200 import transformer as T  # noqa: E402

xa = quant.quantize_activation_tokenwise(torch.randn(4096, 768, device="cuda"), 8)
wqkv = quant.quantize_weight_groupwise(torch.randn(2304, 768, device="cuda") * 0.05, 48, 8)
bqkv = torch.randn(2304, device="cuda") * 0.1
cx = torch.empty(4096, 768, device="cuda")
prof(lambda: T.fused_qkv_attention(xa.values, xa.token_scales, wqkv, bqkv, 12, False, 32, cx))
