"""Per-kernel device times of one GPT decode layer at batch 16 (graph replay of
the same launch, L2-warm weights excluded by rotating sets where large).
python tools/decode_micro.py [gptj-6b|neox-20b]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402
from paper_2206_01861_b200.decoder import CONFIGS  # noqa: E402
from tools.timing import graph_time  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
    cfg = CONFIGS[name]
    B, ctx = 16, 192
    d, f, H, dh = cfg.dim, cfg.ffn, cfg.heads, cfg.head_dim
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {}
    x = torch.randn(B, d, device="cuda")
    u = torch.randn(B, f, device="cuda")
    q = quant.padded_int8(B, f)
    s = torch.empty(B, device="cuda")
    g1, b1 = torch.ones(d, device="cuda"), torch.zeros(d, device="cuda")
    y = torch.empty(B, d, device="cuda")
    res["tok_quant_d"] = graph_time([lambda: N.call("zq_quantize_tokenwise", x.data_ptr(), B, d, d, 8, q.data_ptr(), q.stride(0), s.data_ptr(), flag.data_ptr(), N.stream_ptr())])
    res["ln_quant_d"] = graph_time([lambda: N.call("zq_layer_norm_quantize", x.data_ptr(), x.data_ptr(), g1.data_ptr(), b1.data_ptr(), B, d, 1e-5, 8, y.data_ptr(), q.data_ptr(), q.stride(0), s.data_ptr(), flag.data_ptr(), N.stream_ptr())])
    res["gelu_quant_f"] = graph_time([lambda: N.call("zq_gelu_quantize", u.data_ptr(), B, f, f, 8, None, q.data_ptr(), q.stride(0), s.data_ptr(), flag.data_ptr(), N.stream_ptr())])
    kc = torch.randn(B, 256, d, device="cuda")
    vc = torch.randn(B, 256, d, device="cuda")
    qkv = torch.randn(B, 3 * d, device="cuda")
    cx = torch.empty(B, d, device="cuda")
    lens = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    pos = torch.full((B,), ctx - 1, dtype=torch.int32, device="cuda")
    res["decode_attention"] = graph_time([lambda: N.call("zq_decode_attention_f32", qkv.data_ptr(), qkv.stride(0), kc.data_ptr(), vc.data_ptr(), 256, B, H, dh, lens.data_ptr(), 0.0625, cx.data_ptr(), cx.stride(0), 0, N.stream_ptr())])
    res["kv_append"] = graph_time([lambda: N.call("zq_kv_append", qkv.data_ptr(), qkv.stride(0), B, 1, d, pos.data_ptr(), kc.data_ptr(), vc.data_ptr(), 256, N.stream_ptr())])
    for nm, (n, k) in {"qkv": (3 * d, d), "o": (d, d), "h4h": (f, d), "4hh": (d, f)}.items():
        sets = []
        nset = max(2, int(2 * 126e6 // (n * k)) + 1)
        for _ in range(nset):
            w = quant.QuantizedMatrix(values=torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda"), bits=8,
                                      group_scales=torch.rand(1, device="cuda"), group_layout=[(0, n)])
            w.row_scales()
            sets.append(w)
        xq = quant.padded_int8(B, k)
        out = torch.empty(B, n, device="cuda")
        fs = [(lambda w=w: N.call("zq_linear", xq.data_ptr(), xq.stride(0), s.data_ptr(), 0.0, w.values.data_ptr(), w.ld, 8, w.row_scales().data_ptr(), None, B, n, k, out.data_ptr(), out.stride(0), N.OUT_F32, N.stream_ptr())) for w in sets]
        t = graph_time(fs)
        res[f"linear_{nm}"] = t
        res[f"linear_{nm}_GBps"] = n * k / t / 1e9
    E = torch.randn(cfg.vocab, d, device="cuda")
    hl = torch.randn(B, d, device="cuda")
    lg = torch.empty(B, cfg.vocab, device="cuda")
    res["lm_head_f32_cublas"] = graph_time([lambda: torch.matmul(hl, E.t(), out=lg)])
    print(json.dumps({k: (round(v * 1e6, 2) if not k.endswith("GBps") else round(v, 1)) for k, v in res.items()}))


if __name__ == "__main__":
    main()
