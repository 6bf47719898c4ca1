"""Time the fused attention kernel at the BERT-base shape (32 x 128 tokens,
12 heads x 64) with CUDA-graph replay over rotating buffers > L2."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import transformer as T  # noqa: E402
from tools.timing import graph_time, sets_needed  # noqa: E402


def main():
    batch, seq, heads, dh = 32, 128, 12, 64
    d = heads * dh
    t = batch * seq
    nb = t * 3 * d * 4 + t * d * 4
    ns = sets_needed(nb)
    Q = [torch.randn(t, 3 * d, device="cuda") for _ in range(ns)]
    C = [torch.empty(t, d, device="cuda") for _ in range(ns)]
    for causal in (False, True):
        fs = [(lambda i=i: T.attention(Q[i][:, :d], Q[i][:, d:2 * d], Q[i][:, 2 * d:], heads, causal, batch,
                                       out=C[i])) for i in range(ns)]
        sec = graph_time(fs)
        print(json.dumps({"kernel": "attention", "causal": causal, "us": round(sec * 1e6, 2),
                          "GBps": round(nb / sec / 1e9, 1)}))


if __name__ == "__main__":
    main()


def long_seq():
    """GPT-3 350M prefill attention: batch 8, seq 1024, 16 heads x 64, causal."""
    batch, seq, heads, dh = 8, 1024, 16, 64
    d = heads * dh
    t = batch * seq
    q = torch.randn(t, 3 * d, device="cuda")
    c = torch.empty(t, d, device="cuda")
    sec = graph_time([lambda: T.attention(q[:, :d], q[:, d:2 * d], q[:, 2 * d:], heads, True, batch, out=c)])
    import torch.nn.functional as F
    hq = lambda z: z.reshape(batch, seq, heads, dh).transpose(1, 2)  # noqa: E731
    sec2 = graph_time([lambda: F.scaled_dot_product_attention(hq(q[:, :d]), hq(q[:, d:2 * d]), hq(q[:, 2 * d:]),
                                                              is_causal=True)])
    print(json.dumps({"kernel": "attention_long", "seq": seq, "us": round(sec * 1e6, 1),
                      "torch_sdpa_f32_us": round(sec2 * 1e6, 1)}))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "long":
    long_seq()
