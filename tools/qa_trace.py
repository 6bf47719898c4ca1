"""Per-unit phase timeline of the fused QKV + attention kernel (globaltimer).
Usage: python tools/qa_trace.py [batch seq heads]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402

batch, seq, heads = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 128, 12)))
d = 64 * heads
t = batch * seq
xq = quant.quantize_activation_tokenwise(torch.randn(t, d, device="cuda"), 8)
w = quant.quantize_weight_groupwise(torch.randn(3 * d, d, device="cuda") * 0.05, 48, 8)
bias = torch.randn(3 * d, device="cuda") * 0.1
ctx = torch.empty(t, d, device="cuda")
wp, ldw, _ = w.weight_operand()
rs = w.row_scales()
scale = float(np.float32(1 / math.sqrt(64)))


def fused():
    N.call("zq_qkv_attention", xq.values.data_ptr(), xq.values.stride(0), xq.token_scales.data_ptr(), wp, ldw,
           rs.data_ptr(), bias.data_ptr(), batch, seq, heads, 64, 0, scale, ctx.data_ptr(), ctx.stride(0),
           N.stream_ptr())


for _ in range(5):
    fused()
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
N.call("zq_attention_set_trace", buf.data_ptr())
fused()
torch.cuda.synchronize()
N.call("zq_attention_set_trace", None)
tr = buf.view(148, 64).cpu().numpy().astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()


def med(x):
    x = x[x > 0]
    return round(float(np.median((x - t0) / 1e3)), 2) if x.size else None


print(f"[{batch}x{seq}x{heads}] ctas {len(tr)} start spread {(tr[:, 0].max() - t0) / 1e3:.2f} us")
print("pdl_wait done", med(tr[:, 1]), "first acc", med(tr[:, 2]), "prologue done", med(tr[:, 3]))
for u in range(4):
    print(f"unit {u}: producer first load {med(tr[:, 60 + u])}  mma first stage {med(tr[:, 52 + u])}"
          f"  mma last stage {med(tr[:, 56 + u])}")
names = ["start", "S ready", "P written", "acc(nxt)", "split(nxt) done", "PV done", "end", "loop top"]
ends = []
for it in range(6):
    row = tr[:, 8 + it * 8: 8 + it * 8 + 8]
    if not (row[:, 0] > 0).any():
        break
    print(f"iter {it} ctas {(row[:, 0] > 0).sum()}", {n: med(row[:, i]) for i, n in enumerate(names)})
    e = row[:, 6][row[:, 6] > 0]
    ends.append(((e - t0) / 1e3).max())
print("kernel span (last iteration end) us", round(max(ends), 2))
ss = tr[:, 40:46]
if (ss[:, 0] > 0).any():
    print("epi_split(unit 1) stamps: ld done, dequant+max, bars+scales, Q/K split, V^T, end:",
          [med(ss[:, i]) for i in range(6)])
