"""Per-head phase timeline of the persistent attention kernel (globaltimer)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import transformer as T  # noqa: E402

batch, seq, heads, dh = 32, 128, 12, 64
d = heads * dh
qkv = torch.randn(batch * seq, 3 * d, device="cuda")
ctx = torch.empty(batch * seq, d, device="cuda")
for _ in range(3):
    T.attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], heads, False, batch, out=ctx)
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
N.call("zq_attention_set_trace", buf.data_ptr())
T.attention(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], heads, False, batch, out=ctx)
torch.cuda.synchronize()
N.call("zq_attention_set_trace", None)
tr = buf.view(148, 8, 8).cpu().numpy()
t0 = tr[:, 0, 0].min()
valid = tr[:, :, 0] > 0
end = (tr[:, :, 6][valid] - t0).max() / 1e3
print("kernel span us", end)
for it in range(4):
    m = tr[:, it, 0] > 0
    if not m.any():
        break
    ph = (np.diff(tr[m, it, :7], axis=1)) / 1e3
    print(f"iter {it} ctas {m.sum()} start {np.median(tr[m, it, 0] - t0) / 1e3:.2f} phases(wait, split, S, softmax, PV, store)",
          np.median(ph, axis=0).round(2).tolist())
