"""Phase timeline of the fused QKV + attention kernel inside the BERT forward
graph (the trace buffer is captured as a kernel argument: the last layer's
launch is the one left in it).  L2 flushed before the replay, as the bench."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2206_01861_b200 import _native as N  # noqa: E402

eng = bench.build_engine(torch)
eng._bufs["ids"].copy_(torch.randint(0, bench.BERT["vocab"], (eng.tokens,), device="cuda"))
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
N.call("zq_attention_set_trace", buf.data_ptr())
g = eng.capture()
N.call("zq_attention_set_trace", None)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    g.replay()
flush.zero_()
buf.zero_()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
tr = buf.view(148, 64).cpu().numpy().astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()


def med(x):
    x = x[x > 0]
    return round(float(np.median((x - t0) / 1e3)), 2) if x.size else None


print(f"ctas {len(tr)} start spread {(tr[:, 0].max() - t0) / 1e3:.2f} us (p50 {med(tr[:, 0])})")
print("pdl_wait done", med(tr[:, 1]), "max", round((tr[:, 1].max() - t0) / 1e3, 2), "first acc", med(tr[:, 2]),
      "prologue done", med(tr[:, 3]))
for u in range(3):
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
    print("epi_split(unit 1): ld done, dequant+max, bars, Q/K, V^T, end:", [med(ss[:, i]) for i in range(6)])
