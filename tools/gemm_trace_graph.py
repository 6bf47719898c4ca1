"""Per-tile timeline of one BERT linear inside the captured forward graph (the
trace pointer is a launch argument: set around the chosen call during capture).
Usage: python tools/gemm_trace_graph.py [o|h4h|4hh] [layer]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2206_01861_b200 import _native as N  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "h4h"
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 11
eng = bench.build_engine(torch)
eng._bufs["ids"].copy_(torch.randint(0, bench.BERT["vocab"], (eng.tokens,), device="cuda"))
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
blk = eng.blocks[layer]
target = {"o": blk.w_o, "h4h": blk.w_h4h, "4hh": blk.w_4hh}[which]
orig = eng._linear


def traced(q, s, w, b, o):
    if w is target:
        N.call("zq_gemm_set_trace", buf.data_ptr())
        orig(q, s, w, b, o)
        N.call("zq_gemm_set_trace", None)
    else:
        orig(q, s, w, b, o)


eng._linear = traced
g = eng.capture()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for _ in range(3):
    g.replay()
flush.zero_()
buf.zero_()
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
tr = buf.view(148, 64).cpu().numpy().astype(np.int64)
t0 = tr[:, 0][tr[:, 0] > 0].min()
rel = np.where(tr > 0, tr - t0, -1) / 1000.0
print(f"{which} layer {layer}: kernel end {rel[:, 63].max():.2f} us, setup med {np.median(rel[:, 1][rel[:, 1] >= 0]):.2f}")
for lt in range(15):
    a = rel[:, 2 + 4 * lt]
    m = a >= 0
    if not m.any():
        break
    ms, od, es, ee = (np.median(rel[m, 2 + 4 * lt + i]) for i in range(4))
    print(f"  tile {lt} ctas {m.sum()}: mma {ms:.2f} operands {od:.2f} epi {es:.2f} -> {ee:.2f} (epi {ee - es:.2f} us)")
