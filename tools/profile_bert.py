"""One eager BERT-base W8A8 forward (after a warm-up), for ncu captures of
the kernels exactly as the benchmark launches them."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

eng = bench.build_engine(torch)
eng._bufs["ids"].copy_(torch.randint(0, bench.BERT["vocab"], (eng.tokens,), device="cuda"))
eng._run()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled_forward")
eng._run()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
