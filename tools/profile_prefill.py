"""One GPT prefill (eager) for ncu launch lists: python tools/profile_prefill.py <name> [batch] [T] [layers]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200.decoder import CONFIGS, DecoderEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gpt3-350m"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
layers = int(sys.argv[4]) if len(sys.argv) > 4 else 2
cfg = CONFIGS[name]
eng = DecoderEngine(cfg, batch, T + 8, layers=layers, use_graph=False)
ids = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (batch, T))).cuda()
eng.prefill(ids)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prefill")
eng.prefill(ids)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
