"""GPT-3 350M decode steps (eager) at batch 8, context ~1030, for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200.decoder import CONFIGS, DecoderEngine  # noqa: E402

cfg = CONFIGS["gpt3-350m"]
eng = DecoderEngine(cfg, 8, 1040, layers=4, use_graph=False)
ids = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (8, 1024))).cuda()
eng.prefill(ids)
for _ in range(2):
    eng.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("decode_step")
eng.step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
