"""A few GPT decode steps (eager, no graph) for ncu launch lists:
python tools/profile_decode.py <gptj-6b|neox-20b|gpt3-350m> [layers]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200.decoder import CONFIGS, DecoderEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
eng = DecoderEngine(cfg, 16, 256, layers=layers, use_graph=False)
ids = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (16, 128))).cuda()
eng.prefill(ids)
for _ in range(3):
    eng.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("decode_step")
eng.step()
torch.cuda.synchronize()
