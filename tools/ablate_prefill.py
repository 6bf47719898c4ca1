"""In-stream cost of each kernel family of one GPT prefill (eager launches, CUDA
events), by running the prefill with one family stubbed out:
python tools/ablate_prefill.py [gpt3-350m|gptj-6b|neox-20b] [batch prompt]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import decoder as D  # noqa: E402

FAMILIES = {
    "linear": ("zq_linear", "zq_linear_ws", "zq_linear_kv_ws"),
    "attention": ("zq_attention_f32",),
    "kv_append": ("zq_kv_append",),
    "ln": ("zq_layer_norm_quantize",),
    "gelu": ("zq_gelu_quantize",),
    "tok": ("zq_quantize_tokenwise",),
    "lm_head": ("zq_lm_head_argmax", "zq_lm_head_argmax_split"),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt3-350m"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    prompt = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    cfg = D.CONFIGS[name]
    eng = D.DecoderEngine(cfg, batch, prompt + 16)
    ids = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (batch, prompt))).cuda()
    orig_call = N.call

    def timed(reps=3):
        eng.prefill(ids)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            eng.prefill(ids)
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps * 1e3

    base = timed()
    print(f"{name} batch {batch} prompt {prompt} prefill: {base:.1f} us")
    for fam, names in FAMILIES.items():
        N.call = lambda n, *a, _names=names: None if n in _names else orig_call(n, *a)
        try:
            t = timed()
        finally:
            N.call = orig_call
        print(f"without {fam:10s}: {t:9.1f} us  -> cost {base - t:8.1f} us")


if __name__ == "__main__":
    main()
