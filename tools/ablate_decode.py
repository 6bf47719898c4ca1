"""In-graph cost of each kernel family of one GPT decode step (CUDA graph),
by capturing the step with one family stubbed out:
python tools/ablate_decode.py [gptj-6b|neox-20b|gpt3-350m] [batch prompt]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import decoder as D  # noqa: E402

FAMILIES = {
    "linear": ("zq_linear", "zq_linear_ws", "zq_linear_kv_ws"),
    "decode_attention": ("zq_decode_attention_f32",),
    "kv_append": ("zq_kv_append",),
    "ln": ("zq_layer_norm_quantize",),
    "gelu": ("zq_gelu_quantize",),
    "tok": ("zq_quantize_tokenwise",),
    "lm_head": ("zq_lm_head_argmax", "zq_lm_head_argmax_split"),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gptj-6b"
    cfg = D.CONFIGS[name]
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    prompt = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    eng = D.DecoderEngine(cfg, batch, prompt + 128)
    ids = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, (batch, prompt))).cuda()
    eng.prefill(ids)
    torch.cuda.synchronize()
    orig_call, orig_rc, orig_mm, orig_am = N.call, N.call_rc, torch.matmul, torch.argmax

    def timed(reps=20):
        eng._graph = None
        eng.pos.fill_(prompt)
        eng.host_pos = prompt
        eng.step()  # captures
        eng.pos.fill_(prompt)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            eng._graph.replay()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps * 1e3

    base = timed()
    print(f"{name} batch {batch} prompt {prompt} decode step: {base:.1f} us")
    for fam, names in FAMILIES.items():
        N.call = lambda n, *a, _names=names: None if n in _names else orig_call(n, *a)
        N.call_rc = lambda n, *a, _names=names: 0 if n in _names else orig_rc(n, *a)
        try:
            t = timed()
        finally:
            N.call, N.call_rc, torch.matmul, torch.argmax = orig_call, orig_rc, orig_mm, orig_am
        print(f"without {fam:17s}: {t:8.1f} us  -> in-graph cost {base - t:7.1f} us")


if __name__ == "__main__":
    main()
