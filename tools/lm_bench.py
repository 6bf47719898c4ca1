"""LM head (tied embedding, greedy argmax) timing at GPT-J / NeoX / GPT-3 350M
decode shapes: per-step conversion (zq_lm_head_argmax) vs pre-split embedding
(zq_lm_head_argmax_split); GB/s of embedding streamed."""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402

for name, ntok, vocab, dim in (("gpt3-350m", 8, 50257, 1024), ("gptj-6b", 16, 50400, 4096),
                               ("neox-20b", 16, 50432, 6144)):
    x = torch.randn(ntok, dim, device="cuda")
    emb = torch.randn(vocab, dim, device="cuda") * 0.02
    scale = math.ldexp(1.0, 15 - math.frexp(float(emb.abs().max()))[1])
    eh = torch.empty(vocab, dim, dtype=torch.float16, device="cuda")
    el = torch.empty_like(eh)
    N.call("zq_lm_embed_split", emb.data_ptr(), vocab, dim, scale, eh.data_ptr(), el.data_ptr(), N.stream_ptr())
    xh = torch.zeros(16 * dim, dtype=torch.float16, device="cuda")
    xl = torch.zeros_like(xh)
    xinv = torch.zeros(16, device="cuda")
    keys = torch.zeros(16, dtype=torch.int64, device="cuda")
    ids = torch.zeros(ntok, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for split in (False, True):
        def run():
            if split:
                N.call("zq_lm_head_argmax_split", x.data_ptr(), x.stride(0), ntok, eh.data_ptr(), el.data_ptr(), vocab,
                       dim, scale, xh.data_ptr(), xl.data_ptr(), xinv.data_ptr(), keys.data_ptr(), ids.data_ptr(),
                       N.stream_ptr())
            else:
                N.call("zq_lm_head_argmax", x.data_ptr(), x.stride(0), ntok, emb.data_ptr(), vocab, dim, scale,
                       xh.data_ptr(), xl.data_ptr(), xinv.data_ptr(), keys.data_ptr(), ids.data_ptr(), N.stream_ptr())
        ts = []
        for i in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        print(json.dumps({"case": name, "split": split, "us": round(us, 1),
                          "GBps": round(vocab * dim * 4 / us / 1e3, 1)}), flush=True)
