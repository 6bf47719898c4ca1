"""Decode attention timing at the BASELINE decode shapes (GPT-3 350M batch 8 x
~1030 keys, GPT-J batch 16 x ~192, NeoX batch 16 x ~192): GB/s of K/V cache
read.  Each launch reads a different layer's cache (24 rotating layers, > L2),
as a decode step does.  ZQ_DEC_TMA=0 selects the register-load kernel; argv
chunk counts are swept (0 = the planner's choice)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402

CASES = [("gpt3-350m", 8, 16, 64, 1030, 1040), ("gptj-6b", 16, 16, 256, 192, 256),
         ("neox-20b", 16, 64, 96, 192, 256), ("neox-20b-tp8", 16, 8, 96, 192, 256),
         # head-major cache layout [batch*heads, max_ctx, dh] (one head per "sequence")
         ("gpt3-350m-hm", 128, 1, 64, 1030, 1040), ("gptj-6b-hm", 256, 1, 256, 192, 256),
         ("neox-20b-hm", 1024, 1, 96, 192, 256)]
if os.environ.get("HM_ONLY"):
    CASES = [c for c in CASES if c[0].endswith("-hm")]
chunk_list = [int(a) for a in sys.argv[1:]] or [0]

for name, batch, heads, dh, ctx_len, max_ctx in CASES:
    dl = heads * dh
    L = max(2, int(1.6e9 // (2 * batch * max_ctx * dl * 4)))
    kcs = [torch.randn(batch, max_ctx, dl, device="cuda") for _ in range(L)]
    vcs = [torch.randn(batch, max_ctx, dl, device="cuda") for _ in range(L)]
    q = torch.randn(batch, 3 * dl, device="cuda")
    lens = torch.full((batch,), ctx_len, dtype=torch.int32, device="cuda")
    out = torch.empty(batch, dl, device="cuda")
    for C in chunk_list:
        def run(i):
            N.call("zq_decode_attention_f32", q.data_ptr(), q.stride(0), kcs[i % L].data_ptr(), vcs[i % L].data_ptr(),
                   max_ctx, batch, heads, dh, lens.data_ptr(), dh ** -0.5, out.data_ptr(), out.stride(0), C,
                   N.stream_ptr())

        for i in range(5):
            run(i)
        g = torch.cuda.CUDAGraph()
        n = 2 * L
        with torch.cuda.graph(g):
            for i in range(n):
                run(i)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / n * 1e3
        nbytes = 2 * batch * ctx_len * dl * 4
        print(json.dumps({"case": name, "tma": os.environ.get("ZQ_DEC_TMA", "1"), "kt": os.environ.get("ZQ_DEC_KT", ""),
                          "chunks": C or int(N.load().zq_decode_attention_chunks(batch, heads, max_ctx)),
                          "layers": L, "us": round(us, 2), "GBps": round(nbytes / us / 1e3, 1)}), flush=True)
    del kcs, vcs
    torch.cuda.empty_cache()
