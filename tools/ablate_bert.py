"""In-graph cost of each kernel family of the BERT-base forward: capture the
forward with one family stubbed out (no launch) and compare graph replay times
(L2 flushed before every replay, outside the events).  Delta vs the full graph =
that family's share of the step as it runs inside the graph (PDL overlaps
included) — numbers ncu's serialised launch lists cannot give."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2206_01861_b200 import transformer as T  # noqa: E402


def time_graph(eng, reps=20):
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    g = eng.capture()
    ts = []
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def qkv_ablation(eng):
    """In-graph cost of QKV projection + attention: fused kernel vs the two kernels."""
    d = eng.embedding.shape[1]
    orig_lin, orig_att, orig_fused = eng._linear, T.attention, eng._qkv_attention
    for fused in (True, False):
        eng._fuse_qkv = fused
        eng._graph = None
        base = time_graph(eng)
        if fused:
            eng._qkv_attention = lambda *a, **k: True
        else:
            eng._linear = lambda q, s, w, b, o: None if w.rows == 3 * d else orig_lin(q, s, w, b, o)
            T.attention = lambda *a, **k: None
        eng._graph = None
        t = time_graph(eng)
        eng._linear, T.attention, eng._qkv_attention = orig_lin, orig_att, orig_fused
        print(f"{'fused' if fused else 'two-kernel'} QKV+attention: forward {base * 1e3:.1f} us, without "
              f"{t * 1e3:.1f} us -> in-graph cost {(base - t) * 1e3:.1f} us ({(base - t) * 1e3 / len(eng.blocks):.2f} per layer)")
    eng._fuse_qkv = True
    eng._graph = None


def main():
    eng = bench.build_engine(torch)
    eng._bufs["ids"].copy_(torch.randint(0, bench.BERT["vocab"], (eng.tokens,), device="cuda"))
    if len(sys.argv) > 1 and sys.argv[1] == "qkv":
        qkv_ablation(eng)
        return
    base = time_graph(eng)
    print(f"full forward: {base * 1e3:.1f} us")
    noop = lambda *a, **k: None  # noqa: E731
    orig_att = T.attention
    for name in ("linear", "attention", "gelu", "ln", "tok"):
        saved = {}
        if name == "attention":
            T.attention = noop
        else:
            attr = {"linear": "_linear", "gelu": "_gelu_quant", "ln": "_ln_quant", "tok": "_tok_quant"}[name]
            saved[attr] = getattr(eng, attr)
            setattr(eng, attr, noop)
        t = time_graph(eng)
        T.attention = orig_att
        for k, v in saved.items():
            setattr(eng, k, v)
        print(f"without {name:9s}: {t * 1e3:.1f} us  -> in-graph cost {(base - t) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
