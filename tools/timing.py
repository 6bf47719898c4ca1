"""Device timing helpers: CUDA-graph replay over rotating buffer sets whose
total footprint exceeds L2 (so every launch reads from HBM), timed with CUDA
events on the launching stream."""

from __future__ import annotations

import torch

L2_BYTES = 126 * 1024 * 1024


def sets_needed(bytes_per_set: int, min_total: int = 2 * L2_BYTES, cap: int = 64) -> int:
    return max(2, min(cap, -(-min_total // max(1, bytes_per_set))))


def graph_time(launches, reps: int = 5, warm: int = 3) -> float:
    """launches: list of zero-arg callables (one per buffer set).  Captures one
    pass over all of them in a CUDA graph and returns seconds per launch
    (median over `reps` replays)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(warm):
            for f in launches:
                f()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    inner = max(1, -(-20 // len(launches)))  # >= 20 launches per replay: amortise the graph launch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            for f in launches:
                f()
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e-3 / (inner * len(launches)))
    out.sort()
    return out[len(out) // 2]
