"""GeLU+quantize timing probe: fast path vs the all-exact (gelu_out) path,
for several shapes and input scales (graph replay over > L2 buffer sets)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import quant  # noqa: E402
from tools.timing import graph_time, sets_needed  # noqa: E402


def main():
    f = quant.FiniteFlag()
    for (t, d) in [(4096, 3072), (4096, 768), (16, 24576)]:
        for std in (0.5, 1.0, 3.0):
            ns = sets_needed(5 * t * d)
            X = [torch.randn(t, d, device="cuda") * std for _ in range(ns)]
            Q = [quant.padded_int8(t, d) for _ in range(ns)]
            S = [torch.empty(t, device="cuda") for _ in range(ns)]
            G = [torch.empty(t, d, device="cuda") for _ in range(ns)]
            for exact in (False, True):
                def mk(i, exact=exact):
                    return lambda: N.call("zq_gelu_quantize", X[i].data_ptr(), t, d, d, 8,
                                          G[i].data_ptr() if exact else None, Q[i].data_ptr(), Q[i].stride(0),
                                          S[i].data_ptr(), f.ptr, N.stream_ptr())
                sec = graph_time([mk(i) for i in range(ns)])
                print(f"gelu {t}x{d} std {std} {'exact-all' if exact else 'fast'}: {sec * 1e6:.2f} us")


if __name__ == "__main__":
    main()
