"""Kernel micro-benchmarks: graph replay over rotating buffer sets > L2.
Prints one JSON line per kernel with achieved GB/s (algorithmic bytes) or TOPS."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402
from tools.timing import graph_time, sets_needed  # noqa: E402


def calib_benches(res):
    """Harness calibration: a torch elementwise op of known traffic."""
    for n in (4096 * 768, 4096 * 3072):
        ns = sets_needed(8 * n)
        X = [torch.randn(n, device="cuda") for _ in range(ns)]
        Y = [torch.empty(n, device="cuda") for _ in range(ns)]
        sec = graph_time([(lambda i=i: torch.mul(X[i], 2.0, out=Y[i])) for i in range(ns)])
        res[f"calib_torch_mul_{n}"] = {"us": sec * 1e6, "GBps": 8 * n / sec / 1e9}


def quant_benches(res):
    for (t, d) in [(4096, 768), (4096, 3072), (16, 6144), (2048, 6144), (16, 24576)]:
        nb = 5 * t * d
        ns = sets_needed(nb)
        X = [torch.randn(t, d, device="cuda") for _ in range(ns)]
        Q = [quant.padded_int8(t, d) for _ in range(ns)]
        S = [torch.empty(t, device="cuda") for _ in range(ns)]
        f = quant.FiniteFlag()

        def mk(name, i):
            if name == "tok":
                return lambda: N.call("zq_quantize_tokenwise", X[i].data_ptr(), t, d, d, 8, Q[i].data_ptr(), Q[i].stride(0), S[i].data_ptr(), f.ptr, N.stream_ptr())
            return lambda: N.call("zq_gelu_quantize", X[i].data_ptr(), t, d, d, 8, None, Q[i].data_ptr(), Q[i].stride(0), S[i].data_ptr(), f.ptr, N.stream_ptr())

        for name in ("tok", "gelu"):
            sec = graph_time([mk(name, i) for i in range(ns)])
            res[f"{name}_quant_{t}x{d}"] = {"us": sec * 1e6, "GBps": (nb + 4 * t) / sec / 1e9}
        if d <= 8192:
            g = torch.ones(d, device="cuda")
            b = torch.zeros(d, device="cuda")
            ns2 = sets_needed(13 * t * d)
            R = [torch.randn(t, d, device="cuda") for _ in range(ns2)]
            Y = [torch.empty(t, d, device="cuda") for _ in range(ns2)]
            X2 = [torch.randn(t, d, device="cuda") for _ in range(ns2)]
            Q2 = [quant.padded_int8(t, d) for _ in range(ns2)]
            S2 = [torch.empty(t, device="cuda") for _ in range(ns2)]
            L = [(lambda i=i: N.call("zq_layer_norm_quantize", X2[i].data_ptr(), R[i].data_ptr(), g.data_ptr(), b.data_ptr(), t, d, 1e-5, 8, Y[i].data_ptr(), Q2[i].data_ptr(), Q2[i].stride(0), S2[i].data_ptr(), f.ptr, N.stream_ptr())) for i in range(ns2)]
            sec = graph_time(L)
            res[f"ln_res_quant_{t}x{d}"] = {"us": sec * 1e6, "GBps": (13 * t * d + 4 * t) / sec / 1e9}


SKINNY = [(16, 4096, 12288, 8, torch.float32), (16, 4096, 4096, 8, torch.float32),
          (16, 4096, 16384, 8, torch.float32), (16, 16384, 4096, 8, torch.float32),
          (16, 6144, 18432, 8, torch.float32), (16, 6144, 6144, 8, torch.float32),
          (16, 6144, 24576, 8, torch.float32), (16, 24576, 6144, 8, torch.float32)]


def gemm_benches(res, shapes=None):
    for (t, k, n, wb, od) in shapes or [(4096, 768, 3072, 8, torch.float16), (4096, 768, 3072, 8, torch.float32),
                              (4096, 768, 2304, 8, torch.float32), (4096, 768, 768, 8, torch.float32),
                              (4096, 3072, 768, 8, torch.float32), (8192, 8192, 8192, 8, torch.float16),
                              (4096, 4096, 16384, 8, torch.float16), (2048, 6144, 24576, 8, torch.float16),
                              (16, 6144, 24576, 8, torch.float16), (16, 4096, 4096, 8, torch.float16),
                              (4096, 768, 3072, 4, torch.float16), (1024, 1024, 4096, 4, torch.float32),
                              (1024, 4096, 1024, 4, torch.float32)]:
        esz = torch.tensor([], dtype=od).element_size()
        nb = t * k + n * k * wb // 8 + t * n * esz
        ns = sets_needed(nb, cap=24)
        sets = []
        for _ in range(ns):
            xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda"), bits=8,
                                           token_scales=torch.rand(t, device="cuda"))
            lo, hi = (-7, 8) if wb == 4 else (-127, 128)
            wq = quant.QuantizedMatrix(values=torch.randint(lo, hi, (n, k), dtype=torch.int8, device="cuda"), bits=wb,
                                       group_scales=torch.rand(1, device="cuda"), group_layout=[(0, n)])
            wq.row_scales()
            wq.weight_operand()
            out = torch.empty(t, n, dtype=od, device="cuda")
            sets.append((xq, wq, out))
        sec = graph_time([(lambda s=s: igemm.fused_linear(s[0], s[1], None, out=s[2])) for s in sets])
        ops = 2 * t * k * n
        res[f"linear_w{wb}_{t}x{k}x{n}_{str(od).split('.')[-1]}"] = {
            "us": sec * 1e6, "TOPS": ops / sec / 1e12, "GBps": nb / sec / 1e9}


def main():
    res = {}
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "quant"):
        calib_benches(res)
        quant_benches(res)
    if which in ("all", "gemm"):
        gemm_benches(res)
    if which == "skinny":
        gemm_benches(res, SKINNY)
    for k, v in res.items():
        print(k, json.dumps({a: round(b, 2) for a, b in v.items()}))


if __name__ == "__main__":
    main()
