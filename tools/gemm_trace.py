"""Per-CTA timeline of the fused linear (globaltimer stamps), to see where a
tile's time goes: operand arrival vs MMA vs epilogue."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_01861_b200 import _native as N  # noqa: E402
from paper_2206_01861_b200 import igemm, quant  # noqa: E402


def run(t, k, n, od=torch.float32):
    xq = quant.QuantizedActivation(values=torch.randint(-127, 128, (t, k), dtype=torch.int8, device="cuda"),
                                   bits=8, token_scales=torch.rand(t, device="cuda"))
    wq = quant.QuantizedMatrix(values=torch.randint(-127, 128, (n, k), dtype=torch.int8, device="cuda"), bits=8,
                               group_scales=torch.rand(1, device="cuda"), group_layout=[(0, n)])
    out = torch.empty(t, n, dtype=od, device="cuda")
    for _ in range(3):
        igemm.fused_linear(xq, wq, None, out=out)
    buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    N.call("zq_gemm_set_trace", buf.data_ptr())
    igemm.fused_linear(xq, wq, None, out=out)
    torch.cuda.synchronize()
    N.call("zq_gemm_set_trace", None)
    tr = buf.view(148, 64).cpu().numpy().astype(np.int64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = np.where(tr > 0, tr - t0, -1) / 1000.0  # us
    end = rel[:, 63].max()
    res = {"shape": [t, k, n], "kernel_us": float(end), "setup_us_med": float(np.median(rel[:, 1]))}
    tiles = []
    for lt in range(15):
        a = rel[:, 2 + 4 * lt]
        if (a >= 0).sum() == 0:
            break
        m = a >= 0
        tiles.append({"tile": lt, "ctas": int(m.sum()),
                      "mma_start": float(np.median(a[m])), "operands_done": float(np.median(rel[m, 3 + 4 * lt])),
                      "epi_start": float(np.median(rel[m, 4 + 4 * lt])), "epi_end": float(np.median(rel[m, 5 + 4 * lt]))})
    res["tiles"] = tiles
    print(json.dumps(res))


if __name__ == "__main__":
    for shp in [(4096, 768, 3072), (4096, 768, 768), (4096, 3072, 768), (4096, 768, 2304), (8192, 8192, 8192)]:
        run(*shp)
