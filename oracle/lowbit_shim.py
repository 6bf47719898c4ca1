"""TEST INFRASTRUCTURE ONLY — pytest plugin that makes `import lowbit` resolve
to the B200 drop-in, so the reference's own unit suites run unmodified
against it (tools/run_reference_suite.sh).

  lowbit.quant   -> paper_2206_01861_b200.compat.quant   (the product, numpy API)
  lowbit.igemm   -> paper_2206_01861_b200.compat.igemm   (the product, numpy API)
  lowbit.errors  -> paper_2206_01861_b200.errors
  lowbit.tensor  -> the oracle's restatement of pkg/src/lowbit/tensor.py (the
                    float primitives the suites use as their own oracle:
                    matmul, layer_norm, gelu, softmax, Rng)
"""

import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import lowbit_oracle as O  # noqa: E402
from paper_2206_01861_b200 import errors  # noqa: E402
from paper_2206_01861_b200.compat import igemm, quant  # noqa: E402

F32 = np.float32


def _as_f32(data, shape=None):
    arr = np.ascontiguousarray(data, dtype=F32)
    return arr.reshape(shape) if shape is not None else arr


def _layer_norm(x, gamma, beta, eps=1e-5):
    return O.layer_norm_numpy(_as_f32(x), _as_f32(gamma), _as_f32(beta), eps)


tensor = types.ModuleType("lowbit.tensor")
tensor.F32 = F32
tensor.as_f32 = _as_f32
tensor.matmul = lambda a, b: O.matmul_f32(a, b)
tensor.layer_norm = _layer_norm
tensor.gelu = O.gelu
tensor.softmax = O.softmax
tensor.Rng = O.Rng

pkg = types.ModuleType("lowbit")
pkg.__path__ = []
pkg.quant, pkg.igemm, pkg.errors, pkg.tensor = quant, igemm, errors, tensor
sys.modules.update({"lowbit": pkg, "lowbit.quant": quant, "lowbit.igemm": igemm, "lowbit.errors": errors,
                    "lowbit.tensor": tensor})
