"""B200-native ZeroQuant quantized-inference hot path (arXiv 2206.01861).

Drop-in for the reference package's quantizer / quantized-linear API
(`lowbit.quant`, `lowbit.igemm`), computing in hand-written sm_100a kernels
(libzq_b200.so, C ABI in include/zq_b200.h).  No CPU fallback.
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401
from .errors import ShapeError, UsageError  # noqa: F401
