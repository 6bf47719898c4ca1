"""numpy-in / numpy-out drop-in for the reference's `lowbit.quant` and
`lowbit.igemm` (pkg/src/lowbit/quant.py, pkg/src/lowbit/igemm.py).

A caller of the reference switches with

    from paper_2206_01861_b200.compat import quant, igemm

and keeps its numpy arrays, containers (`QuantizedMatrix`,
`QuantizedActivation`, `IntAccumulator` as numpy dataclasses with the
reference's fields) and error classes; every quantization, integer GEMM,
epilogue and fused LayerNorm / GeLU quantizer runs on the sm_100a kernels of
libzq_b200.so (through the device modules `paper_2206_01861_b200.quant` /
`.igemm`), and results come back as numpy arrays, bit-identical to the
reference.  Device-resident callers use the device modules directly.
"""

from . import igemm, quant  # noqa: F401
