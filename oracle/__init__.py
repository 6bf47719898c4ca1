"""TEST INFRASTRUCTURE ONLY — CPU oracle for the ZeroQuant hot path.

This package is a numpy restatement of the reference `lowbit` package's
quantizer / integer-GEMM / quantize-on-write arithmetic (reference files cited
per function as `pkg/src/lowbit/<file>.py:<line>`).  It exists to *check* the
B200 CUDA path, never to *be* it:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
  `--impl reference` legs may import it;
* the product package `paper_2206_01861_b200` never imports it and has no CPU
  fallback.

Parity pinning: the restatement is checked against golden vectors produced by
the real reference (`oracle/make_golden.py`, committed fixtures under
`tests/golden/`) and against the reference's own known-answer tests (see
`tests/test_oracle_golden.py`).
"""
