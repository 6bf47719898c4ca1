"""CPU: host-side logic of the product package (no GPU): scheme parsing,
group defaults, layouts, error taxonomy, and that the C-ABI library exports
every symbol include/zq_b200.h declares."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_scheme_parsing():
    from paper_2206_01861_b200.transformer import ActivationMode, PrecisionConfig

    cases = [("W16A16", None, None, ActivationMode.FULL), ("W8A16", 8, 8, ActivationMode.FULL),
             ("W8A8", 8, 8, ActivationMode.INT8), ("W4/8A16", 8, 4, ActivationMode.FULL),
             ("W4/8A8", 8, 4, ActivationMode.INT8), ("W8A8/16", 8, 8, ActivationMode.INT8_ATTN_FULL)]
    for label, mhsa, ffc, mode in cases:  # test_transformer.py:60-76
        p = PrecisionConfig.from_scheme(label)
        assert (p.mhsa_weight_bits, p.ffc_weight_bits, p.activation_mode) == (mhsa, ffc, mode)
        assert p.label() == label


@pytest.mark.parametrize("bad", ["W2A8", "A8", "W8", "W8A3", "8A8", "W4A8"])
def test_malformed_scheme(bad):
    from paper_2206_01861_b200.errors import UsageError
    from paper_2206_01861_b200.transformer import PrecisionConfig

    with pytest.raises(UsageError):
        PrecisionConfig.from_scheme(bad)


def test_group_defaults_and_alignment():
    from paper_2206_01861_b200.transformer import default_group_count, hw_aligned

    assert [default_group_count(d) for d in (768, 512, 1024, 2048, 64)] == [48, 48, 64, 128, 16]
    assert hw_aligned(768, 48) and not hw_aligned(64, 16) and hw_aligned(256, 16)


def test_precision_validation():
    from paper_2206_01861_b200.errors import UsageError
    from paper_2206_01861_b200.transformer import ActivationMode, PrecisionConfig

    with pytest.raises(UsageError):
        PrecisionConfig(mhsa_weight_bits=8, ffc_weight_bits=None)
    with pytest.raises(UsageError):
        PrecisionConfig(8, 8, ActivationMode.FULL, activation_static=True)


def test_group_layout_and_quantspec():
    from paper_2206_01861_b200 import quant
    from paper_2206_01861_b200.errors import UsageError

    assert quant.group_layout_for(4, 2) == [(0, 2), (2, 2)]
    assert quant.group_layout_for(5, 2) == [(0, 2), (2, 3)]
    with pytest.raises(UsageError):
        quant.group_layout_for(4, 5)
    with pytest.raises(UsageError):
        quant.QuantSpec(bits=8, granularity=quant.Granularity.PER_GROUP, for_weights=False)
    with pytest.raises(UsageError):
        quant.QuantSpec(bits=8, granularity=quant.Granularity.PER_TOKEN, for_weights=True)
    with pytest.raises(UsageError):
        quant.QuantSpec(bits=8, granularity=quant.Granularity.PER_TOKEN, mode=quant.Mode.STATIC,
                        for_weights=False)
    quant.QuantSpec(bits=8, granularity=quant.Granularity.PER_TENSOR, mode=quant.Mode.STATIC)
    assert quant.qmax(8) == 127 and quant.qmax(4) == 7


def test_overflow_guard_host():
    from paper_2206_01861_b200 import igemm
    from paper_2206_01861_b200.errors import UsageError

    igemm.check_overflow_guard(133000, 8, 8)
    with pytest.raises(UsageError):
        igemm.check_overflow_guard(140000, 8, 8)


def test_calibrator_host_rules():
    from paper_2206_01861_b200 import quant
    from paper_2206_01861_b200.errors import UsageError

    with pytest.raises(UsageError):
        quant.Calibrator(momentum=1.0)
    with pytest.raises(UsageError):
        quant.Calibrator().finalize(8)


def test_product_path_fails_loudly_without_gpu():
    import torch

    from paper_2206_01861_b200 import _native

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    _native._lib = None
    with pytest.raises(_native.NativeUnavailable):
        _native.load()


def test_library_exports_every_header_symbol():
    from paper_2206_01861_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("library not built (run __graft_entry__.build())")
    with open(os.path.join(ROOT, "include", "zq_b200.h")) as f:
        header = f.read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(zq_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    lib = _native.load_for_inspection()
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert declared == set(_native.exported_symbols())


def test_scale_double_rounding_equals_f32_division():
    import numpy as np

    """The device computes token / group scales as one IEEE f32 division
    (zq_common.cuh scale_from_absmax); the reference does f32(f64(a) / qmax)
    (quant.py:80-95).  The two agree for every f32 a and odd qmax: checked on
    random bit patterns over the whole positive range, subnormals included."""
    rng = np.random.default_rng(0)
    bits = rng.integers(1, 0x7F7FFFFF, 4_000_000, dtype=np.uint32)
    a = bits.view(np.float32)
    for qm in (127, 7):
        ref = (a.astype(np.float64) / qm).astype(np.float32)
        dev = a / np.float32(qm)
        assert np.array_equal(ref.view(np.uint32), dev.view(np.uint32)), qm


def test_no_global_load_scheduled_before_the_grid_dependency_wait():
    """Programmatic dependent launch: a kernel may start while its predecessor
    still runs, so reads of the predecessor's output must come after
    griddepcontrol.wait (SASS ACQBULK).  ptxas treats non-coherent loads as
    invariant and once scheduled two of tok_quant_kernel<16, 256>'s row loads
    above the wait: scan every kernel of the built library for an LDG before its
    first ACQBULK.  Allowed: decode attention's lens[b] (written by a non-PDL
    torch op at the start of the step, before any kernel of the step)."""
    import shutil
    import subprocess

    lib = os.path.join(ROOT, "paper_2206_01861_b200", "libzq_b200.so")
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(lib) or not os.path.exists(cuobjdump):
        pytest.skip("library or cuobjdump not available")
    sass = subprocess.run([cuobjdump, "-sass", lib], capture_output=True, text=True, check=True).stdout
    offenders = []
    name, seen_wait, early = None, False, 0
    for line in sass.splitlines() + ["Function : <end>"]:
        if "Function :" in line:
            if name and seen_wait and early and "decode_attention_tma_kernel" not in name:
                offenders.append((name, early))
            name, seen_wait, early = line.split("Function :")[1].strip(), False, 0
        elif "ACQBULK" in line:
            seen_wait = True
        elif re.search(r"\sLDG\.E", line) and not seen_wait:
            early += 1
    assert not offenders, offenders
