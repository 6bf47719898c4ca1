"""The packed f32x2 instructions the row kernels and epilogues use (FADD2 /
FMUL2 / FFMA2) give the scalar _rn results bit for bit (tools/f32x2_exactness.cu;
DESIGN.md §3).  NaN results compare by bit pattern, so a NaN payload difference
would show up as a mismatch too."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_packed_f32x2_matches_scalar(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "f32x2")
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-o", exe,
                    os.path.join(ROOT, "tools", "f32x2_exactness.cu")], check=True, capture_output=True)
    out = subprocess.run([exe], check=True, capture_output=True, text=True, timeout=120).stdout
    assert out.startswith("mismatch"), out
    counts = [int(t) for t in out.split("(")[0].split()[2::2]]
    assert len(counts) == 8 and all(c == 0 for c in counts), out
