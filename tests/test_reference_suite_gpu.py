"""GPU: the reference's OWN hot-path unit suites (pkg/tests/test_quant.py and
pkg/tests/test_igemm.py, unmodified) against the B200 drop-in.

oracle/stage_reference_suite.sh copies them (git-ignored) into
oracle/_ref/suite/, which travels to the GPU box with the snapshot; the
oracle/lowbit_shim.py plugin resolves `lowbit.quant` / `lowbit.igemm` to
paper_2206_01861_b200.compat (numpy in / out over the sm_100a kernels).  Skips
when the suite was not staged (e.g. a checkout without /root/reference)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "suite")


@pytest.mark.skipif(not os.path.exists(os.path.join(SUITE, "test_quant.py")),
                    reason="reference suite not staged (oracle/stage_reference_suite.sh)")
def test_reference_unit_suites_pass_on_the_drop_in():
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "oracle.lowbit_shim", "-p", "no:cacheprovider",
                        "-q", "-rf", "--rootdir", SUITE, "test_quant.py", "test_igemm.py"],
                       cwd=SUITE, env=env, capture_output=True, text=True, timeout=900)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
