#!/bin/sh
# TEST INFRASTRUCTURE: stage the reference's own hot-path unit suites
# (pkg/tests/test_quant.py, pkg/tests/test_igemm.py and their conftest.py) into
# the git-ignored oracle/_ref/suite/, which travels to the GPU box with the
# gpurun snapshot (the box has no /root/reference).  They are run UNMODIFIED
# against the B200 drop-in by tools/run_reference_suite.sh, with `lowbit.quant`
# / `lowbit.igemm` resolved to paper_2206_01861_b200.compat (see
# oracle/lowbit_shim.py).  Nothing here is committed.
set -e
REF=${REF:-/root/reference/pkg/tests}
DST=$(dirname "$0")/_ref/suite
mkdir -p "$DST"
cp "$REF/test_quant.py" "$REF/test_igemm.py" "$REF/conftest.py" "$DST/"
echo "staged $(ls "$DST" | wc -l) files into $DST"
