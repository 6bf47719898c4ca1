# Run the reference's own hot-path unit suites (staged by
# oracle/stage_reference_suite.sh into oracle/_ref/suite/) against the B200
# drop-in (paper_2206_01861_b200.compat) on the GPU; log + pass count to
# gpurun_out/<TAG>_refsuite.log.   Usage: bash tools/run_reference_suite.sh TAG
TAG=${1:-refsuite}
mkdir -p gpurun_out
cd oracle/_ref/suite && PYTHONPATH=../../..:$PYTHONPATH timeout 900 python -m pytest -p oracle.lowbit_shim \
  -p no:cacheprovider -q -rf --rootdir . test_quant.py test_igemm.py > ../../../gpurun_out/${TAG}_refsuite.log 2>&1
echo rc=$? >> ../../../gpurun_out/${TAG}_refsuite.log
tail -15 ../../../gpurun_out/${TAG}_refsuite.log
