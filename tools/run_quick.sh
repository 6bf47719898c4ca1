# Quick GPU check: tests, smoke, default bench, per-tile GEMM trace at BERT shapes.
# Usage: bash tools/run_quick.sh TAG [skip-tests]
TAG=${1:-q}
mkdir -p gpurun_out
if [ "$2" != "skip-tests" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python tools/gemm_trace.py > gpurun_out/${TAG}_trace.jsonl 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
