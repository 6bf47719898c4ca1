set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01d_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r01d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01d_smoke.log 2>&1; echo smoke=$? >> gpurun_out/r01d_smoke.log
for w in bert c1 gpt3-350m gptj-6b neox-20b; do timeout 600 python bench.py --workload $w > gpurun_out/r01d_$w.json 2> gpurun_out/r01d_$w.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01d_ref.json 2>&1
tail -2 gpurun_out/r01d_pytest.log
