# Round-end style check on one GPU: tests, smoke, every bench workload, the
# reference arm, and the ncu evidence (launch list of the default bench command,
# --set full of one BERT forward's first block).  Usage: bash tools/run_round_check.sh TAG
TAG=${1:-r01e}
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${TAG}_smoke.log
for w in bert c1 gpt3-350m gptj-6b neox-20b; do timeout 600 python bench.py --workload $w > gpurun_out/${TAG}_$w.json 2> gpurun_out/${TAG}_$w.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2>&1
timeout 300 python tools/ablate_bert.py > gpurun_out/${TAG}_ablate.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 400 --csv --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --nvtx --nvtx-include "profiled_forward/" -c 9 -o gpurun_out/${TAG}_bert_full python tools/profile_bert.py > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
