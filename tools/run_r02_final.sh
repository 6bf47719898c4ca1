# Round-2 evidence on one GPU: tests, smoke, the default bench, the reference
# arm, the ncu launch list of the default bench's BERT timed region, ncu --set
# full of one BERT forward's first block and of the north-star kernels
# (tools/profile_kernels.py).  Usage: bash tools/run_r02_final.sh TAG
TAG=${1:-r02z}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 400 --csv --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --workload bert --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --nvtx --nvtx-include "profiled_forward/" -c 12 -o gpurun_out/${TAG}_bert_full python tools/profile_bert.py > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled --nvtx --nvtx-include "prof/" -o gpurun_out/${TAG}_kernels_full python tools/profile_kernels.py > gpurun_out/${TAG}_ncu_kernels.log 2>&1
# keep the copy-back under 64 MiB: raw metric CSVs of the captures, reports to /tmp
for r in bert_full kernels_full; do
  if [ -f gpurun_out/${TAG}_${r}.ncu-rep ]; then
    ncu -i gpurun_out/${TAG}_${r}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>/dev/null
    ncu -i gpurun_out/${TAG}_${r}.ncu-rep --page details --csv > gpurun_out/${TAG}_${r}_details.csv 2>/dev/null
    mv gpurun_out/${TAG}_${r}.ncu-rep /tmp/
  fi
done
tail -2 gpurun_out/${TAG}_pytest.log
