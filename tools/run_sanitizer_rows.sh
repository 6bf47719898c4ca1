# compute-sanitizer over the row quantizers' tests (GeLU / LN / token quantize,
# packed f32x2 forms) and the engine forward.  Usage: bash tools/run_sanitizer_rows.sh TAG
TAG=${1:-san5}
mkdir -p gpurun_out
T="tests/test_quant_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 97 \
    python -m pytest $T -m gpu -q -p no:cacheprovider -x -k "gelu or layer_norm or ln or tokenwise or far_negative" > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_${tool}.log
  tail -3 gpurun_out/${TAG}_${tool}.log
done
