# compute-sanitizer over the GPU suite's kernel tests (memcheck, racecheck,
# synccheck).  Usage: bash tools/run_sanitizer.sh TAG
TAG=${1:-san}
mkdir -p gpurun_out
T="tests/test_quant_gpu.py tests/test_igemm_gpu.py tests/test_attention_gpu.py tests/test_decoder_gpu.py tests/test_transformer_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 97 \
    python -m pytest $T -m gpu -q -p no:cacheprovider -x > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_${tool}.log
  tail -5 gpurun_out/${TAG}_${tool}.log
done
