# compute-sanitizer over the round-2 kernels' tests: converted-weight pairs
# (W4A8 / weight-only), stream-K decode GEMM, TMA decode attention, pre-split LM
# head, the fused QKV + attention kernel, the pair GEMM (first-tile dry run).
# Usage: bash tools/run_sanitizer_r02.sh TAG
TAG=${1:-san2}
mkdir -p gpurun_out
T="tests/test_wo_gpu.py tests/test_igemm_gpu.py tests/test_decoder_gpu.py tests/test_qkv_attention_gpu.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 97 \
    python -m pytest $T -m gpu -q -p no:cacheprovider -x -k "not large_vs_float64" > gpurun_out/${TAG}_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_${tool}.log
  tail -4 gpurun_out/${TAG}_${tool}.log
done
