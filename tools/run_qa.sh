# Fused QKV + attention: parity tests, kernel timing, BERT bench with the fusion on / off.
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_qkv_attention_gpu.py -x -q -p no:cacheprovider > gpurun_out/qa_pytest.log 2>&1; echo rc=$? >> gpurun_out/qa_pytest.log
timeout 120 python tools/qkv_att_bench.py > gpurun_out/qa_bench.log 2>&1; timeout 60 python tools/qa_trace.py > gpurun_out/qa_trace.log 2>&1
for f in 1 0 1 0; do
  ZQ_FUSE_QKV=$f timeout 300 python bench.py --steps 20 --warmup 5 --workload bert > gpurun_out/qa_b$f.json 2>>gpurun_out/qa_b.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/qa_b$f.json').read().strip().splitlines()[-1]); print('fuse=$f', d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))"
done
tail -3 gpurun_out/qa_pytest.log; cat gpurun_out/qa_bench.log
cat gpurun_out/qa_trace.log
