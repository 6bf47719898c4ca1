# A/B of library builds on one box: LIBS="exp/a.so exp/b.so ..." bash tools/run_ab.sh
# (alternate the builds, e.g. "a b a b").  Each build is loaded through ZQ_LIB
# (paper_2206_01861_b200/_native.py) for the row-kernel graph timings and one
# BERT bench line (value, ms/step, e2e, in-graph row-kernel costs).  Builds go
# under exp/ (git-ignored, not gpurun-ignored, so they travel to the box).
for L in $LIBS; do
echo "== $L"
ZQ_LIB=$PWD/$L timeout 300 python tools/row_graph_bench.py 2>&1 | grep -v "^$"
ZQ_LIB=$PWD/$L timeout 300 python bench.py --workload bert --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); rk=d.get('row_kernels',{}); print(d['value'], d['ms_per_step'], d['e2e']['value'], {k: round(v.get('in_graph_us_per_launch',0),2) for k,v in rk.items() if isinstance(v, dict)})"
done
