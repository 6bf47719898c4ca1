for L in $LIBS; do
echo "== $L"
ZQ_LIB=$PWD/$L timeout 300 python tools/row_graph_bench.py 2>&1 | grep -v "^$"
ZQ_LIB=$PWD/$L timeout 300 python bench.py --workload bert --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); rk=d.get('row_kernels',{}); print(d['value'], d['ms_per_step'], d['e2e']['value'], {k: round(v.get('in_graph_us_per_launch',0),2) for k,v in rk.items() if isinstance(v, dict)})"
done
