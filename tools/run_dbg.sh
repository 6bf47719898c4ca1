for d in 0 1 2 3; do echo "debug=$d"; ZQ_GEMM_DEBUG=$d timeout -s KILL 120 python tools/gemm_trace.py 2>&1 | head -1 | python -c "
import json,sys
r=json.loads(sys.stdin.read()); print(r['kernel_us'], [(round(t['epi_start'],2), round(t['epi_end'],2)) for t in r['tiles']])"; done
