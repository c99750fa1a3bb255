timeout 300 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -1 gpurun_out/pytest_nd.log
timeout 120 python scripts/nd_flow_check.py 2>&1 | tail -10 | cut -c1-120
for tw in 1 2 4 8; do echo "TOP_WPR=$tw"; TVB_ND_TOP_WPR=$tw timeout 600 python scripts/nd_bench.py C4a 2>&1 | grep -v Warning | tail -1; done
timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"
timeout 300 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters']) for k,v in d.items()})"
