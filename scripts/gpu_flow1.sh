mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -3 gpurun_out/pytest_nd.log
for fl in 1 0; do
 for tm in 600 1200 2400 4608; do
  echo "FLOW=$fl TOP_MAX=$tm"; TVB_ND_FLOW=$fl TVB_ND_TOP_MAX=$tm timeout 120 python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"
 done
done
for tm in 1200 4608; do
TVB_ND_TOP_MAX=$tm timeout 300 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters']) for k,v in d.items()})"
done
