mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -1 gpurun_out/pytest_nd.log
for w in 2368 4736 9472; do
  echo "WARPS=$w"; TVB_ND_WARPS=$w timeout 600 python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"
  TVB_ND_WARPS=$w timeout 900 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters']) for k,v in d.items()})"
done
