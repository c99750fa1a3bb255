timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{c:(v[c]['us_per_iter'], v[c]['iters'], v[c]['J']) for c in v} for k,v in d.items()})"
timeout 300 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters']) for k,v in d.items()})"
