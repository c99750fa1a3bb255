mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -2 gpurun_out/pytest_nd.log
for tm in 1200 2400 4608; do
  echo "TOP_MAX=$tm"; TVB_ND_TOP_MAX=$tm timeout 600 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"
done
TVB_SOLVE_PROFILE=1 python scripts/prof_solve.py 160 80 80 8 24 2>&1 | grep "solve profile" | head -1
timeout 900 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | cut -c1-400
