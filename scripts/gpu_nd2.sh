mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -3 gpurun_out/pytest_gpu.log
for tm in 4608 0 9000; do
  echo "TOP_MAX=$tm"; TVB_ND_TOP_MAX=$tm timeout 600 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1
done
timeout 900 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | cut -c1-400
