for r in cta warp; do
  echo "TVB_RESTRICT=$r"
  TVB_RESTRICT=$r TVB_SOLVE_PROFILE=1 timeout 600 python scripts/prof_solve.py 128 128 128 4 24 2>&1 | grep "solve profile" | tail -1
  TVB_RESTRICT=$r TVB_SOLVE_PROFILE=1 timeout 600 python scripts/prof_solve.py 160 80 80 8 24 2>&1 | grep "solve profile" | tail -1
  TVB_RESTRICT=$r SOLID=1 timeout 600 python scripts/batch_bench.py 160,80,80 8 1 2>&1 | tail -1
  TVB_RESTRICT=$r SOLID=1 timeout 600 python scripts/batch_bench.py 80,40,40 4 1 2>&1 | tail -1
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x 2>&1 | tail -2
