# fused top solve (gather + tiles + reduce in one launch): GPU parity + per-iteration time
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -1 gpurun_out/pytest_gpu.log
for rep in 1 2; do
  echo "C4 $(timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done
echo "batch $(timeout 900 python scripts/batch_bench.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-300)"
