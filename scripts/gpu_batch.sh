mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/pytest_batch.log 2>&1; echo "batch tests exit $?"; tail -15 gpurun_out/pytest_batch.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/batch_bench.py 160,80,80 8 2,4 > gpurun_out/batch_bench.log 2>&1; echo "batch bench $?"; cat gpurun_out/batch_bench.log | tail -4
SOLID=1 timeout 600 python scripts/batch_bench.py 80,40,40 4 2 >> gpurun_out/batch_bench.log 2>&1; tail -1 gpurun_out/batch_bench.log
