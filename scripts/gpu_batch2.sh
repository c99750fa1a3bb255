mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_optimize.py -x -q > gpurun_out/pytest_batch.log 2>&1; echo "batch+opt tests exit $?"; tail -5 gpurun_out/pytest_batch.log
timeout 600 python scripts/batch_bench.py 160,80,80 8 2,4 > gpurun_out/batch_bench.log 2>&1; echo "fork"; cat gpurun_out/batch_bench.log | tail -2
TVB_BATCH_FORK=0 timeout 600 python scripts/batch_bench.py 160,80,80 8 2 2>&1 | tail -1
SOLID=1 timeout 600 python scripts/batch_bench.py 80,40,40 4 2 2>&1 | tail -1
timeout 900 python scripts/opt_run.py C4 3 > gpurun_out/opt_c4.log 2>&1; echo "opt C4 $?"; tail -4 gpurun_out/opt_c4.log
