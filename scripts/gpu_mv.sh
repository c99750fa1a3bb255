mkdir -p gpurun_out
TVB_MV_VARIANT=1 python scripts/mv_bench.py > gpurun_out/mv_v1.json 2>&1; echo "v1 $?"
TVB_MV_VARIANT=0 python scripts/mv_bench.py > gpurun_out/mv_v0.json 2>&1; echo "v0 $?"
TVB_MV_VARIANT=0 timeout 600 python -m pytest tests -m gpu -x -q -k "matvec or seam or dpcg_golden" > gpurun_out/pytest_v0.log 2>&1; echo "pytest v0 $?"
TVB_MV_VARIANT=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v1.log 2>&1; echo "pytest v1 $?"
cat gpurun_out/mv_v1.json gpurun_out/mv_v0.json; tail -2 gpurun_out/pytest_v0.log gpurun_out/pytest_v1.log
