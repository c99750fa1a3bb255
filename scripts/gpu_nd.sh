mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest default $?"; tail -1 gpurun_out/pytest_nd.log
TVB_ND_SPLIT_FRONT=0 timeout 900 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd_split.log 2>&1; echo "pytest split-all $?"; tail -1 gpurun_out/pytest_nd_split.log
python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | cut -c1-300
python scripts/solve_bench.py C3 C4a 2>&1 | tail -1
