timeout 300 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -1 gpurun_out/pytest_nd.log
CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/nd_flow_check.py 2>&1 | tail -10 | cut -c1-150
TVB_ND_RPW=4 timeout 120 python scripts/nd_flow_check.py 2>&1 | tail -3 | cut -c1-150
timeout 600 python scripts/nd_bench.py C3 C4a C5 2>&1 | grep -v Warning | tail -3
TVB_ND_RPW=1 timeout 600 python scripts/nd_bench.py C4a 2>&1 | grep -v Warning | tail -1
TVB_ND_RPW=4 timeout 600 python scripts/nd_bench.py C4a 2>&1 | grep -v Warning | tail -1
