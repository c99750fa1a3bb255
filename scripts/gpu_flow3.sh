CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/nd_flow_check.py 2>&1 | tail -15
