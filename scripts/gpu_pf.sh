timeout 300 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -1 gpurun_out/pytest_nd.log
for pf in 0 1; do echo "PREFETCH=$pf"; TVB_ND_PREFETCH=$pf timeout 600 python scripts/stage_cost.py 2>&1 | tail -2; done
