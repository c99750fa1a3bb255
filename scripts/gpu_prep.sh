timeout 300 python -m pytest tests -m gpu -x -q -k "dpcg or coarse" > gpurun_out/pytest_nd.log 2>&1; echo "pytest nd $?"; tail -1 gpurun_out/pytest_nd.log
timeout 600 python scripts/prep_prof.py 2>&1 | head -22
timeout 600 python scripts/prep_prof.py 160 80 80 8 2>&1 | head -3
