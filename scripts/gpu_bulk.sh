timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu (bulk) $?"; tail -2 gpurun_out/pytest_gpu.log
for b in 0 1; do echo "BULK=$b"; TVB_MV_BULK=$b timeout 300 python scripts/mv_bench.py 2>&1 | tail -1; done
for b in 0 1; do echo "BULK=$b"; TVB_MV_BULK=$b timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"; done
