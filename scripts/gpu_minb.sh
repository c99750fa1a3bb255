timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -1 gpurun_out/pytest_gpu.log
for mb in 4 5 6 8; do
echo "MINB=$mb"; TVB_RP_MINB=$mb timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"
done
