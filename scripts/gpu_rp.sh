timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{c:(v[c]['us_per_iter'], v[c]['iters']) for c in v} for k,v in d.items()})"
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:"k_restrict|k_prolong" --csv --log-file gpurun_out/c4_rp.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_rp.log 2>&1
echo "ncu exit $?"
