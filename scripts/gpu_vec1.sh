mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{c:(v[c]['us_per_iter'], v[c]['iters']) for c in v} for k,v in d.items()})"
TVB_SOLVE_PROFILE=1 python scripts/prof_solve.py 160 80 80 8 24 2>&1 | grep "solve profile" | head -1
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_coarse|k_restrict|k_prolong|k_pcg|k_matvec|k_block_nu|k_finalize" --csv --log-file gpurun_out/c4_launches_vec1.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_vec1.log 2>&1
echo "ncu exit $?"
