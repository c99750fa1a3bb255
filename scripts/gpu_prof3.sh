mkdir -p gpurun_out
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_coarse|k_restrict|k_prolong|k_pcg|k_matvec|k_block_nu|k_finalize" --csv --log-file gpurun_out/solve_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu3.log 2>&1
echo "ncu exit $?"
