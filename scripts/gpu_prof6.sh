mkdir -p gpurun_out
TVB_SOLVE_PROFILE=1 python scripts/prof_solve.py 160 80 80 8 24 2>&1 | grep "solve profile" | head -3
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof6_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --cache-control none -k regex:"k_coarse|k_restrict|k_prolong|k_pcg|k_matvec|k_block_nu|k_finalize" --csv --log-file gpurun_out/r01_c4_dpcg_launches_nd2.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu6.log 2>&1
echo "ncu exit $?"
