mkdir -p gpurun_out
python scripts/prof_c2b_nd.py > gpurun_out/prof5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none --cache-control none -k regex:"k_coarse" --csv --log-file gpurun_out/c2b_nd.csv python scripts/prof_c2b_nd.py > gpurun_out/ncu5.log 2>&1
echo "ncu exit $?"
