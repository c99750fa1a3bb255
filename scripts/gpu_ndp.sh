python scripts/nd_prof.py > gpurun_out/ndp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --cache-control none -k regex:"k_coarse" --csv --log-file gpurun_out/nd_launches_warm.csv python scripts/nd_prof.py > gpurun_out/ncu_ndp.log 2>&1
echo "ncu exit $?"; tail -1 gpurun_out/ndp_plain.log
