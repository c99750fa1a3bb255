# C2(b) coarse solve: stage profile + per-kernel DRAM traffic of the ND solve
mkdir -p gpurun_out
TVB_SOLVE_PROFILE=1 timeout 600 python scripts/prof_solve.py 128 128 128 4 24 2>&1 | grep "solve profile" | tail -1
python scripts/prof_c2b_nd.py > gpurun_out/c2b_nd.log 2>&1; tail -1 gpurun_out/c2b_nd.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --cache-control none -k regex:k_coarse --csv --log-file gpurun_out/c2b_nd_kernels.csv python scripts/prof_c2b_nd.py > gpurun_out/ncu_c2b.log 2>&1; echo "ncu $?"
