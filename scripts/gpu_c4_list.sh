# C4 single-RHS DPCG warm launch list (host-looped graphs) + launch-mode bitwise test
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_launch_modes.py -x -q 2>&1 | tail -1
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c4_dpcg_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_it.log 2>&1; echo "ncu c4 launches $?"
