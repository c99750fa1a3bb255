# round-1 (second session) profiles: bench launch list, matvec C2 full capture,
# C4 single + batched DPCG warm launch lists, multi-column coarse kernels
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bl.log 2>&1; echo "ncu launches $?"
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 5 -c 1 -o gpurun_out/matvec_c2_full python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full matvec $?"
python scripts/prof_batch.py 8 > gpurun_out/prof_batch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c4_batch2_launches_warm.csv python scripts/prof_batch.py 8 > gpurun_out/ncu_b2.log 2>&1; echo "ncu batch launches $?"
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c4_dpcg_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_it.log 2>&1; echo "ncu c4 launches $?"
ncu --set full --clock-control none --import-source on -k regex:"k_coarse_(fwd|top_rows|bwd)" -s 12 -c 3 -o gpurun_out/c4_coarse2_full python scripts/prof_batch.py 8 > gpurun_out/ncu_cf2.log 2>&1; echo "ncu coarse2 full $?"
