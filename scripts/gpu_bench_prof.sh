mkdir -p gpurun_out
python bench.py --steps 100 --warmup 10 > gpurun_out/bench_full.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_full.log | cut -c1-3000
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bl.log 2>&1; echo "ncu launches $?"
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 5 -c 1 -o gpurun_out/matvec_c2_full python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full $?"
