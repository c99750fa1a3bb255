mkdir -p gpurun_out
python scripts/prof_matvec.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 3 -c 1 -o gpurun_out/matvec_c2 python scripts/prof_matvec.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches exit $?"
