mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bl.log 2>&1; echo "ncu launches $?"
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 5 -c 1 -o gpurun_out/matvec_c2_full python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full matvec $?"
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:"k_coarse|k_restrict|k_prolong|k_pcg|k_matvec|k_block_nu|k_finalize" --csv --log-file gpurun_out/c4_dpcg_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_it.log 2>&1; echo "ncu c4 launches $?"
ncu --set full --clock-control none --import-source on -k regex:"k_coarse_(fwd|top_gather|top_rows|bwd)" -c 4 -o gpurun_out/c4_coarse_full python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_cf.log 2>&1; echo "ncu coarse full $?"
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_update" -c 1 -o gpurun_out/c4_update_full python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_uf.log 2>&1; echo "ncu update full $?"
ncu --set full --clock-control none --import-source on -k regex:"k_restrict|k_prolong" -s 330 -c 2 -o gpurun_out/c4_rp_full python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_rpf.log 2>&1; echo "ncu rp full $?"
