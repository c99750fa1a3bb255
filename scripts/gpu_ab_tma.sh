# A/B: bulk-copy pipelined persistent top-tile kernel vs one tile per CTA
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_coarse_nd.py tests/test_gpu_batch.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rep in 1 2; do for t in 1 0; do
  echo "TMA=$t C4 $(TVB_TOP_TMA=$t timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_TOP_TMA=$t timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done
for t in 1 0; do echo "TMA=$t batch $(TVB_TOP_TMA=$t timeout 900 python scripts/batch_bench.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c150-300)"; done
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:k_top --csv --log-file gpurun_out/c4_top_tma.csv python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_it.log 2>&1; echo "ncu $?"
