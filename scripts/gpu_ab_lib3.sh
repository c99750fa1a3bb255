# A/B two prebuilt libraries: DPCG iteration at C4 / C3 / C5 (ND solve) alternating
mkdir -p gpurun_out
L=paper_2203_15115_b200/libtopovox_b200.so
for rep in 1 2; do for v in old new; do
  cp ab_$v.so $L
  echo "$v C4 $(timeout 900 python scripts/iter_bench.py 160 80 80 8 300 2>&1 | tail -1 | cut -c40-75)  C3 $(timeout 900 python scripts/iter_bench.py 80 40 40 4 200 2>&1 | tail -1 | cut -c40-75)  C5nd $(timeout 600 python scripts/nd_solve_time.py 320,160,160 8 2>&1 | tail -1 | cut -c40-70)"
done; done
cp ab_new.so $L
timeout 600 python -m pytest tests/test_coarse_nd.py tests/test_gpu_batch.py -x -q 2>&1 | tail -1
