# A/B: row-coalesced restriction (TVB_RESTRICT=rows) vs CTA-per-block (cta, C4 default) / warp-per-block (warp, C3 default)
mkdir -p gpurun_out
TVB_RESTRICT=rows timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_coarse_nd.py -x -q 2>&1 | tail -1
for rep in 1 2; do for v in rows cta warp; do
  echo "RESTRICT=$v C4 $(TVB_RESTRICT=$v timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_RESTRICT=$v timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done
python scripts/prof_solve.py 160 80 80 8 8 > /dev/null 2>&1
for v in rows cta; do
TVB_RESTRICT=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:k_restrict -s 20 -c 3 --csv python scripts/prof_solve.py 160 80 80 8 8 2>/dev/null | grep -E "duration" | awk -F'","' '{print "'$v'", $NF}'
done
