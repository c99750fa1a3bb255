# A/B of the top-solve fusion bits (1: gather in tiles, 2: row reduction by the last tile CTA)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_coarse_nd.py -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do for f in 0 1 2 3; do
  echo "FUSE=$f C4 $(TVB_TOP_FUSE=$f timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_TOP_FUSE=$f timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done
