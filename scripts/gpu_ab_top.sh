mkdir -p gpurun_out
for m in 1 2 4 8; do
  echo "TVB_ND_TOP_MODE=$m"
  TVB_ND_TOP_MODE=$m SOLID=1 timeout 600 python scripts/batch_bench.py 160,80,80 8 1,2 2>&1 | tail -2
done
echo "TVB_TOP_SMEM=1 mode 2"; TVB_TOP_SMEM=1 TVB_ND_TOP_MODE=2 SOLID=1 timeout 600 python scripts/batch_bench.py 160,80,80 8 1 2>&1 | tail -1
