# A/B: update kernel variant (v2 contiguous, v3 prefetch, v4 grid-strided prefetch) x PDL (wait-only)
mkdir -p gpurun_out
for rep in 1 2; do
for v in 2 3 4; do for p in 0 1; do
  echo "V=$v PDL=$p C4 $(TVB_UPD_V=$v TVB_PDL=$p timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_UPD_V=$v TVB_PDL=$p timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done; done
echo "V=4 CTAS=1184 C4 $(TVB_UPD_V=4 TVB_UPD_CTAS=1184 timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)"
echo "V=4 CTAS=296 C4 $(TVB_UPD_V=4 TVB_UPD_CTAS=296 timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)"
