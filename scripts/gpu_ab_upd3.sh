# A/B: update kernel variant x CTA count (PDL on)
mkdir -p gpurun_out
for rep in 1 2; do
for v in 2 4; do for g in 296 592; do
  echo "V=$v CTAS=$g C4 $(TVB_UPD_V=$v TVB_UPD_CTAS=$g timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_UPD_V=$v TVB_UPD_CTAS=$g timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done; done
for v in 2 4; do for g in 296 592; do
  echo "V=$v CTAS=$g C5 $(TVB_UPD_V=$v TVB_UPD_CTAS=$g timeout 900 python scripts/iter_bench.py 320 160 160 8 100 2>&1 | tail -1 | cut -c40-75)"
done; done
