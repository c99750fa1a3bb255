# A/B an environment switch: gpu_ab_env.sh VAR "v1 v2 ..." (DPCG iteration at C4 / C3, ND solve at C5)
mkdir -p gpurun_out
VAR=$1; VALS=$2
for rep in 1 2; do for v in $VALS; do
  echo "$VAR=$v C4 $(env $VAR=$v timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(env $VAR=$v timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done
