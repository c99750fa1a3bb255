mkdir -p gpurun_out
for tm in 1200 2400 3600; do
  echo "TOP_MAX=$tm"; TVB_ND_TOP_MAX=$tm timeout 600 python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:v['nd']['us_per_iter'] for k,v in d.items()})"
done
for tm in 2400 4608; do
TVB_ND_TOP_MAX=$tm timeout 900 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | cut -c1-600
done
