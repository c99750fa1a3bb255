# A/B: iterations per conditional-WHILE body (TVB_WHILE_BODY), C1 / C3 / C4 full solves at tol 1e-8
mkdir -p gpurun_out
for rep in 1 2; do for v in 1 2 4 8; do
  echo "BODY=$v $(TVB_WHILE_BODY=$v timeout 900 python scripts/solve_bench.py 2>&1 | tail -1 | cut -c1-300)"
done; done
