# A/B: L2 prefetch of each dataflow item's factor rows (TVB_FLOW_PF)
mkdir -p gpurun_out
for rep in 1 2; do for p in 1 0; do
  echo "PF=$p C2b nd $(TVB_FLOW_PF=$p timeout 600 python scripts/nd_solve_time.py 2>&1 | tail -1)"
  echo "PF=$p C5 nd $(TVB_FLOW_PF=$p timeout 600 python scripts/nd_solve_time.py 320,160,160 8 2>&1 | tail -1)"
done; done
timeout 600 python -m pytest tests/test_coarse_nd.py -x -q 2>&1 | tail -1
