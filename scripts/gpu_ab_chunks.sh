# A/B: rows per dataflow item (TVB_FLOW_CHUNKS CTA passes), prefetch off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_coarse_nd.py -x -q 2>&1 | tail -1
for rep in 1 2; do for c in 1 2 4 8; do
  echo "CH=$c C2b nd $(TVB_FLOW_PF=0 TVB_FLOW_CHUNKS=$c timeout 600 python scripts/nd_solve_time.py 2>&1 | tail -1 | cut -c1-70)"
  echo "CH=$c C5 nd $(TVB_FLOW_PF=0 TVB_FLOW_CHUNKS=$c timeout 600 python scripts/nd_solve_time.py 320,160,160 8 2>&1 | tail -1| cut -c1-70)"
done; done
TVB_FLOW_CHUNKS=4 timeout 600 python -m pytest tests/test_coarse_nd.py -x -q 2>&1 | tail -1
