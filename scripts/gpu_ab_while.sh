# A/B: whole-solve conditional-WHILE graph (TVB_GRAPH_WHILE = body iterations; 1 -> 4) vs host-looped graphs (0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_coarse_nd.py -x -q 2>&1 | tail -2
for rep in 1 2; do for v in 0 1 2 8; do
  echo "WHILE=$v C4 $(TVB_GRAPH_WHILE=$v timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(TVB_GRAPH_WHILE=$v timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)  C1 $(TVB_GRAPH_WHILE=$v timeout 900 python scripts/iter_bench.py 40 20 20 4 120 2>&1 | tail -1 | cut -c40-75)"
done; done
for v in 0 1; do echo "WHILE=$v batch $(TVB_GRAPH_WHILE=$v timeout 900 python scripts/batch_bench.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c150-300)"; done
