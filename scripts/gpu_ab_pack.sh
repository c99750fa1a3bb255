timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_coarse_nd.py -q -x 2>&1 | tail -2
for p in 1 0 1 0; do echo "PACK=$p C4 $(TVB_ND_PACK_TOP=$p timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1)"; done
for p in 1 0; do echo "PACK=$p C3 $(TVB_ND_PACK_TOP=$p timeout 900 python scripts/iter_bench.py 80 40 40 4 400 2>&1 | tail -1)"; done
for p in 1 0; do echo "PACK=$p batch2"; TVB_ND_PACK_TOP=$p SOLID=1 timeout 900 python scripts/batch_bench.py 160,80,80 8 2 2>&1 | tail -1; done
