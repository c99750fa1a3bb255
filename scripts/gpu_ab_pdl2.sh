# A/B: PDL with implicit trigger (wait only) on / off, after the update prefetch change
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu parity $?"; tail -1 gpurun_out/pytest_gpu.log
for p in 1 0 1 0; do
  echo "PDL=$p C4 $(TVB_PDL=$p timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c1-80)"
  echo "PDL=$p C3 $(TVB_PDL=$p timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c1-80)"
done
for p in 0; do echo "stage costs PDL=$p"; TVB_PDL=$p timeout 900 python scripts/stage_cost.py 2>&1 | tail -8; done
