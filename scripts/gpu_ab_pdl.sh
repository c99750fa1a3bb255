# A/B: programmatic dependent launch on / off (per-iteration DPCG device time, matvec)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -1 gpurun_out/pytest_gpu.log
for p in 1 0 1 0; do
  echo "PDL=$p C4 $(TVB_PDL=$p timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c1-100)"
  echo "PDL=$p C3 $(TVB_PDL=$p timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c1-100)"
  echo "PDL=$p C1 $(TVB_PDL=$p timeout 900 python scripts/iter_bench.py 40 20 20 4 120 2>&1 | tail -1 | cut -c1-100)"
done
for p in 1 0; do echo "PDL=$p batch $(TVB_PDL=$p timeout 900 python scripts/batch_bench.py 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-300)"; done
