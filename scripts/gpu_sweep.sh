mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest $?"; tail -3 gpurun_out/pytest_gpu.log
python scripts/mv_sweep.py 128x128x128 160x80x80 80x40x40 320x160x160 > gpurun_out/mv_sweep.jsonl 2> gpurun_out/mv_sweep.err; echo "sweep $?"
python scripts/mv_bench.py > gpurun_out/mv_default.json 2>&1; cat gpurun_out/mv_default.json
