mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import torch; import ctypes; p=torch.cuda.get_device_properties(0); print(p)"
for v in "" "TVB_NO_L2_PERSIST=1" "TVB_ND_PERSISTENT=0" "TVB_ND_PERSISTENT=0 TVB_NO_L2_PERSIST=1"; do echo "== $v"; env $v python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:{c:v['us_per_iter'] for c,v in r.items()} for k,r in d.items()})"; done
