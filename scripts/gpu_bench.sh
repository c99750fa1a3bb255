timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','clocks')})
print(d['roofline']['frac'], d['roofline']['north_star']['frac'], d['e2e'])
for k,v in d.get('secondary',{}).items(): print(k, {x: v.get(x) for x in ('iterations','us_per_iter','solve_ms')}, v.get('roofline',{}).get('frac'), v.get('roofline',{}).get('stages_us'))
print(d.get('cpu_baseline'))
"
