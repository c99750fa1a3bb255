# session-3 verification: full GPU suite, smoke, default bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','clocks','gpu_launches')})
print(d['roofline']['frac'], d['roofline'].get('north_star',{}).get('frac'), d['e2e'])
for k,v in d.get('secondary',{}).items(): print(k, {x: v.get(x) for x in ('iterations','us_per_iter','solve_ms')}, v.get('roofline',{}).get('frac'))
print(d.get('cpu_baseline'))
"
