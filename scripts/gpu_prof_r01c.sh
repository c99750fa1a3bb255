# round-1 (third session) evidence: GPU suite, default bench, bench launch list,
# matvec C2 full capture, C4 DPCG warm launch list (single RHS)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','clocks','gpu_launches')}, d['roofline']['frac'], d['e2e']['value'])
for k,v in d.get('secondary',{}).items(): print(k, {x: v.get(x) for x in ('iterations','us_per_iter','solve_ms')}, v.get('roofline',{}).get('frac'))
"
python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bl.log 2>&1; echo "ncu launches $?"
ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 5 -c 1 -o gpurun_out/matvec_c2_full_r01c python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full matvec $?"
python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c4_dpcg_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_it.log 2>&1; echo "ncu c4 launches $?"
