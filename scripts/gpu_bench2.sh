for i in 1 2; do
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(round(d['value'],2), round(d['ms_per_step']*1e3,1), d['clocks'], round(d['roofline']['north_star']['frac'],3), round(d['e2e']['value'],2))
for k,v in d.get('secondary',{}).items(): print(k, round(v.get('us_per_iter'),1), v.get('iterations'), round(v['roofline']['frac'],3), round(v['roofline']['survey_def']['frac'],3))
"
done
timeout 300 python scripts/mv_bench.py 128x128x128 160x80x80 2>&1 | tail -1
