# default bench run with wall time and a summary of the secondaries
mkdir -p gpurun_out
t0=$(date +%s)
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $? wall $(( $(date +%s) - t0 )) s"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])
for k, v in d.get("secondary", {}).items():
    print(k, {x: v.get(x) for x in ("iterations", "us_per_iter", "solve_ms", "setup_s", "J", "error")}, v.get("roofline", {}).get("frac"))
PY
