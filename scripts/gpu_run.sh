#!/bin/bash
# Round-2 GPU driver: build check, then the requested stages (gpurun -- 'bash scripts/gpu_run.sh STAGE...').
#   tests      pytest -m gpu (whole suite)          -> gpurun_out/pytest_gpu.log
#   tests:EXPR pytest -m gpu -k EXPR                -> gpurun_out/pytest_k.log
#   smoke      __graft_entry__.smoke()
#   bench      default bench.py line                -> gpurun_out/bench.json
#   launches   ncu launch list of the bench         -> gpurun_out/bench_launches.csv
#   mvfull     ncu --set full of one C2 k_matvec    -> gpurun_out/matvec_c2_full.ncu-rep
#   c4list     ncu warm launch list of a C4 solve   -> gpurun_out/c4_dpcg_launches_warm.csv
#   fields     ncu --set full of the C4 field kernels -> gpurun_out/fields_c4_full.ncu-rep
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
for st in "$@"; do
  case "$st" in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu $?"; grep -E "^\[|passed|failed" gpurun_out/pytest_gpu.log | tail -30;;
    tests:*) timeout 1500 python -m pytest tests -m gpu -q -s -k "${st#tests:}" > gpurun_out/pytest_k.log 2>&1; echo "pytest -k $?"; grep -E "^\[|passed|failed|Error|assert" gpurun_out/pytest_k.log | tail -40;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log;;
    bench) timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench $?"; tail -3 gpurun_out/bench.err
      python - <<'PY'
import json
d = json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value', 'value_median', 'ms_per_step', 'clocks', 'gpu_launches')})
print('roofline', d['roofline']['frac'], d['roofline']['own_bound'], 'e2e', d['e2e']['value'])
for k, v in d.get('secondary', {}).items():
    print(k, json.dumps(v)[:600])
print('cpu', d.get('cpu_baseline'))
PY
      ;;
    launches) python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_bl.log 2>&1; echo "ncu launches $?";;
    mvfull) ncu --set full --clock-control none --import-source on -k regex:k_matvec -s 5 -c 1 -f -o gpurun_out/matvec_c2_full python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full matvec $?";;
    c4list) python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/prof_plain.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/c4_dpcg_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 8 > gpurun_out/ncu_it.log 2>&1; echo "ncu c4 launches $?";;
    fields) python scripts/prof_fields.py > gpurun_out/prof_fields.log 2>&1 && \
      ncu --set full --clock-control none --import-source on -k regex:"k_element|k_adjoint|k_stress_sens|k_maxabs|k_combine|k_radix|k_eq_count|k_scan_counts|k_apply_threshold" -c 24 -f -o gpurun_out/fields_c4_full python scripts/prof_fields.py > gpurun_out/ncu_fields.log 2>&1; echo "ncu fields $?";;
    *) echo "unknown stage $st";;
  esac
done
