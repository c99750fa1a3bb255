# A/B two prebuilt libraries (ab_old.so / ab_new.so at the repo root): matvec bench + DPCG iteration
mkdir -p gpurun_out
L=paper_2203_15115_b200/libtopovox_b200.so
for rep in 1 2; do for v in old new; do
  cp ab_$v.so $L
  m=$(timeout 600 python bench.py --steps 30 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2))")
  echo "$v matvec C2 GDOF/s,us: $m  C4 $(timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c40-75)  C3 $(timeout 900 python scripts/iter_bench.py 80 40 40 4 300 2>&1 | tail -1 | cut -c40-75)"
done; done
cp ab_new.so $L
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
