# A/B two prebuilt libraries: matvec bench (C2) x3 alternating + ncu bank conflicts of the new one
mkdir -p gpurun_out
L=paper_2203_15115_b200/libtopovox_b200.so
for rep in 1 2 3; do for v in old new; do
  cp ab_$v.so $L
  m=$(timeout 600 python bench.py --steps 30 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), round(d['ms_per_step']*1e3,2))")
  echo "$v matvec C2 GDOF/s,us: $m"
done; done
for v in old new; do cp ab_$v.so $L
ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum --clock-control none -k regex:k_matvec -s 5 -c 1 --csv python bench.py --steps 5 --warmup 3 --no-secondary --no-cpu-baseline 2>/dev/null | grep -E "bank|duration|inst_exec" | awk -F'","' '{print "'$v'", $(NF-2), $NF}'
done
cp ab_new.so $L
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
