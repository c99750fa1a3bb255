timeout 300 python scripts/solve_bench.py C1 C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:{c:(v[c]['us_per_iter'], v[c]['iters']) for c in v} for k,v in d.items()})"
timeout 300 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters']) for k,v in d.items()})"
python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none -k regex:"k_coarse|k_restrict|k_prolong|k_pcg|k_matvec|k_block_nu|k_finalize" --csv --log-file gpurun_out/c4_launches_warm.csv python scripts/prof_solve.py 160 80 80 8 4 > gpurun_out/ncu_it.log 2>&1
echo "ncu exit $?"
