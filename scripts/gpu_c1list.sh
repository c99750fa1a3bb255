#!/bin/bash
# ncu warm launch lists of short C1 / C3 deflated solves (per-kernel times inside the small-problem iteration)
mkdir -p gpurun_out
for cfg in "40 20 20 4 8 c1" "80 40 40 4 8 c3"; do
  set -- $cfg
  python scripts/prof_solve.py $1 $2 $3 $4 $5 > gpurun_out/prof_$6.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv \
      --log-file gpurun_out/$6_dpcg_launches_warm.csv python scripts/prof_solve.py $1 $2 $3 $4 $5 > gpurun_out/ncu_$6.log 2>&1
  echo "ncu $6 $?"
done
