#!/bin/bash
# A/B of library builds on the nested-dissection coarse solve alone (C2(b) and C5) and the C5 DPCG iteration
mkdir -p gpurun_out
LIB=paper_2203_15115_b200/libtopovox_b200.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in "$@"; do
  cp scratch_variants/$v.so $LIB
  echo "== $v (pass $rep)"
  python scripts/nd_solve_time.py 128,128,128 4 2>&1 | tail -1
  python scripts/nd_solve_time.py 320,160,160 8 2>&1 | tail -1
done
done | tee gpurun_out/ab_nd.log
cp /tmp/keep.so $LIB
