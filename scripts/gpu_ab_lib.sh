#!/bin/bash
# A/B of library builds: for each scratch_variants/NAME.so, install it as the package library and
# time K.u at C2 (scripts/mv_ablate.py, warm) and deflated solves at C4 / C3 (scripts/solve_time.py).
mkdir -p gpurun_out
LIB=paper_2203_15115_b200/libtopovox_b200.so
cp $LIB /tmp/keep.so
for rep in 1 2; do
for v in "$@"; do
  cp scratch_variants/$v.so $LIB
  echo "== $v (pass $rep)"
  python scripts/mv_ablate.py 128 2>&1 | tail -1
  python scripts/solve_time.py 160 80 80 8 2>&1 | tail -1
  python scripts/solve_time.py 80 40 40 4 2>&1 | tail -1
done
done | tee gpurun_out/ab_lib.log
cp /tmp/keep.so $LIB
