#!/bin/bash
# A/B of the matvec work split's per-piece overhead charge (TVB_MV_PIECE_COST, plane-steps)
mkdir -p gpurun_out
for rep in 1 2; do
for c in 0 2 3 4 6; do
  echo "== piece_cost $c (pass $rep)"
  TVB_MV_PIECE_COST=$c python scripts/mv_ablate.py 128 2>&1 | tail -1
  TVB_MV_PIECE_COST=$c python scripts/solve_time.py 160 80 80 8 2>&1 | tail -1
  TVB_MV_PIECE_COST=$c python scripts/solve_time.py 80 40 40 4 2>&1 | tail -1
done
done | tee gpurun_out/piece_cost.log
