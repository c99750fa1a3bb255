# post-PDL re-sweep of the ND coarse-solve schedule knobs (C4 / C3 iteration time)
mkdir -p gpurun_out
run() { echo "$1 C4 $(env $1 timeout 900 python scripts/iter_bench.py 160 80 80 8 300 2>&1 | tail -1 | cut -c40-75)  C3 $(env $1 timeout 900 python scripts/iter_bench.py 80 40 40 4 200 2>&1 | tail -1 | cut -c40-75)"; }
for rep in 1 2; do
run TVB_X=0
run TVB_ND_WARPS=1184
run TVB_ND_WARPS=4736
run TVB_ND_SLOTS=592
run TVB_ND_SLOTS=2368
run TVB_ND_TOP_MAX=4608
run TVB_ND_TOP_MAX=8000
run TVB_ND_LEAF=64
run TVB_ND_LEAF=216
done
