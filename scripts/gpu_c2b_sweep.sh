run() { echo "$*: $(env "$@" TVB_SOLVE_PROFILE=1 timeout 600 python scripts/prof_solve.py 128 128 128 4 16 2>&1 | grep 'solve profile' | tail -1 | grep -o 'coarse_solve=[0-9.]*')"; }
run TVB_ND_WARPS=2368
run TVB_ND_WARPS=1184
run TVB_ND_WARPS=4736
run TVB_ND_WARPS=9472
run TVB_ND_WPR=1
run TVB_ND_WPR=1 TVB_ND_RPW=2
run TVB_ND_WPR=2
run TVB_ND_LEAF=125
run TVB_ND_LEAF=27
