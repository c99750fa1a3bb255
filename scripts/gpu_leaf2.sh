for leaf in 27 64 125; do echo "LEAF=$leaf"; TVB_ND_LEAF=$leaf timeout 400 python scripts/big_solves.py C5 C2b 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:(v['us_per_iter'], v['iters'], v['factor_GB'], v['prepare_s']) for k,v in d.items()})"; done
for tm in 2400 4608 7000; do echo "LEAF=125 TOP=$tm"; TVB_ND_LEAF=125 TVB_ND_TOP_MAX=$tm timeout 300 python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"; done
