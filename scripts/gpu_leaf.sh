for leaf in 27 64 125 250; do echo "LEAF=$leaf"; TVB_ND_LEAF=$leaf timeout 600 python scripts/stage_cost.py 2>&1 | tail -1; done
for leaf in 27 64 125; do echo "LEAF=$leaf"; TVB_ND_LEAF=$leaf timeout 300 python scripts/solve_bench.py C3 C4a 2>&1 | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print({k:(v['nd']['us_per_iter'], v['nd']['iters']) for k,v in d.items()})"; done
