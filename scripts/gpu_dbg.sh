mkdir -p gpurun_out
for d in 0 1 2 4 3 7; do for p in 256,24,10 384,28,13 256,20,12; do echo "debug=$d plan=$p $(TVB_MV_DEBUG=$d TVB_MV_PLAN=$p python scripts/mv_bench.py 160x80x80 128x128x128 | python -c 'import json,sys; r=json.load(sys.stdin)["results"]; print({k: round(v["us"],1) for k,v in r.items()})')"; done; done
