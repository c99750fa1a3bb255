for p in "" 256,23,11 256,22,10 256,24,10 256,25,10 256,21,12 256,32,8 256,28,9 256,20,12 256,19,13 384,24,16 384,32,12 384,28,13; do
  echo "plan=$p $(TVB_MV_PLAN=$p python scripts/mv_bench.py 128x128x128 160x80x80 320x160x160 | python -c 'import json,sys; r=json.load(sys.stdin)["results"]; print({k: round(v["us"],1) for k,v in r.items()})')"
done
