for t in 4608 6200 4608 6200; do echo "C5 TOP_MAX=$t $(TVB_ND_TOP_MAX=$t timeout 900 python scripts/iter_bench.py 320 160 160 8 64 2>&1 | tail -1)"; done
