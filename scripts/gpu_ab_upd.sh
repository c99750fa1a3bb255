for g in 296 444 592 0 592 444 296 0; do echo "UPD_CTAS=$g C4 $(TVB_UPD_CTAS=$g timeout 900 python scripts/iter_bench.py 160 80 80 8 400 2>&1 | tail -1 | cut -c1-80)"; done
