timeout 600 python scripts/nd_bench.py C3 C4a C5 2>&1 | grep -v Warning | tail -5
