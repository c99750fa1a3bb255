for sk in 2 34; do echo "SKIP=$sk"; TVB_MVHOST_SKIP=$sk timeout 120 python scripts/pcie_probe.py 2>&1 | grep "slabs 2\|slabs 4\|slabs 8\|torch pipeline K=4"; done
