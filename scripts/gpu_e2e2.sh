for sk in 0 2; do echo "SKIP=$sk"; TVB_MVHOST_SKIP=$sk timeout 120 python scripts/pcie_probe.py 2>&1 | grep "slabs"; done
