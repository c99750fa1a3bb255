for sk in 0 1 2 4 3 5 6; do echo "SKIP=$sk"; TVB_MVHOST_SKIP=$sk timeout 120 python scripts/pcie_probe.py 2>&1 | grep "slabs 1:\|slabs 4:\|slabs 6:\|slabs 8:\|H2D"; done
