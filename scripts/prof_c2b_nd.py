"""ncu driver: the ND coarse solve of C2(b) (a few solves after setup)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
d = tv.Domain(n, n, n, 1.0)
occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, n, n)), (1, 1, 1)),))
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 4, coarse="nd")
defl.prepare(op)
y = torch.randn(6 * defl.n_blocks, dtype=torch.float64, device="cuda")
x = torch.empty_like(y)
for _ in range(3):
    defl.nd.solve_device(y, x)
torch.cuda.synchronize()
print("ok", defl.nd.H0, defl.nd.n_top)
