"""ncu driver: a few ND coarse solves at C4a (warm), for per-kernel launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
import paper_2203_15115_b200.coarse as C  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

nx, ny, nz, b = (160, 80, 80, 8) if len(sys.argv) < 2 else tuple(int(v) for v in sys.argv[1:5])
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),), loads=())
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b, coarse="nd")
defl.prepare(op)
nd = defl.nd
y = torch.randn(6 * nd.nb, dtype=torch.float64, device="cuda")
x = torch.empty_like(y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("solves")
for _ in range(5):
    nd.solve_device(y, x)
torch.cuda.synchronize()
print("ok", nd.H0, nd.n_top, nd.n_items)
