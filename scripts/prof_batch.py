"""ncu driver: a short 2-RHS batched deflated solve on the C4 geometry (both
BASELINE configs[3] load cases) for per-kernel launch lists / captures of the
multi-column coarse kernels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402
from paper_2203_15115_b200.errors import NoConvergence  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 8
d = tv.Domain(160, 80, 80, 1.0)
fs = []
for fv in ((0, 0, -1), (0, -1, 0)):
    case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, 80, 80)), (1, 1, 1)),),
                       loads=((tv.RegionSelector("box", min=(160, 39, 39), max=(160, 41, 41)), fv, "total"),))
    fs.append(torch.from_numpy(tv.assemble_force(d, case)).cuda())
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 8)
defl.prepare(op)
for _ in range(2):
    try:
        fea.solve_static_batch(op, fs, tol=1e-8, deflation=defl, max_iters=iters, check_every=iters)
    except NoConvergence:
        pass
torch.cuda.synchronize()
