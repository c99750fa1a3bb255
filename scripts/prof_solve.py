"""ncu driver: a short deflated solve at a config (default C4a) for per-kernel launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402
from paper_2203_15115_b200.errors import NoConvergence  # noqa: E402

nx, ny, nz, b = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (160, 80, 80, 8)))
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 8
coarse = sys.argv[6] if len(sys.argv) > 6 else "auto"
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=((tv.RegionSelector("box", min=(nx, ny // 2 - 1, nz // 2 - 1), max=(nx, ny // 2 + 1, nz // 2 + 1)),
                           (0, 0, -1), "total"),))
fixed = tv.dirichlet_dofs(d, case)
f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b, coarse=coarse)
defl.prepare(op)
for _ in range(2):
    try:
        fea.solve_static(op, f, tol=1e-8, deflation=defl, max_iters=iters, check_every=iters)
    except NoConvergence:
        pass
torch.cuda.synchronize()
print("ok")
