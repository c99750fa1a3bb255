"""Fixed (iteration-independent) cost of solve_static: wall and device time against max_iters at a config."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402
from paper_2203_15115_b200.errors import NoConvergence  # noqa: E402

nx, ny, nz, b = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (40, 20, 20, 4)))
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=((tv.RegionSelector("box", min=(nx, ny // 2, nz // 2), max=(nx, ny // 2, nz // 2)),
                           (0, 0, -1), "total"),))
fixed = tv.dirichlet_dofs(d, case)
f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b)
defl.prepare(op)
try:
    fea.solve_static(op, f, tol=1e-8, deflation=defl, max_iters=64)
except NoConvergence:
    pass
for k in (8, 16, 32, 64, 96) + (() if os.environ.get('TVB_EXP_NOMASK') else (100000,)):
    ts = []
    for _ in range(7):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            r = fea.solve_static(op, f, tol=1e-8, deflation=defl, max_iters=k)
            it = r.iterations
        except NoConvergence as e:
            it = e.iterations
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"max_iters {k}: {it} iterations, wall {np.median(ts):.3f} ms")
