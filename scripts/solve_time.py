"""Device time of a deflated solve at a config (default C4a), tol 1e-8: `solve_time.py nx ny nz b [reps]`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

nx, ny, nz, b = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (160, 80, 80, 8)))
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=((tv.RegionSelector("box", min=(nx, ny // 2, nz // 2), max=(nx, ny // 2, nz // 2)),
                           (0, 0, -1), "total"),))
fixed = tv.dirichlet_dofs(d, case)
f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b)
defl.prepare(op)
r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
ts = []
for _ in range(reps):
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
    e.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(e))
ms = float(np.median(ts))
print(f"{nx}x{ny}x{nz} b={b}: {r.iterations} iterations, {ms:.2f} ms per solve, {1e3 * ms / r.iterations:.1f} us per iteration "
      f"(J = {float(f @ r.u):.10f})")
