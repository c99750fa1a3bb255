"""Per-iteration DPCG time (device, CUDA events around whole solves) at given configs."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

configs = {"C1": (40, 20, 20, 4), "C3": (80, 40, 40, 4), "C4a": (160, 80, 80, 8)}
which = sys.argv[1:] or list(configs)
out = {}
for name in which:
    nx, ny, nz, b = configs[name]
    d = tv.Domain(nx, ny, nz, 1.0)
    lo = (nx, ny // 2 - (1 if name == "C4a" else 0), nz // 2 - (1 if name == "C4a" else 0))
    hi = (nx, ny // 2 + (1 if name == "C4a" else 0), nz // 2 + (1 if name == "C4a" else 0))
    case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                       loads=((tv.RegionSelector("box", min=lo, max=hi), (0, 0, -1), "total"),))
    fixed = tv.dirichlet_dofs(d, case)
    f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
    op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
    row = {}
    for coarse in ("dense", "nd") if 6 * ((nx - 1) // b + 1) * ((ny - 1) // b + 1) * ((nz - 1) // b + 1) <= 24000 else ("nd",):
        t0 = time.perf_counter()
        defl = fea.build_deflation(d, op.topology, fixed, b, coarse=coarse)
        defl.prepare(op)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
        e.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(e)
        row[coarse] = {"iters": r.iterations, "solve_ms": round(ms, 3), "us_per_iter": round(1e3 * ms / r.iterations, 1),
                       "setup_s": round(setup, 3), "J": float(f @ r.u)}
    out[name] = row
print(json.dumps(out))
