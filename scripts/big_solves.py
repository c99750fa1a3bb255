"""C2(b) and C5 deflated solves (infeasible for the reference's dense coarse factor)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

which = sys.argv[1:] or ["C2b", "C5"]
out = {}
for name in which:
    t_all = time.perf_counter()
    if name == "C2b":
        n = 128
        d = tv.Domain(n, n, n, 1.0)
        occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
        case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, n, n)), (1, 1, 1)),))
        fixed = tv.dirichlet_dofs(d, case)
        f = np.random.default_rng(2).standard_normal(d.n_dofs)
        f[fixed] = 0.0
        b = 4
    else:
        nx, ny, nz = 320, 160, 160
        d = tv.Domain(nx, ny, nz, 1.0)
        occ = np.ones(d.n_elems)
        case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                           loads=((tv.RegionSelector("box", min=(nx, 78, 78), max=(nx, 82, 82)), (0, 0, -1), "total"),))
        fixed = tv.dirichlet_dofs(d, case)
        f = tv.assemble_force(d, case)
        b = 8
    fd = torch.from_numpy(f).cuda()
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    t0 = time.perf_counter()
    defl = fea.build_deflation(d, op.topology, fixed, b)
    torch.cuda.synchronize()
    t_basis = time.perf_counter() - t0
    t0 = time.perf_counter()
    defl.prepare(op)
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t0
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = fea.solve_static(op, fd, tol=1e-8, deflation=defl)
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    out[name] = {"n_dofs": d.n_dofs, "n_coarse": defl.n_vectors, "basis_s": round(t_basis, 3), "prepare_s": round(t_prep, 3),
                 "iters": r.iterations, "solve_ms": round(ms, 2), "us_per_iter": round(1e3 * ms / max(1, r.iterations), 1),
                 "factor_GB": round(defl.nd.bytes / 1e9, 3) if defl.nd is not None else None,
                 "nd_levels": defl.nd.H0 if defl.nd is not None else None, "n_top": defl.nd.n_top if defl.nd is not None else None,
                 "J": float(fd @ r.u), "max_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 2),
                 "total_s": round(time.perf_counter() - t_all, 2)}
    print(json.dumps({name: out[name]}), flush=True)
    del op, defl, r
    torch.cuda.empty_cache()
