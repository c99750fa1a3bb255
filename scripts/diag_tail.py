import os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import large_cases as LC
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea, mesh
from paper_2203_15115_b200.errors import NoConvergence
fx = np.load("/root/repo/tests/golden/large_dpcg.npz")
for name in ("c4_bern_y", "c4_bern_z"):
    spec = LC.CASES[name]
    d, fixed, f, occ = LC.problem(mesh, spec)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, spec["block"])
    fd = torch.from_numpy(f).cuda()
    idx = fx[f"{name}_idx"]
    for proj in ("stabilized", "reference"):
        r = fea.solve_static(op, fd, tol=1e-11, deflation=defl, projection=proj)
        print(name, proj, "tol 1e-11: it", r.iterations, "res", r.residual, "ref it", int(fx[f"{name}_tol1e-11_it"]), "ref res", float(fx[f"{name}_tol1e-11_res"]))
        for k in (1069, 1070, 1071, 1072, 1073):
            try:
                fea.solve_static(op, fd, tol=1e-14, max_iters=k, deflation=defl, projection=proj)
            except NoConvergence as e:
                print("   k", k, "res", e.residual)
