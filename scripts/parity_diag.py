"""Where does the device iterate depart from the reference's? (c3_bern
fixture, x after the reference's tol-1e-8 iteration count): coarse-solve
accuracy of the ND factor against a host solve of the symmetrised E, and the
iterate with the ND factor / the dense inverse, each projection."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import large_cases as LC  # noqa: E402
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import _lib, fea, mesh  # noqa: E402
from paper_2203_15115_b200._lib import ptr, stream_ptr  # noqa: E402
from paper_2203_15115_b200.errors import NoConvergence  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3_bern"
fx = np.load(os.path.join(ROOT, "tests", "golden", "large_dpcg.npz"))
spec = LC.CASES[name]
d, fixed, f, occ = LC.problem(mesh, spec)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
fd = torch.from_numpy(f).cuda()
idx = fx[f"{name}_idx"]
it = int(fx[f"{name}_tol1e-08_it"])
ref = fx[f"{name}_tol1e-08_u"]
for coarse in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("nd", "dense")):
    defl = fea.build_deflation(d, op.topology, fixed, spec["block"], coarse=coarse)
    defl.prepare(op)
    if coarse == "nd":
        nc = 6 * defl.n_blocks
        E = torch.empty(nc * nc, dtype=torch.float64, device="cuda")
        _lib.lib().tvb_coarse_dense(d.nx, d.ny, d.nz, spec["block"], ptr(defl.Es), ptr(E), stream_ptr())
        E = E.view(nc, nc).cpu().numpy()
        Es = 0.5 * (E + E.T)
        y = np.random.default_rng(0).standard_normal(nc)
        xs = np.linalg.solve(Es, y)
        xg = defl.coarse_solve(y)
        print(f"{name}: ND coarse solve vs numpy solve "
              f"{np.linalg.norm(xg - xs) / np.linalg.norm(xs):.2e}", flush=True)
        del E, Es
    for proj in ("stabilized", "reference"):
        try:
            fea.solve_static(op, fd, tol=1e-14, max_iters=it, deflation=defl, projection=proj)
        except NoConvergence as exc:
            x = exc.u[idx].cpu().numpy()
            print(f"{name} coarse={coarse} projection={proj}: x_{it} vs reference "
                  f"{np.linalg.norm(x - ref) / np.linalg.norm(ref):.2e}", flush=True)
