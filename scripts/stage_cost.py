"""In-graph cost of each DPCG stage at C4a: per-iteration time with the stage
left out of the CUDA graph (TVB_SOLVE_SKIP), fixed 200 iterations. Timing only."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, "%s")
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea
from paper_2203_15115_b200.errors import NoConvergence
nx, ny, nz, b = %s
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=((tv.RegionSelector("box", min=(nx, ny//2-1, nz//2-1), max=(nx, ny//2+1, nz//2+1)), (0, 0, -1), "total"),))
fixed = tv.dirichlet_dofs(d, case)
f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b)
defl.prepare(op)
best = 1e9
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    try:
        fea.solve_static(op, f, tol=1e-30 if rep >= 0 else 1e-8, deflation=defl, max_iters=200, check_every=8)
    except NoConvergence:
        pass
    torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
print(best / 200 * 1e6)
'''
dims = sys.argv[1] if len(sys.argv) > 1 else "(160, 80, 80, 8)"
out = {}
for name, mask in [("full", 0), ("-Ap", 1), ("-update", 2), ("-Az", 4), ("-restrict", 8), ("-coarse", 16),
                   ("-prolong", 32)]:
    env = dict(os.environ, TVB_SOLVE_SKIP=str(mask))
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, dims)], env=env, capture_output=True, text=True)
    try:
        out[name] = round(float(r.stdout.strip().splitlines()[-1]), 1)
    except Exception:
        out[name] = r.stderr[-300:]
print(json.dumps(out))
if isinstance(out.get("full"), float):
    print(json.dumps({k: round(out["full"] - v, 1) for k, v in out.items() if isinstance(v, float) and k != "full"}))
