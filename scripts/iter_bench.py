"""Device time per DPCG iteration (CUDA-graph path) over a fixed number of
iterations: `iter_bench.py nx ny nz b iters [bernoulli]` (NoConvergence at the
cap is expected and ignored)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402
from paper_2203_15115_b200.errors import NoConvergence  # noqa: E402

nx, ny, nz, b, iters = (int(v) for v in sys.argv[1:6])
bern = len(sys.argv) > 6
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=())
fixed = tv.dirichlet_dofs(d, case)
occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3) if bern else np.ones(d.n_elems)
f = np.random.default_rng(2).standard_normal(d.n_dofs)
f[fixed] = 0.0
fd = torch.from_numpy(f).cuda()
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b)
defl.prepare(op)


def run():
    try:
        fea.solve_static(op, fd, tol=1e-14, deflation=defl, max_iters=iters, check_every=8)
    except NoConvergence:
        pass


run()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
run()
e.record()
torch.cuda.synchronize()
nd = defl.nd
print(json.dumps({"dims": [nx, ny, nz], "b": b, "us_per_iter": 1e3 * a.elapsed_time(e) / iters,
                  "n_top": nd.n_top if nd is not None else None,
                  "factor_GB": nd.bytes / 1e9 if nd is not None else None}))
