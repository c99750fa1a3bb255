"""Device time of one ND coarse solve (x = E^-1 y) at a grid / block size:
`nd_solve_time.py n b [bernoulli]` (default C2(b): 128^3, b = 4, Bernoulli(0.7))."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,128,128").split(","))
b = int(sys.argv[2]) if len(sys.argv) > 2 else 4
d = tv.Domain(*dims, 1.0)
occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, dims[1], dims[2])), (1, 1, 1)),))
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b, coarse="nd")
defl.prepare(op)
y = torch.randn(6 * defl.n_blocks, dtype=torch.float64, device="cuda")
x = torch.empty_like(y)
for _ in range(3):
    defl.nd.solve_device(y, x)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    defl.nd.solve_device(y, x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(json.dumps({"dims": dims, "b": b, "us": sorted(ts)[len(ts) // 2], "factor_GB": defl.nd.bytes / 1e9,
                  "flow": bool(defl.nd.flow), "x_sum": float(x.sum())}))
