"""Where DeflationSpace.prepare spends its time (GPU): coarse assembly vs the
nested-dissection symbolic / numeric phases."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (320, 160, 160, 8)))
nx, ny, nz, b = dims
d = tv.Domain(nx, ny, nz, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),), loads=())
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    defl = fea.build_deflation(d, op.topology, fixed, b)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pr = cProfile.Profile()
    pr.enable()
    defl.prepare(op)
    torch.cuda.synchronize()
    pr.disable()
    t2 = time.perf_counter()
    print(f"rep {rep}: build {t1 - t0:.3f} s, prepare {t2 - t1:.3f} s", flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
