"""K.u device time at arbitrary grids, with and without Dirichlet masks (public apply path):
`mv_time.py NXxNYxNZ ...` (events, median of 50, L2 warm)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

for spec in sys.argv[1:] or ["100x100x100"]:
    nx, ny, nz = (int(v) for v in spec.split("x"))
    d = tv.Domain(nx, ny, nz, 1.0)
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),), loads=())
    fixed = tv.dirichlet_dofs(d, case)
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
    out = []
    for fx in ((), fixed):
        op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fx)
        y = torch.empty_like(u)
        for _ in range(5):
            op.apply_device(u, y)
        ts = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op.apply_device(u, y)
            b.record()
            torch.cuda.synchronize()
            ts.append(1e3 * a.elapsed_time(b))
        out.append(float(np.median(ts)))
    print(f"{spec} generic={os.environ.get('TVB_MV_GENERIC', '0')}: {out[0]:.1f} us unmasked, {out[1]:.1f} us with Dirichlet masks "
          f"({d.n_dofs / out[0] * 1e-3:.1f} / {d.n_dofs / out[1] * 1e-3:.1f} GDOF/s)")
