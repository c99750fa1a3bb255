"""Small driver for ncu: a few K.u at the C2 (128^3) and C4 (160x80x80) sizes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

for dims in [(128, 128, 128), (160, 80, 80)]:
    d = tv.Domain(*dims, 1.0)
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
    y = torch.empty_like(u)
    for _ in range(4):
        op.apply_device(u, y)
    torch.cuda.synchronize()
print("ok")
