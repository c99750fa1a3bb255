"""ncu driver: one pass of every per-element field / level-set kernel at the
C4 geometry (160x80x80, full solid), after a warm-up pass."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea, levelset, sensitivity  # noqa: E402

d = tv.Domain(160, 80, 80, 1.0)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), ())
u = torch.from_numpy(np.random.default_rng(3).standard_normal(d.n_dofs)).cuda()
lam = torch.from_numpy(np.random.default_rng(4).standard_normal(d.n_dofs)).cuda()
design = torch.from_numpy(d.design_mask.astype(np.uint8)).cuda()
for _ in range(2):
    _, tj, sums = sensitivity.element_fields_device(op, u, 8)
    sensitivity.adjoint_rhs_device(op, u, 8, sums)
    ts = sensitivity.stress_sensitivity(op, u, lam)
    ls = levelset.combine_device([tj, ts], [2.0, 1.0])
    levelset.extract_device(d, ls, 0.5, 1e-3, design)
torch.cuda.synchronize()
print("ok")
