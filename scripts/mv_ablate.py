"""Matvec ablation (tuning only): time K.u at C2 with stages switched off via
TVB_MV_DEBUG (library built with -DTVB_MATVEC_DEBUG): 1 no barrier, 2 no
staging loads, 4 no stores. Results are wrong by design; only the time matters."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
d = tv.Domain(n, n, n, 1.0)
occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
y = torch.empty_like(u)
for _ in range(20):
    op.apply_device(u, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(200):
    op.apply_device(u, y)
b.record()
torch.cuda.synchronize()
print(f"debug={os.environ.get('TVB_MV_DEBUG', '0')} generic={os.environ.get('TVB_MV_GENERIC', '0')}: "
      f"{1e3 * a.elapsed_time(b) / 200:.1f} us per K.u (L2 warm)")
