"""Device time of the element-map kernels at C4 through the device API (events, median of 20):
`TVB_ELEM_KERNEL=tile|march|flat python scripts/fields_time.py`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea, sensitivity  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (160, 80, 80)
d = tv.Domain(*dims, 1.0)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), ())
u = torch.from_numpy(np.random.default_rng(3).standard_normal(d.n_dofs)).cuda()
lam = torch.from_numpy(np.random.default_rng(4).standard_normal(d.n_dofs)).cuda()
_, _, sums = sensitivity.element_fields_device(op, u, 8)


def timed(fn, reps=20):
    ts = []
    for _ in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(1e3 * a.elapsed_time(b))
    return float(np.median(ts[3:]))


print(f"{os.environ.get('TVB_ELEM_KERNEL', 'tile')} {dims}: "
      f"element state + T_J + p-norm {timed(lambda: sensitivity.element_fields_device(op, u, 8)):.1f} us, "
      f"adjoint rhs {timed(lambda: sensitivity.adjoint_rhs_device(op, u, 8, sums)):.1f} us, "
      f"T_sigma {timed(lambda: sensitivity.stress_sensitivity(op, u, lam)):.1f} us")
