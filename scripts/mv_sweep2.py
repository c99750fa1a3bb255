"""Fine matvec plan sweep for NT = 256 (TVB_MV_PLAN override, read per launch):
all wx in [18, 40] with wx * wy in [200, 256] at the given sizes; prints one
JSON line per plan (median us of 20 launches, L2 flushed) and the default plan."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

sizes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1:] or ["128x128x128", "160x80x80"])]
plans = [None] + [f"256,{wx},{wy}" for wx in range(18, 41) for wy in range(3, 15) if 200 <= wx * wy <= 256]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ops = []
for dims in sizes:
    d = tv.Domain(*dims, 1.0)
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
    ops.append((dims, op, u))
for plan in plans:
    if plan is None:
        os.environ.pop("TVB_MV_PLAN", None)
    else:
        os.environ["TVB_MV_PLAN"] = plan
    row = {"plan": plan or "default"}
    for dims, op, u in ops:
        op.apply_device(u)
        ts = []
        for _ in range(20):
            flush.zero_()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op.apply_device(u)
            e.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e) * 1e3)
        row["x".join(map(str, dims))] = round(sorted(ts)[10], 2)
    print(json.dumps(row), flush=True)
