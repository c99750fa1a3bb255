"""Sweep matvec launch plans (TVB_MV_PLAN override, read per launch) at the
given sizes inside one process; prints one JSON line per plan."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

sizes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1:] or ["128x128x128", "160x80x80"])]
plans = []
for nt in (256, 384, 512):
    for wx in (12, 16, 20, 24, 28, 32, 40, 48, 64):
        for wy in sorted({max(3, nt // wx - 1), nt // wx}):
            if wx * wy > nt or wy < 3 or 3 * (wx + 1) * (wy + 1) > 4 * nt:
                continue
            plans.append(f"{nt},{wx},{wy}")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ops = []
for dims in sizes:
    d = tv.Domain(*dims, 1.0)
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
    ref = op.apply_device(u).clone()
    ops.append((dims, op, u, ref))
for p in plans:
    os.environ["TVB_MV_PLAN"] = p
    row = {"plan": p}
    for dims, op, u, ref in ops:
        y = torch.empty_like(u)
        op.apply_device(u, y)
        assert torch.equal(y, ref) or float((y - ref).abs().max()) < 1e-12 * float(ref.abs().max()), p
        ts = []
        for i in range(10):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            op.apply_device(u, y)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        row["x".join(map(str, dims))] = round(float(np.median(ts)) * 1e3, 2)
    print(json.dumps(row), flush=True)
