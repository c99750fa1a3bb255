"""Matvec micro-benchmark: device time per K.u (L2 flushed) at C1..C5 sizes."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import _lib, fea  # noqa: E402

sizes = [(40, 20, 20), (80, 40, 40), (128, 128, 128), (160, 80, 80), (320, 160, 160)]
if len(sys.argv) > 1:
    sizes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
out = {}
for dims in sizes:
    d = tv.Domain(*dims, 1.0)
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).cuda()
    y = torch.empty_like(u)
    for _ in range(3):
        op.apply_device(u, y)
    ts = []
    for i in range(20):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        op.apply_device(u, y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.median(ts)) * 1e-3
    plan = (ctypes.c_int * 7)()
    _lib.lib().tvb_matvec_plan(*dims, ctypes.cast(plan, ctypes.c_void_p))
    nd, ne = d.n_dofs, d.n_elems
    out["x".join(map(str, dims))] = {"us": t * 1e6, "GDOF/s": nd / t / 1e9, "GB/s": 8 * (2 * nd + ne) / t / 1e9,
                                     "dense_TF": 1152 * ne / t / 1e12, "plan": list(plan)}
print(json.dumps({"variant": os.environ.get("TVB_MV_VARIANT", "1"), "results": out}))
