"""Coarse-solve-only timing: the ND solve of a real deflation space (C3/C4a
full-solid cantilever), 50 solves captured in one CUDA graph, warm."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
import paper_2203_15115_b200.coarse as C  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

configs = {"C3": (80, 40, 40, 4), "C4a": (160, 80, 80, 8), "C5": (320, 160, 160, 8)}
variants = [(f, tm) for f in (0, 1) for tm in (600, 2400, 4608)]
out = {}
for name in sys.argv[1:] or ["C3", "C4a"]:
    nx, ny, nz, b = configs[name]
    d = tv.Domain(nx, ny, nz, 1.0)
    case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                       loads=())
    fixed = tv.dirichlet_dofs(d, case)
    op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, b, coarse="nd")
    defl.prepare(op)
    Es = defl.Es
    row = {}
    for flow, tm in variants:
        C.FLOW = "1" if flow else "0"
        nd = C.NDCoarseSolver(defl.grid, Es, top_max=tm)
        y = torch.randn(6 * nd.nb, dtype=torch.float64, device="cuda")
        x = torch.empty_like(y)
        for _ in range(3):
            nd.solve_device(y, x)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(50):
                    nd.solve_device(y, x)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        row[f"flow{flow}_tm{tm}"] = round(a.elapsed_time(e) * 1e3 / 200, 1)
        del nd, g
    out[name] = row
    print(json.dumps({name: row}), flush=True)
