"""GPU check of the ND coarse solve schedules on random SPD block stencils."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_coarse_nd import dense_of, random_block_stencil  # noqa: E402

import paper_2203_15115_b200.coarse as C  # noqa: E402

cases = [((4, 3, 3), 27, 4608), ((5, 5, 10), 27, 0), ((9, 8, 7), 8, 60), ((9, 8, 7), 8, 4608), ((12, 10, 9), 27, 600)]
for flow in (0, 1):
    C.FLOW = "1" if flow else "0"
    for grid, leaf, tm in cases:
        Es = random_block_stencil(*grid, seed=1)
        E = dense_of(Es, *grid)
        nd = C.NDCoarseSolver(grid, torch.from_numpy(Es.reshape(-1)).cuda(), leaf_max=leaf, top_max=tm)
        y = np.random.default_rng(3).standard_normal(E.shape[0])
        ndi = nd.nd_index()
        yn = np.empty_like(y)
        yn[ndi] = y
        errs = []
        for rep in range(3):
            x = nd.solve_device(torch.from_numpy(yn).cuda(), torch.zeros(len(y), dtype=torch.float64, device="cuda"))
            torch.cuda.synchronize()
            xs = x.cpu().numpy()[ndi]
            ref = np.linalg.solve(E, y)
            errs.append(float(np.abs(xs - ref).max() / np.abs(ref).max()))
        print("flow", flow, grid, leaf, tm, "H0", nd.H0, "n_top", nd.n_top, "items", nd.n_items, "err", errs, flush=True)
