"""Two independent C4a deflated solves: sequential vs concurrent (two host threads,
separate operators / deflation spaces, so no shared scratch)."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

nx, ny, nz, b = 160, 80, 80, 8
d = tv.Domain(nx, ny, nz, 1.0)
cases = []
for force in ((0, 0, -1), (0, -1, 0)):
    case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                       loads=((tv.RegionSelector("box", min=(nx, 39, 39), max=(nx, 41, 41)), force, "total"),))
    fixed = tv.dirichlet_dofs(d, case)
    f = torch.from_numpy(tv.assemble_force(d, case)).cuda()
    op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, b)
    defl.prepare(op)
    cases.append((op, f, defl))
for op, f, defl in cases:  # warm (graph capture paths, allocations)
    fea.solve_static(op, f, tol=1e-8, deflation=defl)
torch.cuda.synchronize()
res = {}


def run(i):
    op, f, defl = cases[i]
    with torch.cuda.stream(torch.cuda.Stream()):
        res[i] = fea.solve_static(op, f, tol=1e-8, deflation=defl)


def seq():
    for i in range(2):
        run(i)
    torch.cuda.synchronize()


def con():
    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()


for rep in range(3):
    t0 = time.perf_counter()
    seq()
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    con()
    t_con = time.perf_counter() - t0
    print(f"rep {rep}: iterations {[res[i].iterations for i in range(2)]}; sequential {t_seq*1e3:.1f} ms, "
          f"concurrent {t_con*1e3:.1f} ms, speedup {t_seq/t_con:.2f}", flush=True)
