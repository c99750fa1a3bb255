"""Multi-RHS batching timing: m load vectors on the C4
geometry (160x80x80, 8^3 agglomerates) solved one after another with
solve_static vs together with solve_static_batch. Device-timed (CUDA events)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "160,80,80").split(","))
b = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ms_list = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "2,4").split(",")]
nx, ny, nz = dims
d = tv.Domain(nx, ny, nz, 1.0)
clamp = ((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),)
cy, cz = ny // 2, nz // 2
forces = []
for fv in ((0, 0, -1), (0, -1, 0), (0, 0, 1), (0, 1, 0)):
    case = tv.LoadCase("c", dirichlet=clamp, loads=((tv.RegionSelector("box", min=(nx, cy - 1, cz - 1),
                                                                        max=(nx, cy + 1, cz + 1)), fv, "total"),))
    forces.append(torch.from_numpy(tv.assemble_force(d, case)).cuda())
fixed = tv.dirichlet_dofs(d, case)
occ = np.ones(d.n_elems) if os.environ.get("SOLID") else np.where(
    np.random.default_rng(7).random(d.n_elems) < 0.9, 1.0, 1e-3)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, b)
defl.prepare(op)


def timed(fn):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e), out


for m in ms_list:
    F = forces[:m]
    fea.solve_static_batch(op, F, deflation=defl)  # warm (graph capture, workspace)
    for f in F:
        fea.solve_static(op, f, deflation=defl)
    t_seq, rs = timed(lambda: [fea.solve_static(op, f, deflation=defl) for f in F])
    t_bat, rb = timed(lambda: fea.solve_static_batch(op, F, deflation=defl))
    same = all(torch.equal(x.u, y.u) and x.iterations == y.iterations for x, y in zip(rs, rb))
    its = [r.iterations for r in rb]
    print(json.dumps({"dims": dims, "b": b, "m": m, "iterations": its, "sequential_ms": round(t_seq, 2),
                      "batch_ms": round(t_bat, 2), "speedup": round(t_seq / t_bat, 3),
                      "us_per_rhs_iter_seq": round(1e3 * t_seq / sum(its), 1),
                      "us_per_rhs_iter_batch": round(1e3 * t_bat / sum(its), 1), "bitwise_equal": same}), flush=True)
