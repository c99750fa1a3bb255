import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea
d = tv.Domain(160, 80, 80, 1.0)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, 80, 80)), (1, 1, 1)),))
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 8); defl.prepare(op)
nd = defl.nd
print("H0", nd.H0, "n_top", nd.n_top, "fwd_wpr", nd.fwd_wpr, "bwd_wpr", nd.bwd_wpr, "split", nd.split, "top_wpr", nd.top_wpr)
print("nodes", len(nd.s), "s", np.min(nd.s), np.max(nd.s), np.mean(nd.s), "u", np.min(nd.u), np.max(nd.u), np.mean(nd.u))
