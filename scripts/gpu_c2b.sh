mkdir -p gpurun_out
for flow in "" 0; do
  echo "TVB_ND_FLOW=$flow"
  TVB_ND_FLOW=$flow TVB_SOLVE_PROFILE=1 timeout 600 python scripts/prof_solve.py 128 128 128 4 24 2>&1 | grep "solve profile" | tail -1
done
python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea
d = tv.Domain(128,128,128,1.0)
case = tv.LoadCase('c', dirichlet=((tv.RegionSelector('box', min=(0,0,0), max=(0,128,128)), (1,1,1)),), loads=())
fixed = tv.dirichlet_dofs(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 4); defl.prepare(op)
nd = defl.nd
print('n_c', 6*defl.n_blocks, 'factor GB', nd.bytes/1e9, 'n_top', nd.n_top, 'H0', nd.H0, 'items', nd.n_items, 'leaf', nd.leaf_max)
" 2>&1 | tail -1
