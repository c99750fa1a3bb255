"""Launch-mode switches change scheduling only, never arithmetic: the deflated
solve must be BITWISE identical with programmatic dependent launch on/off
(TVB_PDL) and with the whole-solve conditional-WHILE graph vs the host loop
over fixed-size graphs (TVB_GRAPH_WHILE). The switches are read once per
process by the library, so each mode runs in its own subprocess."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, hashlib
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea
nx, ny, nz = 24, 12, 12
d = tv.Domain(nx, ny, nz, 1.0)
occ = np.where(np.random.default_rng(5).random(d.n_elems) < 0.8, 1.0, 1e-3)
case = tv.LoadCase("c", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                   loads=((tv.RegionSelector("box", min=(nx, 5, 5), max=(nx, 7, 7)), (0, 0, -1), "total"),))
fixed = tv.dirichlet_dofs(d, case)
f = tv.assemble_force(d, case)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 4)
r = fea.solve_static(op, f, tol=1e-10, deflation=defl)
f2 = np.random.default_rng(6).standard_normal(d.n_dofs)
f2[fixed] = 0.0
rb = fea.solve_static_batch(op, [f, f2], tol=1e-10, deflation=defl)
out = {"it": r.iterations, "u": hashlib.sha256(np.ascontiguousarray(r.u).tobytes()).hexdigest(),
       "bit": [x.iterations for x in rb],
       "bu": [hashlib.sha256(np.ascontiguousarray(x.u).tobytes()).hexdigest() for x in rb],
       "J": float(f @ r.u)}
print(json.dumps(out))
"""


def _run(env_extra):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_launch_modes_bitwise():
    base = _run({})
    assert base["it"] > 10
    assert base["bu"][0] == base["u"] and base["bit"][0] == base["it"]  # batch column 0 == single solve
    # TVB_SOLVE_MASKOUT=1: the iteration's matvecs mask their output again (default: the update kernel keeps
    # r = z = 0 on fixed DOFs and the matvecs skip the mask) -- also bitwise identical
    for extra in ({"TVB_PDL": "0"}, {"TVB_GRAPH_WHILE": "1"}, {"TVB_GRAPH_WHILE": "1", "TVB_WHILE_BODY": "3"},
                  {"TVB_SOLVE_MASKOUT": "1"}):
        other = _run(extra)
        assert other == base, (extra, other, base)
    assert np.isfinite(base["J"])
