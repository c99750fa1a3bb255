"""BASELINE.json configurations used for solution-level DPCG parity at full
size (tests/test_gpu_large_parity.py) and their fixture generator
(tests/golden/make_large_fixtures.py). One definition serves both, so the
GPU test rebuilds exactly the problem the reference solved.

``mesh`` is any module with the reference's setup API (``Domain``,
``LoadCase``, ``RegionSelector``, ``dirichlet_dofs``, ``assemble_force``):
the reference's ``topovox.mesh`` when generating, this repo's
``paper_2203_15115_b200.mesh`` when testing.
"""

from __future__ import annotations

import numpy as np

#: name -> spec. ``tols``: stopping tolerances recorded (tol-stop iterates);
#: ``iters``: fixed iteration counts recorded (iterate x_k).
CASES = {
    # BASELINE configs[2] (C3): 80x40x40, b = 4, point load at the x = 80 face centre
    "c3_solid": dict(dims=(80, 40, 40), block=4, load=((80, 20, 20), (80, 20, 20), (0, 0, -1)), occ="solid",
                     tols=(1e-8, 1e-11), iters=(40,)),
    "c3_bern": dict(dims=(80, 40, 40), block=4, load=((80, 20, 20), (80, 20, 20), (0, 0, -1)), occ="bern0.9",
                    tols=(1e-8, 1e-11), iters=(40,)),
    # BASELINE configs[3] (C4): 160x80x80, b = 8, two load cases over the 3x3 patch of the x = 160 face
    "c4_solid_z": dict(dims=(160, 80, 80), block=8, load=((160, 39, 39), (160, 41, 41), (0, 0, -1)), occ="solid",
                       tols=(1e-8, 1e-11), iters=(40,)),
    "c4_solid_y": dict(dims=(160, 80, 80), block=8, load=((160, 39, 39), (160, 41, 41), (0, -1, 0)), occ="solid",
                       tols=(1e-8, 1e-11), iters=(40,)),
    "c4_bern_z": dict(dims=(160, 80, 80), block=8, load=((160, 39, 39), (160, 41, 41), (0, 0, -1)), occ="bern0.9",
                      tols=(1e-8, 1e-11), iters=(40,)),
    "c4_bern_y": dict(dims=(160, 80, 80), block=8, load=((160, 39, 39), (160, 41, 41), (0, -1, 0)), occ="bern0.9",
                      tols=(1e-8, 1e-11), iters=(40,)),
    # BASELINE configs[4] (C5): 320x160x160, b = 8, 5x5 patch load; fixed-iteration iterates
    "c5_solid": dict(dims=(320, 160, 160), block=8, load=((320, 78, 78), (320, 82, 82), (0, 0, -1)), occ="solid",
                     tols=(), iters=(40,)),
    # BASELINE configs[1] part (b) (C2(b)): 128^3 Bernoulli(0.7), N(0,1) load on free DOFs, b = 4
    "c2b": dict(dims=(128, 128, 128), block=4, load=None, occ="bern0.7", tols=(), iters=(40,)),
}

N_SAMPLE = 4096


def occupancy(spec):
    nx, ny, nz = spec["dims"]
    n = nx * ny * nz
    if spec["occ"] == "solid":
        return np.ones(n)
    if spec["occ"] == "bern0.9":
        return np.where(np.random.default_rng(7).random(n) < 0.9, 1.0, 1e-3)
    if spec["occ"] == "bern0.7":  # BASELINE configs[1]: seed 0
        return np.where(np.random.default_rng(0).random(n) < 0.7, 1.0, 1e-3)
    raise ValueError(spec["occ"])


def problem(mesh, spec):
    """(domain, fixed dofs, force vector, occupancy) of a case."""
    nx, ny, nz = spec["dims"]
    d = mesh.Domain(nx, ny, nz, 1.0)
    clamp = ((mesh.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),)
    if spec["load"] is None:
        case = mesh.LoadCase("c", dirichlet=clamp, loads=())
        fixed = mesh.dirichlet_dofs(d, case)
        f = np.random.default_rng(2).standard_normal(d.n_dofs)  # BASELINE configs[1]: seed 2
        f[fixed] = 0.0
    else:
        lo, hi, force = spec["load"]
        case = mesh.LoadCase("c", dirichlet=clamp, loads=((mesh.RegionSelector("box", min=lo, max=hi), force, "total"),))
        fixed = mesh.dirichlet_dofs(d, case)
        f = mesh.assemble_force(d, case)
    return d, np.asarray(fixed, dtype=np.int64), f, occupancy(spec)


def sample_index(n_dofs):
    return np.sort(np.random.default_rng(1234).choice(n_dofs, N_SAMPLE, replace=False)).astype(np.int64)
