"""Golden vectors for the geometric-stiffness seam function, from the REAL
reference (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_geo.py

Calls topovox.elements.geometric_tensor (elements.py:141-153) and the numba
backend's apply_nodal_block8 (backends/numba_kernels.py:61-76) -- the kernel
seam entry point the buckling analysis would call -- on small seeded inputs;
writes reference_golden_geo.npz (committed)."""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from topovox import backends, fea  # noqa: E402
from topovox.elements import Material, geometric_tensor, voigt_to_tensor  # noqa: E402
from topovox.mesh import Domain, Topology  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    g = {"A_h1": geometric_tensor(1.0), "A_h05": geometric_tensor(0.5)}
    rng = np.random.default_rng(321)
    for name, (nx, ny, nz, h) in {"g543": (5, 4, 3, 1.0), "g217": (2, 1, 7, 0.5)}.items():
        d = Domain(nx, ny, nz, h)
        occ = np.where(rng.random(d.n_elems) < 0.7, 1.0, 1e-3)
        op = fea.StiffnessOperator(d, Topology(d, occ), Material(E=1.0, nu=0.3), ())
        # stress field of a random displacement (occupancy-scaled, as fea reports it)
        w = rng.standard_normal(d.n_dofs)
        _, stresses, _ = fea.batch_element_state(op, w)
        A = geometric_tensor(h)
        blocks = np.einsum("epq,pqij->eij", np.stack([voigt_to_tensor(s) for s in stresses]), A)
        u = rng.standard_normal(d.n_dofs)
        out = np.zeros(d.n_dofs)
        backends.apply_nodal_block8(u, out, d.elem_dofs, np.ascontiguousarray(blocks), op._color_perm,
                                    op._color_ptr)
        rb = rng.standard_normal((d.n_elems, 8, 8))
        out_r = np.zeros(d.n_dofs)
        backends.apply_nodal_block8(u, out_r, d.elem_dofs, rb, op._color_perm, op._color_ptr)
        g.update({f"{name}_dims": np.array([nx, ny, nz]), f"{name}_h": np.array(h), f"{name}_occ": occ,
                  f"{name}_w": w, f"{name}_stress": stresses, f"{name}_u": u, f"{name}_KGu": out,
                  f"{name}_blocks": rb, f"{name}_Bu": out_r})
    np.savez_compressed(os.path.join(OUT, "reference_golden_geo.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
