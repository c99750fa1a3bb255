"""Generate golden vectors from the REAL reference package (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here comes from calling the reference's public API
(topovox.elements / topovox.mesh / topovox.fea) on small seeded inputs; the
.npz files are committed and used by tests/test_oracle.py (oracle pinning)
and tests/test_gpu_parity.py (CUDA parity) on machines without the reference.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from topovox import fea  # noqa: E402
from topovox.elements import Material, hex_stiffness  # noqa: E402
from topovox.mesh import (Domain, LoadCase, RegionSelector, Topology, assemble_force,  # noqa: E402
                          dirichlet_dofs)

OUT = os.path.dirname(os.path.abspath(__file__))


def clamp_case(nx, ny, nz, load_sel, force):
    return LoadCase("c", dirichlet=((RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                    loads=((load_sel, force, "total"),))


def main():
    g = {}
    # --- element stiffness -------------------------------------------------
    g["k0_unit"] = hex_stiffness(Material(E=1.0, nu=0.3), 1.0)
    g["k0_steel"] = hex_stiffness(Material(E=2e11, nu=0.25), 0.5)

    # --- matvec / diag on small random grids ----------------------------------
    rng = np.random.default_rng(123)
    for name, (nx, ny, nz) in {"mv333": (3, 3, 3), "mv543": (5, 4, 3), "mv171": (1, 7, 1)}.items():
        d = Domain(nx, ny, nz, 1.0)
        occ = np.where(rng.random(d.n_elems) < 0.7, 1.0, 1e-3)
        topo = Topology(d, occ)
        case = clamp_case(nx, ny, nz, RegionSelector("box", min=(nx, 0, 0), max=(nx, ny, nz)), (0, 0, -1))
        fixed = dirichlet_dofs(d, case)
        op = fea.StiffnessOperator(d, topo, Material(E=1.0, nu=0.3), fixed)
        u = rng.standard_normal(d.n_dofs)
        g[f"{name}_dims"] = np.array([nx, ny, nz])
        g[f"{name}_occ"] = occ
        g[f"{name}_fixed"] = fixed
        g[f"{name}_u"] = u
        g[f"{name}_Ku_raw"] = op.apply(u, raw=True)
        g[f"{name}_Ku"] = op.apply(u)
        g[f"{name}_diag"] = op.diagonal().copy()
        sub = np.array([0, 1, 1, d.n_elems - 1])
        g[f"{name}_sub"] = sub
        g[f"{name}_Ku_sub"] = op.apply_subset(u, sub)
        s, st, vm = fea.batch_element_state(op, u)
        g[f"{name}_strain"] = s
        g[f"{name}_stress"] = st
        g[f"{name}_vm"] = vm

    # --- small deflated solve, Bernoulli topology ---------------------------------
    nx, ny, nz = 8, 6, 5
    d = Domain(nx, ny, nz, 1.0)
    occ = np.where(np.random.default_rng(7).random(d.n_elems) < 0.7, 1.0, 1e-3)
    case = clamp_case(nx, ny, nz, RegionSelector("box", min=(nx, 0, 0), max=(nx, ny, nz)), (0, -1, -1))
    fixed = dirichlet_dofs(d, case)
    f = assemble_force(d, case)
    op = fea.StiffnessOperator(d, Topology(d, occ), Material(E=1.0, nu=0.3), fixed)
    for b in (2, 3):
        defl = fea.build_deflation(d, Topology(d, occ), fixed, b)
        for tol in (1e-8, 1e-12):
            r = fea.solve_static(op, f, tol=tol, deflation=defl)
            key = f"bern865_b{b}_t{int(-np.log10(tol))}"
            g[key + "_u"] = r.u
            g[key + "_iters"] = np.array(r.iterations)
            g[key + "_res"] = np.array(r.residual)
        g[f"bern865_b{b}_nvec"] = np.array(defl.n_vectors)
    r = fea.solve_static(op, f, tol=1e-12)
    g["bern865_plain_t12_u"] = r.u
    g["bern865_plain_t12_iters"] = np.array(r.iterations)
    g["bern865_occ"] = occ
    g["bern865_fixed"] = fixed
    g["bern865_f"] = f

    # --- C1 cantilever (BASELINE configs[0]) -------------------------------------
    nx, ny, nz = 40, 20, 20
    d = Domain(nx, ny, nz, 1.0)
    case = clamp_case(nx, ny, nz, RegionSelector("box", min=(40, 10, 10), max=(40, 10, 10)), (0, 0, -1))
    fixed = dirichlet_dofs(d, case)
    f = assemble_force(d, case)
    occ = np.ones(d.n_elems)
    op = fea.StiffnessOperator(d, Topology(d, occ), Material(E=1.0, nu=0.3), fixed)
    defl = fea.build_deflation(d, Topology(d, occ), fixed, 4)
    for tol in (1e-8, 1e-12):
        r = fea.solve_static(op, f, tol=tol, deflation=defl)
        key = f"c1_t{int(-np.log10(tol))}"
        g[key + "_J"] = np.array(f @ r.u)
        g[key + "_iters"] = np.array(r.iterations)
        if tol == 1e-12:
            g[key + "_u"] = r.u
            s, st, vm = fea.batch_element_state(op, r.u)
            g["c1_vm_max"] = np.array(vm.max())
            g["c1_vm_pmean8"] = np.array(np.mean(vm ** 8) ** 0.125)
    g["c1_nvec"] = np.array(defl.n_vectors)
    g["c1_nfixed"] = np.array(fixed.size)
    g["c1_fnz"] = np.flatnonzero(f)
    rp = fea.solve_static(op, f, tol=1e-8)
    g["c1_plain_t8_iters"] = np.array(rp.iterations)

    # --- load-case setup of the larger configs (counts / nonzeros only) ----------
    for name, (nx, ny, nz), sel, force in [
        ("c3", (80, 40, 40), RegionSelector("box", min=(80, 20, 20), max=(80, 20, 20)), (0, 0, -1)),
        ("c4a", (160, 80, 80), RegionSelector("box", min=(160, 39, 39), max=(160, 41, 41)), (0, 0, -1)),
        ("c4b", (160, 80, 80), RegionSelector("box", min=(160, 39, 39), max=(160, 41, 41)), (0, -1, 0)),
        ("c5", (320, 160, 160), RegionSelector("box", min=(320, 78, 78), max=(320, 82, 82)), (0, 0, -1)),
    ]:
        d = Domain(nx, ny, nz, 1.0)
        case = clamp_case(nx, ny, nz, sel, force)
        fixed = dirichlet_dofs(d, case)
        f = assemble_force(d, case)
        g[f"{name}_nfixed"] = np.array(fixed.size)
        g[f"{name}_fixed_sum"] = np.array(int(fixed.sum()))
        nzf = np.flatnonzero(f)
        g[f"{name}_f_idx"] = nzf
        g[f"{name}_f_val"] = f[nzf]

    np.savez_compressed(os.path.join(OUT, "reference_golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
