"""Generate full-size DPCG fixtures (BASELINE configs C2(b), C3, C4, C5) from
the REAL reference in the build container (it is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_large_fixtures.py [case ...]

What runs is the reference's own code except where it cannot finish:
  * setup: ``topovox.mesh`` (Domain, LoadCase, dirichlet_dofs, assemble_force);
  * operator: ``topovox.fea.StiffnessOperator`` (numba ``apply_block24``) and
    its Jacobi diagonal;
  * deflation at C3/C4: ``topovox.fea.DeflationSpace`` (W, KW, E built by the
    reference's ``_build_basis`` / ``prepare``). Its per-iteration dense
    ``cho_solve`` (1.6 s at n_c = 12,000) is replaced by a sparse direct LU of
    the SAME E -- an exact solve with different rounding;
  * deflation at C2(b)/C5: ``oracle.large.FastDeflation`` (the reference's
    basis/KW/E restated block-locally; the dense E would need 309 GB at
    C2(b)). It is checked below to be bitwise equal to the reference's
    DeflationSpace (W, KW, E) on small grids and at C3. Its coarse solve there
    is CG on E run to the rounding floor (SuperLU's fill on these 3-D
    stencils is impractical; cond(E) ~ 10);
  * loop: ``oracle.topovox_oracle.solve_static`` -- the reference's
    ``solve_static`` (fea.py:218-299) restated step for step, checked below to
    be bitwise equal to it -- with an observer that snapshots the iterate when
    the residual first drops below each recorded tolerance and at fixed
    iteration counts (the reference's loop returns no iterate on
    NoConvergence, and one run serves every tolerance).

Recorded per case (tests/golden/large_dpcg.npz): iteration count, relative
residual, compliance f.u, ||u|| and u at 4096 seeded sample DOFs for every
tolerance stop and fixed iteration count in tests/large_cases.py, plus
checksums of the problem (fixed-DOF count, sum f, n_vectors).
"""

from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
from topovox import fea  # noqa: E402
from topovox import mesh as refmesh  # noqa: E402
from topovox.elements import Material  # noqa: E402

import large_cases as LC  # noqa: E402
from oracle import topovox_oracle as O  # noqa: E402
from oracle.large import FastDeflation, sparse_coarse_solver  # noqa: E402

OUT = os.path.join(HERE, "large_dpcg.npz")


class RefOp:
    """The reference operator seen through the attribute names of the
    oracle's loop (free mask, apply, diagonal)."""

    def __init__(self, op):
        self.op = op
        self.free = op.free_mask
        self.n_dofs = op.n_dofs
        self.apply = op.apply
        self.diagonal = op.diagonal


def self_check():
    """oracle loop == reference loop (bitwise) and FastDeflation == the
    reference's DeflationSpace (bitwise W, KW, E) on C1-sized problems."""
    for dims, b, lo, hi, p in (((40, 20, 20), 4, (40, 10, 10), (40, 10, 10), 1.0),
                                ((13, 7, 5), 4, (13, 0, 0), (13, 7, 5), 0.7)):
        nx, ny, nz = dims
        d = refmesh.Domain(nx, ny, nz, 1.0)
        occ = np.where(np.random.default_rng(3).random(d.n_elems) < p, 1.0, 1e-3)
        case = refmesh.LoadCase("c", dirichlet=((refmesh.RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)),
                                                 (1, 1, 1)),),
                                loads=((refmesh.RegionSelector("box", min=lo, max=hi), (0, 0, -1), "total"),))
        fixed = refmesh.dirichlet_dofs(d, case)
        f = refmesh.assemble_force(d, case)
        op = fea.StiffnessOperator(d, refmesh.Topology(d, occ), Material(E=1.0, nu=0.3), fixed)
        R = fea.DeflationSpace(d, refmesh.Topology(d, occ), fixed, b)
        R.prepare(op)
        F = FastDeflation(nx, ny, nz, 1.0, occ, fixed, b, op.k0)
        assert (R.W != F.W).nnz == 0 and (R.KW != F.KW).nnz == 0, "FastDeflation W/KW differ"
        E = np.asarray((R.W.T @ R.KW).todense())
        assert np.array_equal(0.5 * (E + E.T), F.coarse_matrix().toarray()), "FastDeflation E differs"
        ref = fea.solve_static(op, f, tol=1e-8, deflation=R)
        R.prepare = lambda *_a: None  # prepared for op above
        u, it, res = O.solve_static(RefOp(op), f, tol=1e-8, deflation=R)
        assert it == ref.iterations and np.array_equal(u, ref.u) and res == ref.residual, "oracle loop differs"
    print("self-check: oracle loop and FastDeflation bitwise equal to the reference", flush=True)


def run_case(name, spec, cache):
    t0 = time.time()
    d, fixed, f, occ = LC.problem(refmesh, spec)
    nx, ny, nz = spec["dims"]
    b = spec["block"]
    op = fea.StiffnessOperator(d, refmesh.Topology(d, occ), Material(E=1.0, nu=0.3), fixed)
    key = (spec["dims"], spec["occ"], b)
    if key in cache:
        defl = cache[key]
    elif d.n_elems <= 1_100_000:  # C3 / C4: the reference's own deflation space
        defl = fea.DeflationSpace(d, refmesh.Topology(d, occ), fixed, b)
        defl.prepare(op)
        E = np.asarray((defl.W.T @ defl.KW).todense())
        E = 0.5 * (E + E.T)
        if d.n_elems <= 130_000:  # C3: FastDeflation must agree bitwise at full size too
            F = FastDeflation(nx, ny, nz, 1.0, occ, fixed, b, op.k0)
            assert (defl.W != F.W).nnz == 0 and (defl.KW != F.KW).nnz == 0
            assert np.array_equal(E, F.coarse_matrix().toarray())
            print(f"  {name}: FastDeflation bitwise equal to the reference at full size", flush=True)
        defl.coarse_solve = sparse_coarse_solver(E)
        defl._prepared_for = op
        del E
        cache.clear()
        cache[key] = defl
    else:  # C2(b) / C5: iterative coarse solve to rounding level (see FastDeflation.prepare)
        defl = FastDeflation(nx, ny, nz, 1.0, occ, fixed, b, op.k0)
        defl.prepare(op, direct=False)
        cache.clear()
        cache[key] = defl
    defl.prepare = lambda *_a: None  # already prepared for this operator / topology
    setup = time.time() - t0
    idx = LC.sample_index(d.n_dofs)
    tols = sorted(spec["tols"], reverse=True)
    iters = sorted(spec["iters"])
    snaps = {}
    last_k = iters[-1] if iters else 0

    def record(tag, it, x, res):
        snaps[tag] = dict(it=it, res=res, J=float(f @ x), norm=float(np.linalg.norm(x)), u=x[idx].copy())

    def observer(it, x, res):
        for t in tols:
            if f"tol{t:g}" not in snaps and res <= t:
                record(f"tol{t:g}", it, x, res)
        if it in iters:
            record(f"k{it}", it, x, res)
        return not tols and it >= last_k

    out = {}
    t1 = time.time()
    try:
        u, it, res = O.solve_static(RefOp(op), f, tol=tols[-1] if tols else 1e-14,
                                    max_iters=None if tols else last_k, deflation=defl, observer=observer)
        if tols:
            record(f"tol{tols[-1]:g}", it, u, res)
        status = "ok"
    except O.OracleNoConvergence as exc:
        status = f"no convergence at {tols[-1] if tols else 0:g}: residual {exc.residual:.3e}"
    solve = time.time() - t1
    out[f"{name}_nvec"] = np.int64(defl.n_vectors)
    out[f"{name}_nfixed"] = np.int64(len(fixed))
    out[f"{name}_fsum"] = np.float64(np.abs(f).sum())
    out[f"{name}_idx"] = idx
    out[f"{name}_status"] = np.array(status)
    for tag, s in snaps.items():
        for k, v in s.items():
            out[f"{name}_{tag}_{k}"] = np.asarray(v)
    print(f"{name}: n_vec {defl.n_vectors} setup {setup:.0f}s solve {solve:.0f}s status {status}; "
          + ", ".join(f"{t}: it {s['it']} J {s['J']:.12g}" for t, s in snaps.items()), flush=True)
    return out


def main(argv):
    names = argv or list(LC.CASES)
    self_check()
    data = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    cache = {}
    for name in names:
        for k in [k for k in data if k.startswith(name + "_")]:
            del data[k]
        data.update(run_case(name, LC.CASES[name], cache))
        np.savez_compressed(OUT, **data)


if __name__ == "__main__":
    main(sys.argv[1:])
