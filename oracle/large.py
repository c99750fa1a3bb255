"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Deflation space of the reference for LARGE grids, where the reference's own
``DeflationSpace`` (topovox/fea.py:95-211) cannot run in reasonable time or
memory: it scans every element per block (``np.flatnonzero`` over N_e,
fea.py:172-175), builds each KW column with a full-length ``np.zeros(N_d)``
(fea.py:190-195) and factors a DENSE E (fea.py:197-200; 309 GB at C2(b)).

``FastDeflation`` produces the same W (same blocks, same structural nodes,
same centroid, same masked rigid-body basis, same numpy QR and rank rule --
fea.py:113-183, restated line for line), the same KW columns (the serial
element loop of ``apply_block24_subset``, numba_kernels.py:31-46, evaluated
block-locally with the same element order) and the same symmetrised
E = W^T K W (fea.py:196-198); only the factorisation differs: a sparse
direct LU (SuperLU) of E instead of the dense Cholesky -- an exact solve with
different rounding. It duck-types the reference's DeflationSpace
(``W``, ``KW``, ``prepare(op)``, ``coarse_solve``), so the reference's own
``solve_static`` loop runs over it. Checked against the reference's
DeflationSpace on small grids (tests/test_oracle.py, tests/golden/
make_large_fixtures.py).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse
import scipy.sparse.linalg

OFFS = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                 [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]])


class FastDeflation:
    def __init__(self, nx, ny, nz, h, occ, fixed_dofs, block, k0, design_mask=None, origin=(0.0, 0.0, 0.0),
                 reverse=False):
        """reverse=True (rounding studies only, tests/golden/noise_floor.py):
        accumulate the KW columns over the near elements in descending order."""
        if block < 2:
            raise ValueError("agglomerate side must be >= 2")
        self.dims = (nx, ny, nz)
        self.block = b = int(block)
        n_nodes = (nx + 1) * (ny + 1) * (nz + 1)
        n_dofs = 3 * n_nodes
        occ = np.asarray(occ, dtype=float)
        design = np.ones(nx * ny * nz, bool) if design_mask is None else np.asarray(design_mask, bool)
        fixed = np.zeros(n_dofs, dtype=bool)
        fixed[np.asarray(fixed_dofs, dtype=np.int64)] = True
        solid3 = ((occ == 1.0) & design).reshape(nz, ny, nx)
        occ3 = occ.reshape(nz, ny, nx)
        # structural nodes: adjacent to a solid element (fea.py:119-123)
        st3 = np.zeros((nz + 1, ny + 1, nx + 1), dtype=bool)
        for dx, dy, dz in OFFS:
            st3[dz:dz + nz, dy:dy + ny, dx:dx + nx] |= solid3
        structural = st3.ravel()
        origin = np.asarray(origin, dtype=float)
        mx, my, mz = (nx - 1) // b + 1, (ny - 1) // b + 1, (nz - 1) // b + 1
        k0 = np.ascontiguousarray(k0, dtype=float)
        kw_rows, kw_cols, kw_vals = [], [], []
        w_rows, w_cols, w_vals = [], [], []
        ncols = 0
        self.block_of_col = []
        for bz in range(mz):
            for by in range(my):
                for bx in range(mx):
                    x0, x1 = b * bx, min(b * bx + b, nx)  # element ranges [x0, x1)
                    y0, y1 = b * by, min(b * by + b, ny)
                    z0, z1 = b * bz, min(b * bz + b, nz)
                    if not solid3[z0:z1, y0:y1, x0:x1].any():
                        continue
                    Z, Y, X = np.meshgrid(np.arange(z0, z1 + 1), np.arange(y0, y1 + 1), np.arange(x0, x1 + 1),
                                          indexing="ij")
                    nodes = (X + (nx + 1) * (Y + (ny + 1) * Z)).ravel()  # ascending == np.unique order
                    keepn = structural[nodes]
                    nodes = nodes[keepn]
                    if nodes.size == 0:
                        continue
                    coords = origin + h * np.stack([X.ravel()[keepn], Y.ravel()[keepn], Z.ravel()[keepn]], 1)
                    rel = coords - coords.mean(axis=0)
                    basis = np.zeros((3 * nodes.size, 6))
                    basis[0::3, 0] = 1.0
                    basis[1::3, 1] = 1.0
                    basis[2::3, 2] = 1.0
                    basis[1::3, 3] = -rel[:, 2]
                    basis[2::3, 3] = rel[:, 1]
                    basis[0::3, 4] = rel[:, 2]
                    basis[2::3, 4] = -rel[:, 0]
                    basis[0::3, 5] = -rel[:, 1]
                    basis[1::3, 5] = rel[:, 0]
                    dofs = (3 * nodes[:, None] + np.arange(3)[None, :]).ravel()
                    basis[fixed[dofs]] = 0.0
                    q, r = np.linalg.qr(basis)
                    rd = np.abs(np.diag(r))
                    keep = rd > 1e-10 * max(rd.max(), 1e-300)
                    q = q[:, keep]
                    k = q.shape[1]
                    if k == 0:
                        continue
                    # near elements (fea.py:168-176): the block's element box grown by one, clipped
                    ex0, ex1 = max(x0 - 1, 0), min(x1, nx - 1)
                    ey0, ey1 = max(y0 - 1, 0), min(y1, ny - 1)
                    ez0, ez1 = max(z0 - 1, 0), min(z1, nz - 1)
                    Lx, Ly, Lz = ex1 - ex0 + 2, ey1 - ey0 + 2, ez1 - ez0 + 2
                    # local node box of the near elements; the block's dofs in it
                    xl = X.ravel()[keepn] - ex0
                    yl = Y.ravel()[keepn] - ey0
                    zl = Z.ravel()[keepn] - ez0
                    ln = xl + Lx * (yl + Ly * zl)
                    ldofs = (3 * ln[:, None] + np.arange(3)[None, :]).ravel()
                    wl = np.zeros((3 * Lx * Ly * Lz, k))
                    wl[ldofs] = q
                    # near elements in ascending global id (z, y, x nesting)
                    EZ, EY, EX = np.meshgrid(np.arange(ez0, ez1 + 1), np.arange(ey0, ey1 + 1),
                                             np.arange(ex0, ex1 + 1), indexing="ij")
                    ex, ey, ez = EX.ravel() - ex0, EY.ravel() - ey0, EZ.ravel() - ez0
                    s = occ3[EZ.ravel(), EY.ravel(), EX.ravel()]
                    en = np.stack([(ex + dx) + Lx * ((ey + dy) + Ly * (ez + dz)) for dx, dy, dz in OFFS], 1)
                    ed = (3 * en[:, :, None] + np.arange(3)[None, None, :]).reshape(-1, 24)
                    ue = wl[ed]                                       # (n_near, 24, k)
                    ye = s[:, None, None] * np.einsum("ab,ebk->eak", k0, ue)
                    ye[s == 0.0] = 0.0
                    out = np.zeros_like(wl)
                    if reverse:
                        ed, ye = ed[::-1], ye[::-1]
                    np.add.at(out, ed.ravel(), ye.reshape(-1, k))     # element-ascending accumulation
                    # global dofs of the local node box; Dirichlet rows zeroed (fea.py:73-75)
                    LZ, LY, LX = np.meshgrid(np.arange(ez0, ez1 + 2), np.arange(ey0, ey1 + 2),
                                             np.arange(ex0, ex1 + 2), indexing="ij")
                    gn = (LX + (nx + 1) * (LY + (ny + 1) * LZ)).ravel()
                    gd = (3 * gn[:, None] + np.arange(3)[None, :]).ravel()
                    out[fixed[gd]] = 0.0
                    for j in range(k):
                        nzr = np.flatnonzero(out[:, j])
                        kw_rows.append(gd[nzr])
                        kw_cols.append(np.full(nzr.size, ncols + j, dtype=np.int64))
                        kw_vals.append(out[nzr, j])
                        w_rows.append(dofs)
                        w_cols.append(np.full(dofs.size, ncols + j, dtype=np.int64))
                        w_vals.append(q[:, j])
                        self.block_of_col.append(bx + mx * (by + my * bz))
                    ncols += k
        self.n_vectors = ncols
        self.W = self.KW = None
        if ncols:
            self.W = scipy.sparse.csc_matrix((np.concatenate(w_vals), (np.concatenate(w_rows), np.concatenate(w_cols))),
                                             shape=(n_dofs, ncols))
            del w_rows, w_cols, w_vals
            self.KW = scipy.sparse.csc_matrix(
                (np.concatenate(kw_vals), (np.concatenate(kw_rows), np.concatenate(kw_cols))), shape=(n_dofs, ncols))
        self._lu = None

    def coarse_matrix(self):
        E = (self.W.T @ self.KW).tocsc()
        return (0.5 * (E + E.T)).tocsc()

    def prepare(self, op=None, direct=True) -> None:
        """direct: sparse LU of E. direct=False (C2(b)/C5 fixtures, where
        SuperLU's fill makes the LU impractical): conjugate gradients on E
        (cond(E) ~ 10 for these rigid-mode coarse operators) iterated until
        the residual stops decreasing -- exact to a few units of rounding."""
        if self.W is None or self._lu is not None:
            return
        self.E = self.coarse_matrix()
        if direct:
            self._lu = scipy.sparse.linalg.splu(self.E, permc_spec="MMD_AT_PLUS_A")
        else:
            self._lu = "cg"
            self._dinv = 1.0 / self.E.diagonal()

    def _cg(self, b):
        E, dinv = self.E, self._dinv
        x = np.zeros_like(b)
        r = b.copy()
        z = dinv * r
        p = z.copy()
        rz = r @ z
        best = np.inf
        stall = 0
        # the recursively updated r keeps shrinking long after the true
        # residual has reached the rounding floor (~1e-16 |b|) and would
        # underflow (0/0) after ~640 steps: stop 4 decades below the floor
        floor = 1e-20 * np.linalg.norm(b)
        for _ in range(2000):
            q = E @ p
            a = rz / (p @ q)
            x += a * p
            r -= a * q
            rn = np.linalg.norm(r)
            if rn < best * 0.5:
                best, stall = rn, 0
            else:
                stall += 1
            if stall >= 20 or rn <= floor:
                break
            z = dinv * r
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x

    def coarse_solve(self, rhs):
        rhs = np.asarray(rhs, dtype=float)
        if isinstance(self._lu, str):
            return self._cg(rhs)
        return self._lu.solve(rhs)


def sparse_coarse_solver(E_dense_or_sparse):
    """Sparse direct solve of a (reference-built) coarse matrix E: used to
    replace the reference's per-iteration dense ``cho_solve`` (1.6 s/iter at
    n_c = 12,000) when generating large fixtures."""
    E = scipy.sparse.csc_matrix(E_dense_or_sparse)
    lu = scipy.sparse.linalg.splu(E, permc_spec="MMD_AT_PLUS_A")
    return lambda rhs: lu.solve(np.asarray(rhs, dtype=float))
