"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU restatement of the reference hot path, function by function:

FEA (reference code exists; restated from it):
  hex_stiffness            topovox/elements.py:117-132
  centroid_b / elasticity  topovox/elements.py:72-79, 135-138
  elem_dofs                topovox/mesh.py:92-104
  element_coloring         topovox/backends/__init__.py:59-66
  Operator.apply/subset/diagonal   topovox/fea.py:49-85 (kernels in oracle/kernels.c)
  Deflation (W, KW, E, Cholesky)   topovox/fea.py:95-215
  solve_static (deflated Jacobi PCG) topovox/fea.py:218-299
  batch_element_state      topovox/fea.py:302-309

SPEC-only stages (no reference code; restated from the SPEC text):
  compliance_sensitivity   SPEC.md:283-291 (Eq 3.2)
  pnorm_stress
  stress_adjoint_rhs       SPEC.md:301-309 (chain rule)
  stress_sensitivity
  normalize_field/combine
  extract
  AL scalars               SPEC.md:466-501 (Eqs 3.9, 3.11, 3.12)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import scipy.linalg
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OracleError(Exception):
    pass


class OracleNoConvergence(OracleError):
    def __init__(self, msg, residual, iterations):
        super().__init__(msg)
        self.residual = residual
        self.iterations = iterations


def build_lib(force: bool = False) -> str:
    so = os.path.join(HERE, "_build", "liboracle.so")
    src = os.path.join(HERE, "kernels.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-B", "-C", HERE], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        so = os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(so):
            build_lib()
        L = ctypes.CDLL(so)
        P = ctypes.c_void_p
        L.oracle_apply_block24.argtypes = [P, P, P, P, P, P, P, ctypes.c_int]
        L.oracle_apply_block24_subset.argtypes = [P, P, P, ctypes.c_int64, P, P, P]
        L.oracle_diag_block24.argtypes = [P, P, P, ctypes.c_int64, P]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# element constants
# ---------------------------------------------------------------------------
OFFS = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                 [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]])
Q_VM = np.array([[1.0, -0.5, -0.5, 0, 0, 0], [-0.5, 1.0, -0.5, 0, 0, 0], [-0.5, -0.5, 1.0, 0, 0, 0],
                 [0, 0, 0, 3.0, 0, 0], [0, 0, 0, 0, 3.0, 0], [0, 0, 0, 0, 0, 3.0]])


def elasticity(E, nu):
    c = E / ((1.0 + nu) * (1.0 - 2.0 * nu))
    D = np.zeros((6, 6))
    D[:3, :3] = c * nu
    for i in range(3):
        D[i, i] = c * (1.0 - nu)
        D[i + 3, i + 3] = c * (1.0 - 2.0 * nu) / 2.0
    return D


def _bmat(dn):
    B = np.zeros((6, 24))
    for i in range(8):
        bx, by, bz = dn[i]
        B[0, 3 * i] = bx
        B[1, 3 * i + 1] = by
        B[2, 3 * i + 2] = bz
        B[3, 3 * i], B[3, 3 * i + 1] = by, bx
        B[4, 3 * i + 1], B[4, 3 * i + 2] = bz, by
        B[5, 3 * i], B[5, 3 * i + 2] = bz, bx
    return B


def _dshape(xi, eta, zeta):
    s = 2.0 * OFFS - 1.0
    g = np.empty((8, 3))
    g[:, 0] = s[:, 0] * (1 + s[:, 1] * eta) * (1 + s[:, 2] * zeta) / 8.0
    g[:, 1] = s[:, 1] * (1 + s[:, 0] * xi) * (1 + s[:, 2] * zeta) / 8.0
    g[:, 2] = s[:, 2] * (1 + s[:, 0] * xi) * (1 + s[:, 1] * eta) / 8.0
    return g


def hex_stiffness(E, nu, h):
    D = elasticity(E, nu)
    k = np.zeros((24, 24))
    a = 1.0 / np.sqrt(3.0)
    for gp in a * (2.0 * OFFS - 1.0):
        B = _bmat(_dshape(*gp) * (2.0 / h))
        k += B.T @ D @ B * (h / 2.0) ** 3
    return 0.5 * (k + k.T)


def centroid_b(h):
    return _bmat(_dshape(0.0, 0.0, 0.0) * (2.0 / h))


def von_mises(s):
    return np.sqrt(np.maximum(np.einsum("...i,ij,...j->...", s, Q_VM, s), 0.0))


# ---------------------------------------------------------------------------
# mesh numbering
# ---------------------------------------------------------------------------
def elem_dofs(nx, ny, nz):
    e = np.arange(nx * ny * nz)
    ix, iy, iz = e % nx, (e // nx) % ny, e // (nx * ny)
    nxy = (nx + 1) * (ny + 1)
    out = np.empty((e.size, 24), dtype=np.int32)
    for i, (dx, dy, dz) in enumerate(OFFS):
        n = (ix + dx) + (nx + 1) * (iy + dy) + nxy * (iz + dz)
        out[:, 3 * i] = 3 * n
        out[:, 3 * i + 1] = 3 * n + 1
        out[:, 3 * i + 2] = 3 * n + 2
    return out


def coloring(nx, ny, nz):
    e = np.arange(nx * ny * nz)
    ix, iy, iz = e % nx, (e // nx) % ny, e // (nx * ny)
    color = (ix & 1) + 2 * (iy & 1) + 4 * (iz & 1)
    perm = np.argsort(color, kind="stable").astype(np.int64)
    ptr = np.concatenate([[0], np.cumsum(np.bincount(color, minlength=8))]).astype(np.int64)
    return perm, ptr


def node_coords(nx, ny, nz, h):
    n = np.arange((nx + 1) * (ny + 1) * (nz + 1))
    return h * np.stack([n % (nx + 1), (n // (nx + 1)) % (ny + 1), n // ((nx + 1) * (ny + 1))], axis=1).astype(float)


# ---------------------------------------------------------------------------
# operator (topovox/fea.py:30-85)
# ---------------------------------------------------------------------------
class Operator:
    def __init__(self, nx, ny, nz, h, occ, E=1.0, nu=0.3, dirichlet=(), design_mask=None):
        self.nx, self.ny, self.nz, self.h = nx, ny, nz, h
        self.E, self.nu = E, nu
        self.occ = np.ascontiguousarray(occ, dtype=float)
        self.k0 = np.ascontiguousarray(hex_stiffness(E, nu, h))
        self.n_dofs = 3 * (nx + 1) * (ny + 1) * (nz + 1)
        self.dirichlet = np.unique(np.asarray(dirichlet, dtype=np.int64))
        self.free = np.ones(self.n_dofs, dtype=bool)
        self.free[self.dirichlet] = False
        self.edofs = np.ascontiguousarray(elem_dofs(nx, ny, nz))
        self.perm, self.ptr = coloring(nx, ny, nz)
        self.design_mask = np.ones(nx * ny * nz, dtype=bool) if design_mask is None else np.asarray(design_mask, bool)
        self._diag = None

    def apply(self, u, raw=False):
        u = np.asarray(u, dtype=float)
        if not raw and self.dirichlet.size:
            u = u.copy()
            u[self.dirichlet] = 0.0
        u = np.ascontiguousarray(u)
        out = np.zeros(self.n_dofs)
        lib().oracle_apply_block24(_p(u), _p(out), _p(self.edofs), _p(self.occ), _p(self.k0), _p(self.perm),
                                   _p(self.ptr), 8)
        if not raw and self.dirichlet.size:
            out[self.dirichlet] = 0.0
        return out

    def apply_subset(self, u, elems):
        u = np.ascontiguousarray(u, dtype=float)
        el = np.ascontiguousarray(elems, dtype=np.int64)
        out = np.zeros(self.n_dofs)
        lib().oracle_apply_block24_subset(_p(u), _p(out), _p(el), el.size, _p(self.edofs), _p(self.occ), _p(self.k0))
        if self.dirichlet.size:
            out[self.dirichlet] = 0.0
        return out

    def diagonal(self):
        if self._diag is None:
            d = np.zeros(self.n_dofs)
            kd = np.ascontiguousarray(np.diag(self.k0))
            lib().oracle_diag_block24(_p(d), _p(self.edofs), _p(self.occ), self.occ.size, _p(kd))
            self._diag = d
        return self._diag


# ---------------------------------------------------------------------------
# deflation (topovox/fea.py:95-211)
# ---------------------------------------------------------------------------
class Deflation:
    def __init__(self, op: Operator, block=4):
        if block < 2:
            raise ValueError("agglomerate side must be >= 2")
        self.op = op
        self.block = b = int(block)
        nx, ny, nz = op.nx, op.ny, op.nz
        fixed = ~op.free
        solid = (op.occ == 1.0) & op.design_mask
        structural = np.zeros(op.n_dofs // 3, dtype=bool)
        structural[(op.edofs[solid][:, ::3] // 3).ravel()] = True
        e = np.arange(nx * ny * nz)
        ix, iy, iz = e % nx, (e // nx) % ny, e // (nx * ny)
        mx, my = (nx - 1) // b + 1, (ny - 1) // b + 1
        bid = ix // b + mx * (iy // b + my * (iz // b))
        coords = node_coords(nx, ny, nz, op.h)
        order = np.argsort(bid, kind="stable")
        bounds = np.searchsorted(bid[order], np.arange(bid.max() + 2))
        ci, cj, cv = [], [], []
        self.block_elems = []
        self.block_of_col = []
        ncols = 0
        for blk in range(bid.max() + 1):
            elems = order[bounds[blk]:bounds[blk + 1]]
            if elems.size == 0 or not solid[elems].any():
                continue
            nodes = np.unique(op.edofs[elems][:, ::3] // 3)
            nodes = nodes[structural[nodes]]
            if nodes.size == 0:
                continue
            rel = coords[nodes] - coords[nodes].mean(axis=0)
            basis = np.zeros((3 * nodes.size, 6))
            basis[0::3, 0] = 1.0
            basis[1::3, 1] = 1.0
            basis[2::3, 2] = 1.0
            basis[1::3, 3], basis[2::3, 3] = -rel[:, 2], rel[:, 1]
            basis[0::3, 4], basis[2::3, 4] = rel[:, 2], -rel[:, 0]
            basis[0::3, 5], basis[1::3, 5] = -rel[:, 1], rel[:, 0]
            dofs = (3 * nodes[:, None] + np.arange(3)).ravel()
            basis[fixed[dofs]] = 0.0
            q, r = np.linalg.qr(basis)
            rd = np.abs(np.diag(r))
            keep = rd > 1e-10 * max(rd.max(), 1e-300)
            q = q[:, keep]
            if q.shape[1] == 0:
                continue
            x0, x1 = max(ix[elems].min() - 1, 0), min(ix[elems].max() + 1, nx - 1)
            y0, y1 = max(iy[elems].min() - 1, 0), min(iy[elems].max() + 1, ny - 1)
            z0, z1 = max(iz[elems].min() - 1, 0), min(iz[elems].max() + 1, nz - 1)
            near = np.flatnonzero((ix >= x0) & (ix <= x1) & (iy >= y0) & (iy <= y1) & (iz >= z0) & (iz <= z1))
            for j in range(q.shape[1]):
                ci.append(dofs)
                cj.append(np.full(dofs.size, ncols + j))
                cv.append(q[:, j])
                self.block_elems.append(near)
                self.block_of_col.append(blk)
            ncols += q.shape[1]
        self.n_vectors = ncols
        self.W = None
        if ncols:
            self.W = scipy.sparse.csc_matrix((np.concatenate(cv), (np.concatenate(ci), np.concatenate(cj))),
                                             shape=(op.n_dofs, ncols))
        self._prepared = False

    def prepare(self):
        if self.W is None or self._prepared:
            return
        op = self.op
        cols = []
        for j in range(self.n_vectors):
            w = np.zeros(op.n_dofs)
            a, b = self.W.indptr[j], self.W.indptr[j + 1]
            w[self.W.indices[a:b]] = self.W.data[a:b]
            cols.append(scipy.sparse.csc_matrix(op.apply_subset(w, self.block_elems[j]).reshape(-1, 1)))
        self.KW = scipy.sparse.hstack(cols, format="csc")
        E = np.asarray((self.W.T @ self.KW).todense())
        self.E = 0.5 * (E + E.T)
        try:
            self._chol = scipy.linalg.cho_factor(self.E)
            self._pinv = None
        except scipy.linalg.LinAlgError:
            self._chol = None
            self._pinv = np.linalg.pinv(self.E)
        self._prepared = True

    def coarse_solve(self, y):
        if self._chol is not None:
            return scipy.linalg.cho_solve(self._chol, y)
        return self._pinv @ y


def solve_static(op: Operator, f, tol=1e-8, max_iters=None, deflation: Deflation | None = None, observer=None):
    """Deflated Jacobi PCG, step for step topovox/fea.py:218-299.
    Returns (u, iterations, residual).

    ``observer(it, x, res)`` (fixture generation only) is called after every
    iteration's residual update; a true return value ends the loop there and
    returns that iterate (fixed DOFs zeroed) as if it had converged. It does
    not change any arithmetic of the loop."""
    if not 0.0 < tol <= 1e-2:
        raise ValueError("tolerance must lie in (0, 1e-2]")
    f = np.asarray(f, dtype=float)
    d = op.diagonal()
    free = op.free
    fnorm = np.linalg.norm(f[free])
    if fnorm == 0.0:
        return np.zeros(op.n_dofs), 0, 0.0
    if np.any(d[free] == 0.0):
        raise OracleError("zero stiffness diagonal on a loaded free DOF")
    inv_d = np.zeros(op.n_dofs)
    inv_d[free] = 1.0 / d[free]
    if max_iters is None:
        max_iters = max(200, int(10 * np.sqrt(op.n_dofs)))
    defl = deflation if (deflation is not None and deflation.W is not None) else None
    if defl is not None:
        defl.prepare()

        def project_out(v):
            return defl.W @ defl.coarse_solve(np.asarray(defl.KW.T @ v).ravel())

        x = np.asarray(defl.W @ defl.coarse_solve(np.asarray(defl.W.T @ f).ravel())).ravel()
    else:
        x = np.zeros(op.n_dofs)
    r = f - op.apply(x) if np.any(x) else f.copy()
    r[~free] = 0.0
    res = np.linalg.norm(r) / fnorm
    if res <= tol:
        return x, 0, res
    z = inv_d * r
    p = z - project_out(z) if defl is not None else z.copy()
    rz = r @ z
    for it in range(1, max_iters + 1):
        q = op.apply(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        res = np.linalg.norm(r) / fnorm
        if res <= tol:
            break
        if observer is not None and observer(it, x, res):
            break
        z = inv_d * r
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p - project_out(z) if defl is not None else z + beta * p
    else:
        raise OracleNoConvergence(f"CG did not reach {tol:g} in {max_iters} iterations", res, max_iters)
    x[~free] = 0.0
    return x, it, res


def dense_stiffness(op: Operator):
    """Assembled raw K (small systems only, topovox/fea.py:324-332)."""
    K = np.zeros((op.n_dofs, op.n_dofs))
    for e in range(op.occ.size):
        dd = op.edofs[e]
        K[np.ix_(dd, dd)] += op.occ[e] * op.k0
    return K


# ---------------------------------------------------------------------------
# element state + sensitivities
# ---------------------------------------------------------------------------
def batch_element_state(op: Operator, u):
    """topovox/fea.py:302-309"""
    B = centroid_b(op.h)
    D = elasticity(op.E, op.nu)
    strains = np.asarray(u)[op.edofs] @ B.T
    stresses = (strains @ D.T) * op.occ[:, None]
    return strains, stresses, von_mises(stresses)


def compliance_sensitivity(strains, stresses, nu):
    """SPEC.md:286  T_J = 4/(1+nu) s:e - (1-3nu)/(1-nu^2) tr(s) tr(e)."""
    se = np.einsum("ij,ij->i", stresses, strains)
    tr = stresses[:, :3].sum(axis=1) * strains[:, :3].sum(axis=1)
    return 4.0 / (1.0 + nu) * se - (1.0 - 3.0 * nu) / (1.0 - nu * nu) * tr


def stress_sensitivity(stresses_u, strains_lam, nu):
    """SPEC.md:313  symmetric primal-adjoint form."""
    return compliance_sensitivity(strains_lam, stresses_u, nu)


def pnorm_stress(vm, occ, p):
    """SPEC.md:295  (sum w vm^p)^(1/p), w = occ / sum(occ)."""
    w = occ / occ.sum()
    return float(np.sum(w * vm ** p) ** (1.0 / p))


def stress_adjoint_rhs(op: Operator, u, p):
    """d sigma_PN / du (derivation SURVEY §8a a12),
    fixed DOFs zeroed."""
    strains, stresses, vm = batch_element_state(op, u)
    w = op.occ / op.occ.sum()
    S = np.sum(w * vm ** p)
    if not S > 0.0:
        raise OracleError("sigma_PN is zero: adjoint undefined")
    B = centroid_b(op.h)
    D = elasticity(op.E, op.nu)
    coef = S ** (1.0 / p - 1.0) * w * vm ** (p - 2) * op.occ
    h6 = (stresses @ Q_VM.T) @ D.T * coef[:, None]   # D Q sigma, per element
    ge = h6 @ B                                       # (N_e, 24)
    rhs = np.zeros(op.n_dofs)
    np.add.at(rhs, op.edofs, ge)
    rhs[~op.free] = 0.0
    return rhs


# ---------------------------------------------------------------------------
# eigen / buckling -- dense, small
# problems only (<= a few thousand DOFs)
# ---------------------------------------------------------------------------
def geometric_tensor(h):
    """topovox/elements.py:141-153: A[p,q,i,j] = sum_gp dNi/dx_p dNj/dx_q detJ."""
    A = np.zeros((3, 3, 8, 8))
    a = 1.0 / np.sqrt(3.0)
    for gp in a * (2.0 * OFFS - 1.0):
        dn = _dshape(*gp) * (2.0 / h)
        A += np.einsum("ip,jq->pqij", dn, dn) * (h / 2.0) ** 3
    return A


def voigt_tensor(s):
    """(..., 6) Voigt (xx, yy, zz, xy, yz, zx) -> (..., 3, 3)."""
    s = np.asarray(s)
    t = np.empty(s.shape[:-1] + (3, 3))
    t[..., 0, 0], t[..., 1, 1], t[..., 2, 2] = s[..., 0], s[..., 1], s[..., 2]
    t[..., 0, 1] = t[..., 1, 0] = s[..., 3]
    t[..., 1, 2] = t[..., 2, 1] = s[..., 4]
    t[..., 2, 0] = t[..., 0, 2] = s[..., 5]
    return t


def stress_blocks(stresses, h):
    """Per-element 8x8 initial-stress blocks sum_pq sigma_pq A[p,q]."""
    return np.einsum("epq,pqij->eij", voigt_tensor(stresses), geometric_tensor(h))


def apply_nodal_block8(op: Operator, u, blocks):
    """topovox/backends/numpy_kernels.py:26-30 (numba_kernels.py:61-76):
    sum_e P_e^T (B_e (x) I3) P_e u, unmasked."""
    dofs = op.edofs.reshape(-1, 8, 3)
    fe = np.einsum("eij,eja->eia", blocks, np.asarray(u)[dofs])
    out = np.zeros(op.n_dofs)
    np.add.at(out, dofs, fe)
    return out


def dense_geometric(op: Operator, stresses):
    """Assembled K_G (raw) from the element stresses."""
    blocks = stress_blocks(stresses, op.h)
    K = np.zeros((op.n_dofs, op.n_dofs))
    for e in range(op.occ.size):
        d = op.edofs[e].reshape(8, 3)
        for a in range(3):
            K[np.ix_(d[:, a], d[:, a])] += blocks[e]
    return K


def lumped_mass(op: Operator, rho):
    """rho h^3 / 8 occupancy_e to each corner, per DOF."""
    m = np.zeros(op.n_dofs)
    np.add.at(m, op.edofs, np.repeat(rho * op.h ** 3 / 8.0 * op.occ[:, None], 24, axis=1))
    return m


def dense_modal(op: Operator, rho, k):
    """k smallest eigenpairs of K u = lambda M u on the free DOFs (scipy eigh)."""
    import scipy.linalg

    f = op.free
    K = dense_stiffness(op)[np.ix_(f, f)]
    M = lumped_mass(op, rho)[f]
    w, V = scipy.linalg.eigh(K, np.diag(M))
    U = np.zeros((op.n_dofs, k))
    U[f] = V[:, :k]
    return w[:k], U


def buckling_cap(strains, frac=0.1):
    """Search cap of the load factor ("below a search cap"): the
    factor at which the largest reference strain component reaches `frac`
    (10 %), far outside linear buckling theory (builder decision)."""
    m = float(np.abs(strains).max()) if np.size(strains) else 0.0
    return frac / m if m > 0.0 else np.inf


def dense_buckling(op: Operator, stresses, k, cap=np.inf):
    """k smallest positive lambda <= cap of K phi = lambda K_sigma phi,
    K_sigma = -K_G, on the free DOFs: via K^-1 K_sigma's largest
    positive mu."""
    import scipy.linalg

    f = op.free
    K = dense_stiffness(op)[np.ix_(f, f)]
    Ks = -dense_geometric(op, stresses)[np.ix_(f, f)]
    mu, V = scipy.linalg.eigh(Ks, K)  # Ks v = mu K v, mu = 1 / lambda
    order = np.argsort(-mu)
    mu, V = mu[order], V[:, order]
    pos = (mu > 1e-8 * np.abs(mu).max()) & (mu >= 1.0 / cap)
    lam = 1.0 / mu[pos][:k]
    U = np.zeros((op.n_dofs, lam.size))
    U[f] = V[:, pos][:, :k]
    return lam, U


def eigen_sensitivity(op: Operator, mode, omega2, rho):
    """T_lambda = sigma(u):eps(u) - omega^2 rho_e |u_centroid|^2,
    rho_e = rho occupancy_e (the mass operator's density)."""
    strains, stresses, _ = batch_element_state(op, mode)
    se = np.einsum("ij,ij->i", stresses, strains)
    uc = np.asarray(mode)[op.edofs].reshape(-1, 8, 3).mean(axis=1)
    return se - omega2 * rho * op.occ * np.einsum("ij,ij->i", uc, uc)


def buckling_sensitivity(op: Operator, stresses, mode, lam):
    """T_p = u_e^T K^e u_e - lambda u_e^T K_sigma^e u_e with
    K^e = occ_e k0 and K_sigma^e = -(B_e (x) I3)."""
    ue = np.asarray(mode)[op.edofs]  # (ne, 24)
    e1 = op.occ * np.einsum("ei,ij,ej->e", ue, op.k0, ue)
    blocks = stress_blocks(stresses, op.h)
    u3 = ue.reshape(-1, 8, 3)
    e2 = np.einsum("eia,eij,eja->e", u3, blocks, u3)
    return e1 + lam * e2


def normalize_field(t):
    """SPEC.md:378"""
    t = np.asarray(t, dtype=float)
    m = np.abs(t).max() if t.size else 0.0
    return t.copy() if m == 0.0 else t / m


def combine(fields, weights, fallback=0):
    """sum_i w_i * normalize(T_i); all-zero weights fall
    back to field `fallback` with unit weight."""
    weights = [float(w) for w in weights]
    if all(w == 0.0 for w in weights):
        return normalize_field(fields[fallback]), True
    out = np.zeros_like(np.asarray(fields[0], dtype=float))
    for f, w in zip(fields, weights):
        if w != 0.0:
            out = out + w * normalize_field(f)
    return out, False


def extract_count(target_vf, n_design):
    return int(min(max(np.floor(target_vf * n_design + 0.5), 0), n_design))


def extract(levelset, design_mask, target_vf, ersatz, all_ties=False):
    """SPEC.md:396 order-statistic threshold over design elements; equal
    values are taken in ascending element index (all_ties: every design
    element equal to the threshold, the casting mode). Returns (occ, tau, k)."""
    ls = np.asarray(levelset, dtype=float)
    idx = np.flatnonzero(design_mask)
    k = extract_count(target_vf, idx.size)
    order = np.lexsort((idx, -ls[idx]))  # value descending, index ascending
    occ = np.full(ls.size, ersatz)
    chosen = idx[order[:k]]
    occ[chosen] = 1.0
    tau = ls[idx[order[k - 1]]] if k > 0 else np.inf
    if all_ties and k > 0:
        occ[idx[ls[idx] == tau]] = 1.0
    return occ, tau, k


def casting_project(field, dims, axis, parting):
    """SPEC.md:402-410 (PAPER §3.7): along every element column parallel to
    `axis` (0/1/2), the running minimum moving away from the parting plane;
    element layers >= parting are the +axis mold half, < parting the -axis
    half. Field in element order e = x + nx (y + ny z)."""
    nx, ny, nz = dims
    f = np.asarray(field, dtype=float).reshape(nz, ny, nx)  # [z, y, x]
    ax = 2 - axis
    f = np.moveaxis(f, ax, 0).copy()  # [axis, ...]
    if parting < f.shape[0]:
        f[parting:] = np.minimum.accumulate(f[parting:], axis=0)
    if parting > 0:
        f[:parting] = np.minimum.accumulate(f[:parting][::-1], axis=0)[::-1]
    return np.moveaxis(f, 0, ax).reshape(-1)


def undercut_violations(occ, dims, axis, parting):
    """Exhaustive column audit: per column and mold half,
    the occupied cells (occ == 1) must form one run starting at the parting
    plane. Returns the number of violating (column, half) pairs."""
    nx, ny, nz = dims
    o = np.moveaxis((np.asarray(occ) == 1.0).reshape(nz, ny, nx), 2 - axis, 0)
    bad = 0
    for half in (o[parting:], o[:parting][::-1]):
        if half.shape[0] == 0:
            continue
        run = np.logical_and.accumulate(half, axis=0)  # contiguous from the plane
        bad += int(np.any(half != run, axis=0).sum())
    return bad


# --- augmented Lagrangian scalars --------------------------
def constraint_g(q, q0, alpha, sense):
    return q / (alpha * q0) - 1.0 if sense == "upper" else 1.0 - q / (alpha * q0)


def auglag_term(g, mu, gamma):
    return mu * g + 0.5 * gamma * g * g if mu + gamma * g > 0.0 else 0.5 * mu * mu / gamma


def update_multiplier(mu, gamma, g):
    return max(mu + gamma * g, 0.0)


def update_penalty(gamma, g_prev, g_new, k, varsigma=0.25, eta=10.0):
    if min(g_new, 0.0) <= varsigma * min(g_prev, 0.0):
        return gamma
    return max(eta * gamma, float(k * k))


# ---------------------------------------------------------------------------
# optimizer loop (SPEC.md:146-154 fixed point, SPEC.md:237-246 run), restated
# independently for whole-run checks on small grids. Constraints: compliance
# and p-norm stress per load case (the SPEC kinds used by the configs).
# ---------------------------------------------------------------------------
def _analyses(nx, ny, nz, occ, cases, specs, E, nu, tol, block, need_fields=True, rho=1.0):
    """cases: list of (fixed_dofs, f); specs: list of dicts(kind, alpha, soft,
    case, p[, sense]). Eigenvalue / buckling kinds use the dense eigen
    oracles (small problems only)."""
    out = {"q": {}, "fields": {}, "J": 0.0}
    for ci, (fixed, f) in enumerate(cases):
        op = Operator(nx, ny, nz, 1.0, occ, E=E, nu=nu, dirichlet=fixed)
        defl = Deflation(op, block) if block else None
        u, _, _ = solve_static(op, f, tol=tol, deflation=defl)
        J = float(f @ u)
        out["J"] += J
        strains, stresses, vm = batch_element_state(op, u)
        for i, s in enumerate(specs):
            if s["case"] != ci:
                continue
            if s["kind"] == "compliance":
                out["q"][i] = J
                out["fields"][i] = compliance_sensitivity(strains, stresses, nu)
            elif s["kind"] == "pnorm_stress":
                out["q"][i] = pnorm_stress(vm, op.occ, s["p"])
                if need_fields:
                    lam, _, _ = solve_static(op, stress_adjoint_rhs(op, u, s["p"]), tol=tol, deflation=defl)
                    ls, _, _ = batch_element_state(op, lam)
                    out["fields"][i] = stress_sensitivity(stresses, ls, nu)
            elif s["kind"] == "eigenvalue":
                w, U = dense_modal(op, rho, 1)
                out["q"][i] = float(w[0])
                out["fields"][i] = eigen_sensitivity(op, U[:, 0], w[0], rho)
            elif s["kind"] == "buckling":
                lam, U = dense_buckling(op, stresses, 1, buckling_cap(strains))
                if lam.size == 0:
                    out["q"][i] = np.inf
                    out["fields"][i] = np.zeros(op.occ.size)
                else:
                    phi = U[:, 0] / np.linalg.norm(U[:, 0].reshape(-1, 3), axis=1).max()
                    out["q"][i] = float(lam[0])
                    out["fields"][i] = buckling_sensitivity(op, stresses, phi, lam[0])
    return out


def constraint_value(q, q0, alpha, sense):
    """SPEC.md:469 with the +inf sentinel rule of the device driver."""
    if np.isinf(q) or np.isinf(q0):
        if (sense == "lower" and q > 0) or np.isinf(q0):
            return -1.0
    return constraint_g(q, q0, alpha, sense)


def run_optimizer(nx, ny, nz, cases, specs, E=1.0, nu=0.3, tol=1e-8, block=4, ersatz=1e-6, mu0=100.0, gamma0=10.0,
                  varsigma=0.25, eta=10.0, dv0=0.025, dv_min=0.005, growth=1.1, growth_after=3, inner_cap=10,
                  ctol=0.01, ttol=0.001, feas=1e-6, max_outer=400, casting=None, rho=1.0, trace=None):
    """Returns (occ, history list of dicts, reason). casting: (axis, parting
    element layer) -> casting-projected extraction with all ties retained.
    trace(record) (fixture generation only) receives every extraction:
    dict(k, it, occ = topology the fields were computed on, weights, target,
    levelset, tau, new_occ)."""
    ne = nx * ny * nz
    design = np.ones(ne, dtype=bool)
    occ = np.ones(ne)
    base = _analyses(nx, ny, nz, occ, cases, specs, E, nu, tol, block, rho=rho)
    q0 = dict(base["q"])
    sense = [s.get("sense", "lower" if s["kind"] in ("eigenvalue", "buckling") else "upper") for s in specs]
    gfun = lambda q: {i: constraint_value(q[i], q0[i], s["alpha"], sense[i])  # noqa: E731
                      for i, s in enumerate(specs)}
    g = gfun(base["q"])
    mu = {i: mu0 for i in range(len(specs))}
    gam = {i: gamma0 for i in range(len(specs))}
    acc_occ, acc = occ, base
    dv, streak, hist, reason = dv0, 0, [], "max_outer"
    fb = next((i for i, s in enumerate(specs) if s["kind"] == "compliance"), 0)
    for k in range(1, max_outer + 1):
        v = float(np.count_nonzero(acc_occ == 1.0)) / ne
        target = v - dv
        if target <= 1.0 / ne:
            reason = "minimum volume reached"
            break
        w = {i: max(mu[i] + gam[i] * g[i], 0.0) for i in range(len(specs))}
        cur, cur_occ = acc, acc_occ
        conv, inner = False, 0
        for it in range(1, inner_cap + 1):
            inner = it
            ls, _ = combine([cur["fields"][i] for i in range(len(specs))], [w[i] for i in range(len(specs))],
                            fallback=fb)
            if casting is not None:
                ls = casting_project(ls, (nx, ny, nz), *casting)
            new_occ, tau, _ = extract(ls, design, target, ersatz, all_ties=casting is not None)
            if trace is not None:
                trace(dict(k=k, it=it, occ=cur_occ, weights=[w[i] for i in range(len(specs))], target=target,
                           levelset=ls, tau=tau, new_occ=new_occ))
            if it > 1 and np.count_nonzero((new_occ == 1.0) != (cur_occ == 1.0)) < ttol * ne:
                conv = True
                break
            nxt = _analyses(nx, ny, nz, new_occ, cases, specs, E, nu, tol, block, rho=rho)
            if it > 1 and abs(nxt["J"] - cur["J"]) < ctol * cur["J"]:
                cur, cur_occ, conv = nxt, new_occ, True
                break
            cur, cur_occ = nxt, new_occ
        g_new = gfun(cur["q"])
        hard = any((not s.get("soft", False)) and g_new[i] > feas for i, s in enumerate(specs))
        hist.append({"k": k, "v": float(np.count_nonzero(cur_occ == 1.0)) / ne, "dv": dv, "accepted": not hard,
                     "g": dict(g_new), "J": cur["J"], "inner": inner})
        if hard:
            dv *= 0.5
            streak = 0
            if dv < dv_min:
                reason = "volume step below dv_min with a hard constraint violated"
                break
            continue
        for i in range(len(specs)):
            nm = update_multiplier(mu[i], gam[i], g_new[i])
            gam[i] = update_penalty(gam[i], g[i], g_new[i], k, varsigma, eta)
            mu[i] = nm
        g, acc, acc_occ = g_new, cur, cur_occ
        streak += 1
        if streak >= growth_after:
            dv = min(dv * growth, dv0)
    return acc_occ, hist, reason
