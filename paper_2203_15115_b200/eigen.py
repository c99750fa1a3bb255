"""Eigen and buckling analyses on the GPU (SPEC
``eigen_buckling``, fields SPEC.md:319-336).

The reference ships only the building blocks -- the geometric-stiffness seam
``apply_nodal_block8`` (``topovox/backends/numba_kernels.py:61-76``) and
``geometric_tensor`` (``topovox/elements.py:141-153``) -- so the operations
follow the SPEC:

* ``MassOperator``                lumped rho h^3/8 * occupancy per corner  (``tvb_lumped_mass``)
* ``geometric_stiffness``         K_sigma from the element stresses of a static solve
                                  (``tvb_geo_matvec``: stress contracted with geometric_tensor on the fly)
* ``solve_modal``                 K u = lambda M u, k smallest pairs
* ``solve_buckling``              K phi = lambda K_sigma phi, smallest positive factor
* ``eigen_sensitivity``           T_lambda = sigma:eps - omega^2 rho |u_c|^2   (``tvb_eigen_sens``)
* ``buckling_sensitivity``        T_p = u^T (K^e - lambda K_sigma^e) u       (``tvb_buckling_sens``)

Eigensolver: shift-invert subspace iteration whose inner
inverse is the deflated-CG solver -- the q subspace columns of an iteration
are ONE multi-RHS batch (``fea.solve_static_batch``), so the operator, the
coarse factor and the CUDA graph are shared. The q x q Rayleigh-Ritz problem
is solved on the device (cuSOLVER via torch; plumbing, q <= 16).

Sign convention (documented builder decision): ``K_G`` is the
reference's initial-stress operator (blocks sum_pq sigma_pq A[p,q], positive
for tension); buckling uses ``K_sigma = -K_G`` so a compressive reference
load has positive critical factors and pure tension has none.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr, require_cuda, stream_ptr
from .elements import geometric_voigt_blocks
from .errors import DimensionMismatch, NoConvergence, ZeroMassSubspace
from .fea import StiffnessOperator, solve_static, solve_static_batch, to_device, to_host_if

#: default relative residual of an eigenpair
EIGEN_TOL = 1.0e-6
#: buckling search cap: factors whose scaled reference state strains beyond this are not reported
BUCKLING_CAP_STRAIN = 0.1


def _t():
    return require_cuda()


@dataclass
class EigenResult:
    """ascending values, their modes, per-pair residuals.
    Modal vectors are M-normalised; buckling vectors have unit maximum nodal
    displacement. ``no_positive_factor``: buckling found no positive factor
    (values == [inf], the P = +inf sentinel)."""

    values: list
    vectors: list
    residuals: list
    iterations: int = 0
    solves: int = 0
    no_positive_factor: bool = False
    excluded_dofs: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))


class MassOperator:
    """Lumped (diagonal) mass: rho h^3 occupancy_e / 8 to each corner node
    (SPEC.md:207-210). Fixed DOFs carry zero mass (Dirichlet applied to K and
    M consistently)."""

    def __init__(self, op: StiffnessOperator, rho: float | None = None):
        torch = _t()
        d = op.domain
        self.op = op
        self.rho = float(op.material.rho if rho is None else rho)
        if not self.rho > 0.0:
            raise ValueError(f"density must be positive, got {self.rho}")
        coef = self.rho * d.h ** 3 / 8.0
        self.diag_d = torch.empty(d.n_dofs, dtype=torch.float64, device="cuda")
        check(lib().tvb_lumped_mass(d.nx, d.ny, d.nz, coef, ptr(op.occ_d), ptr(self.diag_d), stream_ptr()),
              "lumped mass")
        self.total = float(self.diag_d[0::3].sum()) if d.n_dofs else 0.0  # rho h^3 sum occ (before masking)
        if op.dirichlet.size:
            self.diag_d[op.fixed_d] = 0.0

    @property
    def n_dofs(self) -> int:
        return self.op.n_dofs

    def apply_device(self, v):
        return self.diag_d * v

    def apply(self, v):
        v_d, np_in = to_device(v, self.n_dofs, "vector")
        return to_host_if(self.apply_device(v_d), np_in)

    def diagonal(self) -> np.ndarray:
        return self.diag_d.cpu().numpy()


class GeometricStiffnessOperator:
    """K_sigma = -K_G of a static stress state.

    ``stresses``: (Ne, 6) occupancy-scaled Voigt centroid stresses of the
    reference static solve; element blocks are contracted from them on the fly
    (never stored). Linear in the reference load; zero stress -> zero operator."""

    def __init__(self, op: StiffnessOperator, stresses_d, strain_max: float | None = None):
        torch = _t()
        ne = op.domain.n_elems
        if tuple(stresses_d.shape) != (ne, 6):
            raise DimensionMismatch(f"stress field has shape {tuple(stresses_d.shape)}, expected ({ne}, 6)")
        self.op = op
        self.stresses_d = stresses_d.to(device="cuda", dtype=torch.float64).contiguous()
        self.Bk_d = torch.from_numpy(geometric_voigt_blocks(op.domain.h)).cuda().contiguous()
        #: largest |strain component| of the reference state (buckling search cap), if known
        self.strain_max = strain_max

    def search_cap(self, frac: float = BUCKLING_CAP_STRAIN) -> float:
        """Load factor at which the reference strain reaches ``frac`` (SPEC.md:242
        "search cap"; builder decision: beyond 10 % strain linear buckling
        theory is void). inf when the strains are unknown or zero."""
        if not self.strain_max:
            return math.inf
        return frac / self.strain_max

    @property
    def n_dofs(self) -> int:
        return self.op.n_dofs

    def apply_device(self, v, out=None, raw: bool = False):
        """K_sigma v on device tensors (Dirichlet rows/columns zeroed unless raw)."""
        torch = _t()
        d = self.op.domain
        if out is None:
            out = torch.empty_like(v)
        flags = 0 if (raw or not self.op.dirichlet.size) else 3
        check(lib().tvb_geo_matvec(d.nx, d.ny, d.nz, ptr(self.Bk_d), ptr(self.stresses_d), ptr(v), ptr(out),
                                   ptr(self.op.nflags), flags, -1.0, stream_ptr()), "geometric stiffness")
        return out

    def apply(self, v, raw: bool = False):
        v_d, np_in = to_device(v, self.n_dofs, "vector")
        return to_host_if(self.apply_device(v_d, raw=raw), np_in)


def geometric_stiffness(u_ref, op: StiffnessOperator) -> GeometricStiffnessOperator:
    """K_sigma of the static state u_ref."""
    from .sensitivity import element_state_device

    u_d, _ = to_device(u_ref, op.n_dofs, "reference displacement")
    strains, stresses, _ = element_state_device(op, u_d, want=("strains", "stresses"))
    return GeometricStiffnessOperator(op, stresses, strain_max=float(strains.abs().max()))


# ---------------------------------------------------------------------------
# shift-invert subspace iteration
# ---------------------------------------------------------------------------
def _inner_tol(tol: float) -> float:
    """Inner (deflated-CG) tolerance for an eigen residual target `tol`."""
    return min(1e-8, max(1e-13, 1e-2 * tol))


def _inner_iters(op) -> int:
    """Generous inner cap: low-volume ersatz topologies stagnate slowly."""
    from .fea import default_max_iters

    return 4 * default_max_iters(op.n_dofs)


def _inner_solver(op, deflation, shift, mass, inner_tol):
    """X -> (K + shift M)^-1 X column batch on the device."""
    torch = _t()
    if shift == 0.0:
        return lambda cols: [r.u for r in solve_static_batch(op, cols, tol=inner_tol, deflation=deflation,
                                                             max_iters=_inner_iters(op))]
    kd = op.diagonal_device() + shift * mass.diag_d

    def apply(v):
        return op.apply_device(v) + shift * mass.diag_d * v

    return lambda cols: [solve_static(op, c, tol=inner_tol, apply_op=apply, diag=kd, max_iters=_inner_iters(op)).u
                         for c in cols]


def _rayleigh_ritz(A, B):
    """Generalised symmetric q x q problem A v = w B v (B SPD): ascending w, V
    with V^T B V = I."""
    torch = _t()
    A = 0.5 * (A + A.T)
    B = 0.5 * (B + B.T)
    L = torch.linalg.cholesky(B)
    Li = torch.linalg.inv(L)
    C = Li @ A @ Li.T
    w, Y = torch.linalg.eigh(0.5 * (C + C.T))
    return w, Li.T @ Y


def _start_block(n, q, active, seed):
    torch = _t()
    X = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, q))).cuda()
    X[~active] = 0.0
    return X


def solve_modal(op: StiffnessOperator, mass: MassOperator, k: int = 1, tol: float = EIGEN_TOL, deflation=None,
                max_iters: int = 300, subspace: int | None = None, shift: float | None = None, seed: int = 0,
                inner_tol: float | None = None) -> EigenResult:
    """k smallest eigenpairs of K u = lambda M u; lambda = omega^2.

    Shift-invert subspace iteration, inner solves (K + s M)^-1 by the
    deflated-CG batch (s = 0 when the Dirichlet set makes K SPD; a free-free
    operator is shifted, s > 0, and solved with the generic PCG path).
    Raises NoConvergence with the attained residuals."""
    torch = _t()
    if k < 1:
        raise ValueError("k must be >= 1")
    n = op.n_dofs
    free = torch.from_numpy(op.free_mask).cuda()
    m = mass.diag_d
    zero = free & (m == 0.0)
    excluded = np.flatnonzero(zero.cpu().numpy())
    if excluded.size:
        warnings.warn(f"{excluded.size} free DOFs have zero lumped mass; excluded from the eigen subspace",
                      ZeroMassSubspace, stacklevel=2)
    active = free & (m > 0.0)
    n_act = int(active.sum())
    if n_act < k:
        raise ValueError(f"only {n_act} DOFs carry mass, cannot find {k} eigenpairs")
    q = min(subspace or max(2 * k, k + 7), n_act)
    if shift is None:
        if op.dirichlet.size:
            shift = 0.0
        else:  # free-free: K singular (rigid modes); shift by ~1e-2 of the mean diagonal ratio
            kd = op.diagonal_device()
            shift = 1e-2 * float((kd[active] / m[active]).mean())
    inner_tol = inner_tol if inner_tol is not None else _inner_tol(tol)
    solve = _inner_solver(op, deflation, shift, mass, inner_tol)
    X = _start_block(n, q, active, seed)
    w = None
    solves = 0
    res = [math.inf] * k
    for it in range(1, max_iters + 1):
        Y = m[:, None] * X
        cols = solve([Y[:, j].contiguous() for j in range(q)])
        solves += q
        Xb = torch.stack(cols, dim=1)
        Xb[~active] = 0.0
        A = Xb.T @ Y                       # X^T (K + sM) X with (K + sM) Xb = Y
        B = Xb.T @ (m[:, None] * Xb)
        w, V = _rayleigh_ritz(A, B)
        X = Xb @ V                         # M-orthonormal Ritz vectors
        lam = w[:k] - shift
        scale = float(w[-1] - shift)  # largest Ritz value: the problem's elastic scale
        res = []
        for j in range(k):
            x = X[:, j].contiguous()
            kx = op.apply_device(x)
            r = kx - lam[j] * (m * x)
            num = float(torch.linalg.norm(r[free]))
            # ||K u - lambda M u|| / ||K u||; a rigid mode (K u ~ 0)
            # is measured against the subspace's elastic scale instead
            den = float(torch.linalg.norm(kx[free]))
            if not float(lam[j]) > 1e-8 * scale:
                den = max(den, scale * float(torch.linalg.norm((m * x)[free])))
            res.append(num / den if den > 0.0 else num)
        if all(r <= tol for r in res):
            vals = [float(v) for v in lam.cpu()]
            vecs = [X[:, j].contiguous() for j in range(k)]
            return EigenResult(vals, vecs, res, iterations=it, solves=solves, excluded_dofs=excluded)
    raise NoConvergence(f"modal subspace iteration did not reach {tol:g} in {max_iters} iterations "
                        f"(residuals {res})", residual=max(res), iterations=max_iters)


def solve_buckling(op: StiffnessOperator, geo: GeometricStiffnessOperator, k: int = 1, tol: float = EIGEN_TOL,
                   deflation=None, max_iters: int = 300, subspace: int | None = None, seed: int = 0,
                   inner_tol: float | None = None, positive_rel: float = 1e-8,
                   lambda_cap: float | None = None) -> EigenResult:
    """Smallest positive load factors of K phi = lambda K_sigma phi
    (SPEC.md:238-248). Subspace iteration on K^-1 K_sigma (mu = 1/lambda,
    largest positive mu first); the q inner solves per iteration are one
    deflated-CG batch. No factor in (0, lambda_cap] (pure tension / zero
    stress; cap default ``geo.search_cap()``) -> P = +inf sentinel
    (no_positive_factor)."""
    torch = _t()
    if k < 1:
        raise ValueError("k must be >= 1")
    n = op.n_dofs
    free = torch.from_numpy(op.free_mask).cuda()
    n_free = int(free.sum())
    q = min(subspace or max(2 * k, k + 7), n_free)
    inner_tol = inner_tol if inner_tol is not None else _inner_tol(tol)
    cap = geo.search_cap() if lambda_cap is None else float(lambda_cap)
    mu_min = 1.0 / cap if cap > 0.0 else math.inf
    X = _start_block(n, q, free, seed)
    solves = 0
    res = [math.inf] * k
    inf_result = lambda it: EigenResult([math.inf], [], [0.0], iterations=it, solves=solves,  # noqa: E731
                                        no_positive_factor=True)
    for it in range(1, max_iters + 1):
        Y = torch.stack([geo.apply_device(X[:, j].contiguous()) for j in range(q)], dim=1)
        if not bool(Y.any()):
            return inf_result(it)  # zero stress state: K_sigma = 0
        cols = [r.u for r in solve_static_batch(op, [Y[:, j].contiguous() for j in range(q)], tol=inner_tol,
                                                deflation=deflation, max_iters=_inner_iters(op))]
        solves += q
        Xb = torch.stack(cols, dim=1)
        B = Xb.T @ Y                       # Xb^T K Xb
        KsXb = torch.stack([geo.apply_device(Xb[:, j].contiguous()) for j in range(q)], dim=1)
        A = Xb.T @ KsXb
        mu, V = _rayleigh_ritz(A, B)       # ascending mu
        mu = torch.flip(mu, (0,))
        V = torch.flip(V, (1,))
        X = Xb @ V
        mmax = float(mu.abs().max())
        pos = [j for j in range(q) if float(mu[j]) > positive_rel * mmax and float(mu[j]) >= mu_min]
        if not pos:
            if it >= 3:
                return inf_result(it)
            continue
        take = pos[:k]
        lam = [1.0 / float(mu[j]) for j in take]
        res = []
        for j, lj in zip(take, lam):
            x = X[:, j].contiguous()
            kx = op.apply_device(x)
            r = kx - lj * geo.apply_device(x)
            den = float(torch.linalg.norm(kx[free]))
            res.append(float(torch.linalg.norm(r[free])) / den if den > 0.0 else math.inf)
        if len(take) == k and all(r <= tol for r in res):
            vecs = []
            for j in take:
                x = X[:, j].contiguous()
                mag = x.view(-1, 3).norm(dim=1)
                i = int(torch.argmax(mag))
                node = x.view(-1, 3)[i]
                sgn = 1.0 if float(node[int(torch.argmax(node.abs()))]) >= 0.0 else -1.0
                vecs.append(sgn * x / float(mag[i]))
            return EigenResult(lam, vecs, res, iterations=it, solves=solves)
    raise NoConvergence(f"buckling subspace iteration did not reach {tol:g} in {max_iters} iterations "
                        f"(residuals {res})", residual=max(res), iterations=max_iters)


# ---------------------------------------------------------------------------
# sensitivity fields
# ---------------------------------------------------------------------------
def eigen_sensitivity(op: StiffnessOperator, mode, omega2: float, rho: float | None = None):
    """T_lambda,e = sigma(u):eps(u) - omega^2 rho_e |u(centroid)|^2 for an
    M-normalised mode; rho_e = rho * occupancy_e, the density
    the mass operator uses (builder decision)."""
    torch = _t()
    u_d, np_in = to_device(mode, op.n_dofs, "mode")
    d = op.domain
    mat = op.material
    rho = float(mat.rho if rho is None else rho)
    out = torch.empty(d.n_elems, dtype=torch.float64, device="cuda")
    check(lib().tvb_eigen_sens(d.nx, d.ny, d.nz, d.h, mat.E, mat.nu, ptr(u_d), ptr(op.occ_d), float(omega2) * rho,
                               ptr(out), stream_ptr()), "eigen sensitivity")
    return to_host_if(out, np_in)


def buckling_sensitivity(op: StiffnessOperator, geo: GeometricStiffnessOperator, mode, lam: float):
    """T_p,e = u_e^T K^e u_e - lambda u_e^T K_sigma^e u_e."""
    torch = _t()
    u_d, np_in = to_device(mode, op.n_dofs, "mode")
    d = op.domain
    if getattr(op, "_k0_d", None) is None:
        op._k0_d = torch.from_numpy(np.ascontiguousarray(op.k0)).cuda()
    out = torch.empty(d.n_elems, dtype=torch.float64, device="cuda")
    check(lib().tvb_buckling_sens(d.nx, d.ny, d.nz, ptr(op._k0_d), ptr(geo.Bk_d), ptr(geo.stresses_d), ptr(u_d),
                                  ptr(op.occ_d), float(lam), ptr(out), stream_ptr()), "buckling sensitivity")
    return to_host_if(out, np_in)


__all__ = ["BUCKLING_CAP_STRAIN", "EigenResult", "MassOperator", "GeometricStiffnessOperator", "geometric_stiffness", "solve_modal",
           "solve_buckling", "eigen_sensitivity", "buckling_sensitivity", "EIGEN_TOL"]
