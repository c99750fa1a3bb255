"""How far does the REFERENCE's own DPCG iterate move under a benign rounding
change? (build container only; evidence for the parity tolerances in
tests/test_gpu_large_parity.py.)

    python tests/golden/noise_floor.py [case] [--only NAME[,NAME]]

(experiments: inverse, stabilised, noise, cancel, reverse. Measured with
"--only cancel" at c4_bern_y: x_40 4.8e-15, x_933 8.5e-12.)

Runs the reference's loop (oracle restatement, bitwise equal to it) on the
reference's operator and deflation space twice: coarse solve by sparse LU
(the fixtures' choice) and by an explicit dense inverse of the same E (the
reference's dense Cholesky is 1.6 s/iteration at n_c = 12,000). Prints the
relative difference of the iterates at the fixture's recorded iteration
counts, measured exactly like the GPU test (4096 sample DOFs)."""
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402
from topovox import fea  # noqa: E402
from topovox import mesh as refmesh  # noqa: E402
from topovox.elements import Material  # noqa: E402

import large_cases as LC  # noqa: E402
from oracle import topovox_oracle as O  # noqa: E402
from oracle.large import sparse_coarse_solver  # noqa: E402
from make_large_fixtures import RefOp  # noqa: E402

_args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = _args[0] if _args else "c3_bern"
_only = None
for _i, _a in enumerate(sys.argv):
    if _a == "--only":
        _only = set(sys.argv[_i + 1].split(","))
        _args = [a for a in _args if a != sys.argv[_i + 1]]
        name = _args[0] if _args else "c3_bern"


def want(exp):
    return _only is None or exp in _only


spec = LC.CASES[name]
fx = np.load(os.path.join(HERE, "large_dpcg.npz"))
d, fixed, f, occ = LC.problem(refmesh, spec)
op = fea.StiffnessOperator(d, refmesh.Topology(d, occ), Material(E=1.0, nu=0.3), fixed)
defl = fea.DeflationSpace(d, refmesh.Topology(d, occ), fixed, spec["block"])
defl.prepare(op)
E = np.asarray((defl.W.T @ defl.KW).todense())
E = 0.5 * (E + E.T)
idx = LC.sample_index(d.n_dofs)
tags = sorted({k[len(name) + 1:].rsplit("_", 1)[0] for k in fx.files if k.startswith(name + "_") and k.endswith("_u")})
its = sorted({int(fx[f"{name}_{t}_it"]) for t in tags})
solvers = {"splu": sparse_coarse_solver(E)}
if want("inverse"):
    solvers["dense_inverse"] = (lambda Ei: (lambda y: Ei @ y))(np.linalg.inv(E))
snaps = {}
for sname, cs in solvers.items():
    defl.coarse_solve = cs
    defl.prepare = lambda *_a: None
    got = {}

    def obs(it, x, res):
        if it in its:
            got[it] = x[idx].copy()
        return it >= its[-1]

    O.solve_static(RefOp(op), f, tol=1e-14, max_iters=its[-1], deflation=defl, observer=obs)
    snaps[sname] = got
for it in its:
    a = snaps["splu"][it]
    ref = [fx[f"{name}_{t}_u"] for t in tags if int(fx[f"{name}_{t}_it"]) == it][0]
    print(f"{name} x_{it}: splu vs fixture {np.linalg.norm(a - ref) / np.linalg.norm(ref):.2e}", flush=True)
    if want("inverse"):
        b = snaps["dense_inverse"][it]
        print(f"{name} x_{it}: splu vs dense inverse {np.linalg.norm(a - b) / np.linalg.norm(a):.2e}", flush=True)


def stabilised_loop(op, f, defl, n_iter):
    """The device solver's stabilised projection (solver.cu):
    p = z + beta p - W E^-1 W^T (A z + beta q), otherwise the reference loop."""
    free = op.free_mask
    d = op.diagonal()
    inv_d = np.zeros(op.n_dofs)
    inv_d[free] = 1.0 / d[free]
    W, cs = defl.W, defl.coarse_solve
    x = np.asarray(W @ cs(np.asarray(W.T @ f).ravel())).ravel()
    r = f - op.apply(x)
    r[~free] = 0.0
    z = inv_d * r
    p = z - W @ cs(np.asarray(W.T @ op.apply(z)).ravel())
    rz = r @ z
    out = {}
    for it in range(1, n_iter + 1):
        q = op.apply(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        if it in its:
            out[it] = x[idx].copy()
        z = inv_d * r
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p - W @ cs(np.asarray(W.T @ (op.apply(z) + beta * q)).ravel())
    return out


defl.coarse_solve = solvers["splu"]
if want("stabilised"):
    st = stabilised_loop(op, f, defl, its[-1])
    for it in its:
        a = snaps["splu"][it]
        print(f"{name} x_{it}: reference recurrence vs stabilised projection "
              f"{np.linalg.norm(a - st[it]) / np.linalg.norm(a):.2e}", flush=True)


class NoisyOp(RefOp):
    """The reference operator with each K.u entry perturbed by one rounding
    unit (relative 2^-53 x N(0, 1)): the size of the difference between two
    correct fp64 evaluations of K.u in different summation orders."""

    def __init__(self, op, seed=0):
        super().__init__(op)
        self.rng = np.random.default_rng(seed)
        self.apply = self.noisy_apply

    def noisy_apply(self, u):
        y = self.op.apply(u)
        return y * (1.0 + 2.0 ** -53 * self.rng.standard_normal(y.size))


defl.coarse_solve = solvers["splu"]
got = {}


def obs2(it, x, res):
    if it in its:
        got[it] = x[idx].copy()
    return it >= its[-1]


if want("noise"):
    O.solve_static(NoisyOp(op), f, tol=1e-14, max_iters=its[-1], deflation=defl, observer=obs2)
    for it in its:
        a = snaps["splu"][it]
        print(f"{name} x_{it}: reference vs reference with K.u rounding noise "
              f"{np.linalg.norm(a - got[it]) / np.linalg.norm(a):.2e}", flush=True)


class CancelNoiseOp(RefOp):
    """K.u with one rounding unit of error per entry RELATIVE TO (|K| |u|)_i,
    the error size of any fp64 evaluation that sums the element terms in a
    different order (where K u cancels, |K u| << |K| |u|)."""

    def __init__(self, op, seed=0):
        super().__init__(op)
        self.rng = np.random.default_rng(seed)
        self.absop = O.Operator(d.nx, d.ny, d.nz, d.h, occ, dirichlet=fixed)
        self.absop.k0 = np.ascontiguousarray(np.abs(self.absop.k0))
        self.apply = self.noisy_apply

    def noisy_apply(self, u):
        y = self.op.apply(u)
        scale = self.absop.apply(np.abs(u))
        return y + 2.0 ** -53 * self.rng.standard_normal(y.size) * scale


got = {}
if want("cancel"):
    O.solve_static(CancelNoiseOp(op), f, tol=1e-14, max_iters=its[-1], deflation=defl, observer=obs2)
    floors = {}
    for it in its:
        a = snaps["splu"][it]
        floors[it] = float(np.linalg.norm(a - got[it]) / np.linalg.norm(a))
        print(f"{name} x_{it}: reference vs reference with K.u rounding noise relative to |K||u| "
              f"{floors[it]:.2e}", flush=True)
if not want("reverse"):
    sys.exit(0)


from oracle.large import FastDeflation  # noqa: E402

# the coarse operator itself with different rounding: KW accumulated over the
# near elements in the opposite order (E = W^T K W has cancellation: W are
# near-kernel rigid modes, so its rounding error is relative to |W||K||W|)
F = FastDeflation(d.nx, d.ny, d.nz, d.h, occ, fixed, spec["block"], op.k0, reverse=True)
F.prepare()
F.prepare = lambda *_a: None
Ef = F.E.toarray()
print(f"{name}: E reversed-accumulation vs reference E: max rel entry diff "
      f"{np.abs(Ef - E).max() / np.abs(E).max():.2e}", flush=True)
got = {}
O.solve_static(RefOp(op), f, tol=1e-14, max_iters=its[-1], deflation=F, observer=obs2)
for it in its:
    a = snaps["splu"][it]
    print(f"{name} x_{it}: reference vs reference with E / KW accumulated in reverse element order "
          f"{np.linalg.norm(a - got[it]) / np.linalg.norm(a):.2e}", flush=True)
