"""Pin the CPU oracle (test infrastructure) against the real reference's
golden vectors and the SPEC's known-answer examples. CPU only."""

import numpy as np
import pytest


def test_k0_matches_reference(oracle, golden):
    assert np.array_equal(oracle.hex_stiffness(1.0, 0.3, 1.0), golden["k0_unit"])
    assert np.allclose(oracle.hex_stiffness(2e11, 0.25, 0.5), golden["k0_steel"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("name", ["mv333", "mv543", "mv171"])
def test_kernels_bitwise(oracle, golden, name):
    nx, ny, nz = golden[name + "_dims"]
    op = oracle.Operator(nx, ny, nz, 1.0, golden[name + "_occ"], dirichlet=golden[name + "_fixed"])
    u = golden[name + "_u"]
    assert np.array_equal(op.apply(u, raw=True), golden[name + "_Ku_raw"])
    assert np.array_equal(op.apply(u), golden[name + "_Ku"])
    assert np.array_equal(op.diagonal(), golden[name + "_diag"])
    assert np.array_equal(op.apply_subset(u, golden[name + "_sub"]), golden[name + "_Ku_sub"])
    s, st, vm = oracle.batch_element_state(op, u)
    assert np.array_equal(s, golden[name + "_strain"])
    assert np.array_equal(st, golden[name + "_stress"])
    assert np.array_equal(vm, golden[name + "_vm"])


@pytest.mark.parametrize("b", [2, 3])
def test_dpcg_matches_reference(oracle, golden, b):
    op = oracle.Operator(8, 6, 5, 1.0, golden["bern865_occ"], dirichlet=golden["bern865_fixed"])
    defl = oracle.Deflation(op, b)
    assert defl.n_vectors == int(golden[f"bern865_b{b}_nvec"])
    for t in (8, 12):
        u, it, res = oracle.solve_static(op, golden["bern865_f"], tol=10.0 ** -t, deflation=defl)
        ref = golden[f"bern865_b{b}_t{t}_u"]
        assert it == int(golden[f"bern865_b{b}_t{t}_iters"])
        assert np.abs(u - ref).max() <= 1e-10 * np.abs(ref).max()


def test_plain_pcg_matches_reference(oracle, golden):
    op = oracle.Operator(8, 6, 5, 1.0, golden["bern865_occ"], dirichlet=golden["bern865_fixed"])
    u, it, _ = oracle.solve_static(op, golden["bern865_f"], tol=1e-12)
    assert it == int(golden["bern865_plain_t12_iters"])
    ref = golden["bern865_plain_t12_u"]
    assert np.abs(u - ref).max() <= 1e-12 * np.abs(ref).max()


def test_dense_oracle_consistency(oracle, golden):
    nx, ny, nz = golden["mv333_dims"]
    op = oracle.Operator(nx, ny, nz, 1.0, golden["mv333_occ"])
    K = oracle.dense_stiffness(op)
    u = golden["mv333_u"]
    assert np.allclose(K @ u, golden["mv333_Ku_raw"], rtol=0, atol=1e-13 * np.abs(K @ u).max())


# --- SPEC known-answer examples ---

def test_spec_compliance_kat(oracle):
    nu, E = 0.3, 1.0
    # uniaxial unit stress: eps = (1, -nu, -nu)/E
    sig = np.array([[1.0, 0, 0, 0, 0, 0]])
    eps = np.array([[1.0, -nu, -nu, 0, 0, 0]]) / E
    assert oracle.compliance_sensitivity(eps, sig, nu)[0] == pytest.approx(3.032967, abs=1e-6)
    # pure shear sigma_12 = s: gamma = s/G = 2(1+nu)s/E -> 8 s^2 / E
    s = 0.7
    sig = np.array([[0, 0, 0, s, 0, 0]])
    eps = np.array([[0, 0, 0, 2 * (1 + nu) * s / E, 0, 0]])
    assert oracle.compliance_sensitivity(eps, sig, nu)[0] == pytest.approx(8 * s * s / E, rel=1e-12)


def test_spec_pnorm_kat(oracle):
    s = 2.5
    assert oracle.pnorm_stress(np.full(7, s), np.ones(7), 6) == pytest.approx(s, rel=1e-14)
    assert oracle.pnorm_stress(np.array([0.0, s]), np.ones(2), 6) == pytest.approx(s * 0.5 ** (1 / 6), rel=1e-14)


def test_spec_levelset_kats(oracle):
    assert np.allclose(oracle.normalize_field([2, -4, 1]), [0.5, -1, 0.25])
    assert np.all(oracle.normalize_field(np.zeros(3)) == 0)
    occ, tau, k = oracle.extract(np.array([0.1, 0.5, 0.9, 0.7]), np.ones(4, bool), 0.5, 1e-3)
    assert np.array_equal(np.flatnonzero(occ == 1.0), [2, 3])
    occ, _, _ = oracle.extract(np.random.default_rng(0).random(10), np.ones(10, bool), 1.0, 1e-3)
    assert np.all(occ == 1.0)
    a, b = np.array([1.0, -2.0]), np.array([3.0, 1.0])
    out, fb = oracle.combine([a, b], [2.0, 3.0])
    assert not fb and np.allclose(out, 2 * a / 2 + 3 * b / 3)
    out, fb = oracle.combine([a, b], [0.0, 0.0])
    assert fb and np.allclose(out, a / 2)


def test_spec_auglag_kats(oracle):
    assert oracle.constraint_g(2.0, 1.0, 2.0, "upper") == 0.0
    assert oracle.constraint_g(1.27, 1.0, 100.0, "upper") == pytest.approx(-0.9873)
    assert oracle.constraint_g(0.16, 1.0, 0.1, "lower") == pytest.approx(-0.6)
    assert oracle.auglag_term(0.5, 1.0, 2.0) == pytest.approx(0.75)
    assert oracle.auglag_term(-1.0, 1.0, 2.0) == pytest.approx(0.25)
    assert oracle.update_multiplier(100.0, 10.0, -0.2) == pytest.approx(98.0)
    assert oracle.update_multiplier(1.0, 10.0, -0.5) == 0.0
    assert oracle.update_penalty(10.0, -0.1, -0.05, 3) == 10.0
    assert oracle.update_penalty(10.0, -0.1, -0.01, 3) == 100.0
    assert oracle.update_penalty(10.0, 0.0, 0.0, 3) == 10.0


def test_adjoint_rhs_finite_difference(oracle):
    rng = np.random.default_rng(3)
    occ = np.where(rng.random(24) < 0.7, 1.0, 1e-3)
    op = oracle.Operator(4, 3, 2, 1.0, occ)
    u = rng.standard_normal(op.n_dofs)
    p = 8
    g = oracle.stress_adjoint_rhs(op, u, p)

    def spn(v):
        return oracle.pnorm_stress(oracle.batch_element_state(op, v)[2], op.occ, p)

    h = 1e-6 * np.linalg.norm(u)
    for i in rng.choice(op.n_dofs, 20, replace=False):
        e = np.zeros(op.n_dofs)
        e[i] = h
        fd = (spn(u + e) - spn(u - e)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-4 * np.abs(g).max()


def test_spec_casting_kats(oracle):
    """SPEC.md:402-410 casting_project examples + invariants (idempotence,
    undercut audit after extraction at 20 random thresholds)."""
    # column (plane -> outward) [0.5, 0.2, 0.7] -> [0.5, 0.2, 0.2], along each axis
    for axis, dims in ((0, (3, 1, 1)), (1, (1, 3, 1)), (2, (1, 1, 3))):
        out = oracle.casting_project([0.5, 0.2, 0.7], dims, axis, 0)
        assert np.array_equal(out, [0.5, 0.2, 0.2])
        # the -axis half walks downwards from the plane
        out = oracle.casting_project([0.7, 0.2, 0.5], dims, axis, 3)
        assert np.array_equal(out, [0.2, 0.2, 0.5])
    # two halves, plane at layer 2: [.3 .9 | .8 .1 .4] -> [.3 .9 | .8 .1 .1]
    out = oracle.casting_project([0.3, 0.9, 0.8, 0.1, 0.4], (5, 1, 1), 0, 2)
    assert np.array_equal(out, [0.3, 0.9, 0.8, 0.1, 0.1])
    rng = np.random.default_rng(0)
    dims = (7, 5, 6)
    f = rng.standard_normal(7 * 5 * 6)
    for axis in range(3):
        for parting in (0, 2, dims[axis]):
            p1 = oracle.casting_project(f, dims, axis, parting)
            assert np.array_equal(oracle.casting_project(p1, dims, axis, parting), p1)  # idempotent
            assert np.all(p1 <= f)
            design = np.ones(f.size, dtype=bool)
            for vf in rng.random(20):
                occ, _, _ = oracle.extract(p1, design, max(vf, 0.02), 1e-3, all_ties=True)
                assert oracle.undercut_violations(occ, dims, axis, parting) == 0
    # monotone columns are unchanged
    mono = np.repeat(np.arange(6, 0, -1, dtype=float), 35).reshape(6, 5, 7).reshape(-1)
    assert np.array_equal(oracle.casting_project(mono, dims, 2, 0), mono)


def test_geometric_tensor_and_nodal_block8_vs_reference(oracle):
    """The oracle's geometric_tensor / apply_nodal_block8 restatements against
    the REAL reference (tests/golden/make_golden_geo.py)."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden_geo.npz"))
    assert np.abs(oracle.geometric_tensor(1.0) - g["A_h1"]).max() <= 1e-15
    assert np.abs(oracle.geometric_tensor(0.5) - g["A_h05"]).max() <= 1e-15 * np.abs(g["A_h05"]).max()
    for name in ("g543", "g217"):
        dims, h = tuple(int(v) for v in g[f"{name}_dims"]), float(g[f"{name}_h"])
        op = oracle.Operator(*dims, h, g[f"{name}_occ"])
        _, st, _ = oracle.batch_element_state(op, g[f"{name}_w"])
        assert np.abs(st - g[f"{name}_stress"]).max() <= 1e-14 * np.abs(st).max()
        kg = oracle.apply_nodal_block8(op, g[f"{name}_u"], oracle.stress_blocks(g[f"{name}_stress"], h))
        assert np.abs(kg - g[f"{name}_KGu"]).max() <= 1e-13 * np.abs(g[f"{name}_KGu"]).max()
        bu = oracle.apply_nodal_block8(op, g[f"{name}_u"], g[f"{name}_blocks"])
        assert np.abs(bu - g[f"{name}_Bu"]).max() <= 1e-13 * np.abs(g[f"{name}_Bu"]).max()


def test_spec_eigen_kats(oracle):
    """SPEC.md:226-227, 245-247, 324-335 on the dense oracle."""
    # free-free single element: six rigid modes, |lambda| / lambda_7 <= 1e-6
    op = oracle.Operator(1, 1, 1, 1.0, np.ones(1))
    w, _ = oracle.dense_modal(op, 1.0, 7)
    assert np.all(np.abs(w[:6]) <= 1e-6 * w[6])
    # density scaling rho -> c rho scales eigenvalues by 1/c
    op = oracle.Operator(4, 2, 2, 1.0, np.ones(16), dirichlet=np.arange(3 * 15))
    w1, _ = oracle.dense_modal(op, 1.0, 3)
    w4, _ = oracle.dense_modal(op, 4.0, 3)
    assert np.allclose(w4, w1 / 4.0, rtol=1e-12)
    # T_lambda direct substitution and rigid mode -> 0
    u = np.tile([0.3, -0.2, 0.5], op.n_dofs // 3)
    assert np.abs(oracle.eigen_sensitivity(op, u, 0.0, 1.0)).max() <= 1e-15
    # T_p sums to u^T (K - lambda K_sigma) u and vanishes at a buckling pair
    col = oracle.Operator(2, 2, 8, 1.0, np.ones(32), dirichlet=np.arange(27))
    f = np.zeros(col.n_dofs)
    top = [3 * (x + 3 * (y + 3 * 8)) + 2 for x in range(3) for y in range(3)]
    f[top] = -1.0 / 9
    import scipy.linalg

    Kf = oracle.dense_stiffness(col)[np.ix_(col.free, col.free)]
    uref = np.zeros(col.n_dofs)
    uref[col.free] = scipy.linalg.solve(Kf, f[col.free])
    sn, st, _ = oracle.batch_element_state(col, uref)
    cap = oracle.buckling_cap(sn)
    lam, U = oracle.dense_buckling(col, st, 1, cap)
    tp = oracle.buckling_sensitivity(col, st, U[:, 0], lam[0])
    ktot = U[:, 0] @ oracle.dense_stiffness(col) @ U[:, 0]
    assert abs(tp.sum()) <= 1e-8 * ktot
    # halving the load doubles P; tension has no positive factor
    lam2, _ = oracle.dense_buckling(col, 0.5 * st, 1, oracle.buckling_cap(0.5 * sn))
    assert lam2[0] == pytest.approx(2 * lam[0], rel=1e-10)
    # pure tension: only local factors far beyond the search cap (27.8 vs cap ~ 0.3)
    lamt, _ = oracle.dense_buckling(col, -st, 1, cap)
    assert lamt.size == 0
    # Euler: P within 15 % of pi^2 E I / (4 L^2) / F on the 2x2x8 column
    assert lam[0] == pytest.approx(np.pi ** 2 * (2 ** 4 / 12) / (4 * 64), rel=0.15)
