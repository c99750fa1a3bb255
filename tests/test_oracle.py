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
