"""Eigen / buckling (SPEC eigen_buckling, SPEC.md:201-266,
fields SPEC.md:319-336) on the device.

* the geometric-stiffness kernel against the REAL reference's
  apply_nodal_block8 / geometric_tensor (tests/golden/reference_golden_geo.npz)
  and a dense assembly (1e-9);
* solve_modal / solve_buckling against dense scipy eigensolutions of the
  oracle's assembled operators, plus the SPEC's examples (rigid modes, density
  scaling, clamped-bar axial frequency, Euler column, pure tension, load
  scaling);
* T_lambda / T_p against the oracle's restatement (1e-8 relative).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden_geo.npz")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(scope="module")
def tv():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2203_15115_b200 import _build

    _build.build()
    import paper_2203_15115_b200 as tv

    return tv


def _op(tv, dims, occ, fixed=(), h=1.0, rho=1.0):
    from paper_2203_15115_b200 import fea

    d = tv.Domain(*dims, h)
    return fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3, rho=rho), fixed)


def test_nodal_block8_seam_golden(tv):
    import torch

    from paper_2203_15115_b200 import backends, eigen
    from paper_2203_15115_b200.elements import geometric_tensor

    g = np.load(GOLD)
    assert rel(geometric_tensor(1.0), g["A_h1"]) <= 1e-15
    for name in ("g543", "g217"):
        dims, h = tuple(int(v) for v in g[f"{name}_dims"]), float(g[f"{name}_h"])
        d = tv.Domain(*dims, h)
        out = np.zeros(d.n_dofs)
        backends.apply_nodal_block8(g[f"{name}_u"], out, d.elem_dofs, g[f"{name}_blocks"])
        assert rel(out, g[f"{name}_Bu"]) <= 1e-12
        op = _op(tv, dims, g[f"{name}_occ"], h=h)
        geo = eigen.GeometricStiffnessOperator(op, torch.from_numpy(g[f"{name}_stress"]).cuda())
        kg = -geo.apply(g[f"{name}_u"], raw=True)  # K_sigma = -K_G
        assert rel(kg, g[f"{name}_KGu"]) <= 1e-12
        # the stresses of the reference state through geometric_stiffness()
        geo2 = eigen.geometric_stiffness(g[f"{name}_w"], op)
        assert rel(-geo2.apply(g[f"{name}_u"], raw=True), g[f"{name}_KGu"]) <= 1e-11


def test_geometric_stiffness_dense_zero_linear(tv, oracle):
    import torch

    from paper_2203_15115_b200 import eigen

    rng = np.random.default_rng(3)
    occ = np.array([1.0, 1e-3])
    op = _op(tv, (2, 1, 1), occ)
    w = rng.standard_normal(op.n_dofs)
    geo = eigen.geometric_stiffness(w, op)
    ref = oracle.Operator(2, 1, 1, 1.0, occ)
    _, st, _ = oracle.batch_element_state(ref, w)
    Kd = -oracle.dense_geometric(ref, st)
    v = rng.standard_normal(op.n_dofs)
    assert rel(geo.apply(v), Kd @ v) <= 1e-9
    zero = eigen.GeometricStiffnessOperator(op, torch.zeros((2, 6), dtype=torch.float64, device="cuda"))
    assert not np.any(zero.apply(v))
    geo2 = eigen.geometric_stiffness(2.0 * w, op)
    assert np.array_equal(geo2.apply(v), 2.0 * geo.apply(v))  # doubling f_ref doubles the action exactly


def test_lumped_mass(tv, oracle):
    from paper_2203_15115_b200 import eigen

    occ = np.where(np.random.default_rng(1).random(5 * 4 * 3) < 0.6, 1.0, 1e-3)
    op = _op(tv, (5, 4, 3), occ, h=0.5, rho=7.5)
    m = eigen.MassOperator(op)
    ref = oracle.lumped_mass(oracle.Operator(5, 4, 3, 0.5, occ), 7.5)
    assert rel(m.diagonal(), ref) <= 1e-14
    assert m.total == pytest.approx(7.5 * 0.125 * occ.sum(), rel=1e-13)
    assert np.all(m.diagonal() >= 0.0)


def test_modal_free_free_element(tv):
    from paper_2203_15115_b200 import eigen

    op = _op(tv, (1, 1, 1), np.ones(1))
    r = eigen.solve_modal(op, eigen.MassOperator(op), k=7, tol=1e-8)
    lam = np.array(r.values)
    assert np.all(np.abs(lam[:6]) <= 1e-6 * lam[6])


def test_modal_vs_dense_oracle(tv, oracle):
    import torch

    from paper_2203_15115_b200 import eigen, fea

    from conftest import cantilever

    dims = (6, 3, 3)
    occ = np.where(np.random.default_rng(2).random(54) < 0.8, 1.0, 1e-3)
    d, case, fixed, f = cantilever(*dims, (6, 0, 0), (6, 3, 3))
    op = _op(tv, dims, occ, fixed)
    mass = eigen.MassOperator(op)
    defl = fea.build_deflation(d, op.topology, fixed, 3)
    r = eigen.solve_modal(op, mass, k=3, tol=1e-8, deflation=defl)
    ref = oracle.Operator(*dims, 1.0, occ, dirichlet=fixed)
    w, U = oracle.dense_modal(ref, 1.0, 3)
    assert np.allclose(r.values, w, rtol=1e-9)
    assert all(x <= 1e-8 for x in r.residuals)
    X = torch.stack(r.vectors, 1)
    G = (X.T @ (mass.diag_d[:, None] * X)).cpu().numpy()
    assert np.abs(G - np.eye(3)).max() <= 1e-6  # M-orthonormal
    assert r.values[0] >= -1e-9 * r.values[-1]
    # density scaling: rho -> 4 rho scales every eigenvalue by 1/4
    op4 = _op(tv, dims, occ, fixed, rho=4.0)
    r4 = eigen.solve_modal(op4, eigen.MassOperator(op4), k=3, tol=1e-8, deflation=defl)
    assert np.allclose(np.array(r4.values) * 4.0, r.values, rtol=1e-9)
    # T_lambda of the first mode vs the oracle
    t = eigen.eigen_sensitivity(op, r.vectors[0], r.values[0]).cpu().numpy()
    to = oracle.eigen_sensitivity(ref, r.vectors[0].cpu().numpy(), r.values[0], 1.0)
    assert rel(t, to) <= 1e-8


def test_modal_clamped_bar_axial_frequency(tv):
    """20x2x2 clamped-free bar, axial fundamental within 10 % of
    (pi / 2L) sqrt(E / rho)."""
    from paper_2203_15115_b200 import eigen, fea

    from conftest import cantilever

    d, case, fixed, f = cantilever(20, 2, 2, (20, 1, 1), (20, 1, 1))
    op = _op(tv, (20, 2, 2), np.ones(80), fixed)
    r = eigen.solve_modal(op, eigen.MassOperator(op), k=6, tol=1e-8,
                          deflation=fea.build_deflation(d, op.topology, fixed, 2))
    axial = []
    for lam, v in zip(r.values, r.vectors):
        u = v.view(-1, 3).cpu().numpy()
        axial.append((np.sum(u[:, 0] ** 2) / np.sum(u ** 2), lam))
    frac, lam = max(axial)
    assert frac > 0.9
    assert np.sqrt(lam) == pytest.approx(np.pi / 40.0, rel=0.10)


def _column(tv, n=2, L=8, sign=-1.0, E=1.0):
    from paper_2203_15115_b200 import fea

    d = tv.Domain(n, n, L, 1.0)
    case = tv.LoadCase("col", dirichlet=((tv.RegionSelector("box", min=(0, 0, 0), max=(n, n, 0)), (1, 1, 1)),),
                       loads=((tv.RegionSelector("box", min=(0, 0, L), max=(n, n, L)), (0, 0, sign), "total"),))
    fixed = tv.dirichlet_dofs(d, case)
    f = tv.assemble_force(d, case)
    op = fea.StiffnessOperator(d, tv.Topology(d, np.ones(d.n_elems)), tv.Material(E=E, nu=0.3), fixed)
    return d, op, fixed, f


def test_buckling_vs_dense_and_spec(tv, oracle):
    from paper_2203_15115_b200 import eigen, fea

    d, op, fixed, f = _column(tv)
    u = fea.solve_static(op, f, tol=1e-12).u
    geo = eigen.geometric_stiffness(u, op)
    r = eigen.solve_buckling(op, geo, k=1, tol=1e-8)
    ref = oracle.Operator(2, 2, 8, 1.0, np.ones(32), dirichlet=fixed)
    sn, st, _ = oracle.batch_element_state(ref, u)
    lam, U = oracle.dense_buckling(ref, st, 1, oracle.buckling_cap(sn))
    assert r.values[0] == pytest.approx(lam[0], rel=1e-9)
    phi = r.vectors[0].cpu().numpy()
    assert np.abs(phi.reshape(-1, 3)).max() <= 1.0 + 1e-12
    assert np.linalg.norm(phi.reshape(-1, 3), axis=1).max() == pytest.approx(1.0, rel=1e-12)
    # T_p vs the oracle, and sum_e T_p = phi^T (K - lambda K_sigma) phi ~ 0
    tp = eigen.buckling_sensitivity(op, geo, phi, r.values[0])
    tpo = oracle.buckling_sensitivity(ref, st, phi, r.values[0])
    assert rel(tp, tpo) <= 1e-8
    assert abs(tp.sum()) <= 1e-6 * float(phi @ oracle.dense_stiffness(ref) @ phi)
    # Euler: pi^2 E I / (4 L^2) / F within 15 %
    assert r.values[0] == pytest.approx(np.pi ** 2 * (16 / 12) / (4 * 64), rel=0.15)
    # halving the load doubles P; E -> 3E scales P by 3
    r2 = eigen.solve_buckling(op, eigen.geometric_stiffness(0.5 * u, op), k=1, tol=1e-8)
    assert r2.values[0] == pytest.approx(2.0 * r.values[0], rel=1e-7)
    d3, op3, _, f3 = _column(tv, E=3.0)
    u3 = fea.solve_static(op3, f3, tol=1e-12).u
    r3 = eigen.solve_buckling(op3, eigen.geometric_stiffness(u3, op3), k=1, tol=1e-8)
    assert r3.values[0] == pytest.approx(3.0 * r.values[0], rel=1e-7)


def test_buckling_tension_and_zero_stress(tv):
    import torch

    from paper_2203_15115_b200 import eigen, fea

    d, op, fixed, f = _column(tv, sign=+1.0)
    u = fea.solve_static(op, f, tol=1e-12).u
    r = eigen.solve_buckling(op, eigen.geometric_stiffness(u, op), k=1)
    assert r.no_positive_factor and r.values == [np.inf]
    z = eigen.GeometricStiffnessOperator(op, torch.zeros((d.n_elems, 6), dtype=torch.float64, device="cuda"))
    assert eigen.solve_buckling(op, z).no_positive_factor


def test_euler_column_deflated_4x4x40(tv):
    """SPEC.md:245 exactly as written: 4x4x40 column (h = 1) clamped at the
    base, axial compressive tip load, deflated inner solves (b = 4)."""
    from paper_2203_15115_b200 import eigen, fea

    d, op, fixed, f = _column(tv, n=4, L=40)
    defl = fea.build_deflation(d, op.topology, fixed, 4)
    u = fea.solve_static(op, f, tol=1e-12, deflation=defl).u
    r = eigen.solve_buckling(op, eigen.geometric_stiffness(u, op), k=1, tol=1e-6, deflation=defl)
    assert r.values[0] == pytest.approx(np.pi ** 2 * (256 / 12) / (4 * 1600), rel=0.15)
