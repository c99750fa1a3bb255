"""CUDA path vs the oracle / the reference's golden vectors (needs a B200).

Tolerances (BASELINE.json north_star): matvec and PCG solutions within 1e-10
relative in fp64 (solutions compared at tol 1e-12, where the reference's own
backends agree to ~4e-13), compliance and sensitivities within
1e-8 relative, extracted masks identical (exact selection on identical input).
"""

import numpy as np
import pytest

from conftest import cantilever

pytestmark = pytest.mark.gpu


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
    from paper_2203_15115_b200 import fea, levelset, sensitivity  # noqa: F401

    return tv


def make_op(tv, dims, occ, fixed, E=1.0, nu=0.3, h=1.0):
    from paper_2203_15115_b200 import fea

    d = tv.Domain(*dims, h)
    return fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=E, nu=nu), fixed)


@pytest.mark.parametrize("name", ["mv333", "mv543", "mv171"])
def test_matvec_golden(tv, golden, name):
    dims = tuple(int(v) for v in golden[name + "_dims"])
    op = make_op(tv, dims, golden[name + "_occ"], golden[name + "_fixed"])
    u = golden[name + "_u"]
    assert rel(op.apply(u, raw=True), golden[name + "_Ku_raw"]) < 1e-13
    assert rel(op.apply(u), golden[name + "_Ku"]) < 1e-13
    assert rel(op.diagonal(), golden[name + "_diag"]) < 1e-14
    assert rel(op.apply_subset(u, golden[name + "_sub"]), golden[name + "_Ku_sub"]) < 1e-13


@pytest.mark.parametrize("name", ["mv333", "mv543"])
def test_seam_functions_golden(tv, golden, name):
    from paper_2203_15115_b200 import backends
    from paper_2203_15115_b200.elements import hex_stiffness

    dims = tuple(int(v) for v in golden[name + "_dims"])
    d = tv.Domain(*dims, 1.0)
    k0 = hex_stiffness(tv.Material(E=1.0, nu=0.3), 1.0)
    u, occ = golden[name + "_u"], golden[name + "_occ"]
    out = np.zeros(d.n_dofs)
    backends.apply_block24(u, out, d.elem_dofs, occ, k0, None, None)
    assert rel(out, golden[name + "_Ku_raw"]) < 1e-13
    out2 = np.zeros(d.n_dofs)
    backends.apply_block24_subset(u, out2, golden[name + "_sub"], d.elem_dofs, occ, k0)
    free = np.ones(d.n_dofs, dtype=bool)
    free[golden[name + "_fixed"]] = False  # the golden came through op.apply_subset (fixed rows zeroed)
    assert rel(out2[free], golden[name + "_Ku_sub"][free]) < 1e-13
    dg = np.zeros(d.n_dofs)
    backends.diag_block24(dg, d.elem_dofs, occ, np.diag(k0).copy())
    assert rel(dg, golden[name + "_diag"]) < 1e-14


@pytest.mark.parametrize("dims", [(37, 29, 23), (1, 1, 1), (64, 3, 2), (5, 70, 9), (2, 2, 150)])
def test_matvec_vs_oracle_ragged(tv, oracle, dims):
    rng = np.random.default_rng(sum(dims))
    ne = dims[0] * dims[1] * dims[2]
    occ = np.where(rng.random(ne) < 0.7, 1.0, 1e-3)
    d, case, fixed, f = cantilever(*dims, (dims[0], 0, 0), (dims[0], dims[1], dims[2]))
    op = make_op(tv, dims, occ, fixed)
    ref = oracle.Operator(*dims, 1.0, occ, dirichlet=fixed)
    u = rng.standard_normal(op.n_dofs)
    assert rel(op.apply(u, raw=True), ref.apply(u, raw=True)) < 1e-13
    assert rel(op.apply(u), ref.apply(u)) < 1e-13
    assert rel(op.diagonal(), ref.diagonal()) < 1e-14


@pytest.mark.parametrize("slabs", [0, 1, 3, 64])
def test_matvec_host_pipeline(tv, oracle, slabs):
    """Host-buffer K.u (z-slab copy/compute pipeline) == device K.u, pinned and
    pageable inputs, with and without the Dirichlet masks."""
    import torch

    dims = (33, 17, 41)
    rng = np.random.default_rng(5)
    occ = np.where(rng.random(dims[0] * dims[1] * dims[2]) < 0.7, 1.0, 1e-3)
    d, case, fixed, f = cantilever(*dims, (dims[0], 0, 0), (dims[0], dims[1], dims[2]))
    op = make_op(tv, dims, occ, fixed)
    u = rng.standard_normal(op.n_dofs)
    ud = torch.from_numpy(u).cuda()
    for raw in (False, True):
        dev = op.apply_device(ud, raw=raw).cpu().numpy()
        host = op.apply_host(u, raw=raw, slabs=slabs)
        assert rel(host, dev) < 1e-15
        pin = torch.from_numpy(u).pin_memory()
        out = torch.empty(op.n_dofs, dtype=torch.float64).pin_memory()
        op.apply_host(pin, out, raw=raw, slabs=slabs)
        assert rel(out.numpy(), dev) < 1e-15
    ref = oracle.Operator(*dims, 1.0, occ, dirichlet=fixed)
    assert rel(op.apply(u), ref.apply(u)) < 1e-13


def test_matvec_c2_full_size_properties(tv, oracle):
    """C2(a) workload (128^3, Bernoulli(0.7) seed 0, u ~ N(0,1) seed 1): vs the
    oracle at full size, plus symmetry / linearity / determinism."""
    import torch

    n = 128
    occ = np.where(np.random.default_rng(0).random(n ** 3) < 0.7, 1.0, 1e-3)
    op = make_op(tv, (n, n, n), occ, ())
    u = np.random.default_rng(1).standard_normal(op.n_dofs)
    ud = torch.from_numpy(u).cuda()
    y1 = op.apply_device(ud).clone()
    y2 = op.apply_device(ud).clone()
    assert torch.equal(y1, y2), "matvec is not bitwise deterministic"
    ref = oracle.Operator(n, n, n, 1.0, occ).apply(u)
    assert rel(y1.cpu().numpy(), ref) < 1e-12
    v = torch.from_numpy(np.random.default_rng(2).standard_normal(op.n_dofs)).cuda()
    kv = op.apply_device(v)
    assert abs(float(ud @ kv) - float(v @ y1)) <= 1e-12 * float(ud.norm() * kv.norm())
    lin = op.apply_device(2.0 * ud + v)
    assert float((lin - (2.0 * y1 + kv)).abs().max()) <= 1e-12 * float(lin.abs().max())


def test_element_state_and_fields(tv, golden, oracle):
    from paper_2203_15115_b200 import fea, sensitivity

    for name in ("mv333", "mv543", "mv171"):
        dims = tuple(int(v) for v in golden[name + "_dims"])
        op = make_op(tv, dims, golden[name + "_occ"], golden[name + "_fixed"])
        u = golden[name + "_u"]
        s, st, vm = fea.batch_element_state(op, u)
        assert rel(s, golden[name + "_strain"]) < 1e-13
        assert rel(st, golden[name + "_stress"]) < 1e-13
        assert rel(vm, golden[name + "_vm"]) < 1e-13
        ref = oracle.Operator(*dims, 1.0, golden[name + "_occ"], dirichlet=golden[name + "_fixed"])
        rs, rst, rvm = oracle.batch_element_state(ref, u)
        assert rel(sensitivity.compliance_sensitivity(op, u), oracle.compliance_sensitivity(rs, rst, 0.3)) < 1e-12
        for p in (2, 6, 8):
            assert sensitivity.pnorm_stress(op, u, p) == pytest.approx(oracle.pnorm_stress(rvm, ref.occ, p), rel=1e-12)
            assert rel(sensitivity.adjoint_rhs(op, u, p), oracle.stress_adjoint_rhs(ref, u, p)) < 1e-11
        lam = np.random.default_rng(5).standard_normal(op.n_dofs)
        ls, _, _ = oracle.batch_element_state(ref, lam)
        assert rel(sensitivity.stress_sensitivity(op, u, lam), oracle.stress_sensitivity(rst, ls, 0.3)) < 1e-12
        # self-adjoint reduction: T_sigma(u, u) == T_J(u)
        assert rel(sensitivity.stress_sensitivity(op, u, u), sensitivity.compliance_sensitivity(op, u)) < 1e-14


def test_plain_pcg_golden(tv, golden):
    from paper_2203_15115_b200 import fea

    op = make_op(tv, (8, 6, 5), golden["bern865_occ"], golden["bern865_fixed"])
    r = fea.solve_static(op, golden["bern865_f"], tol=1e-12)
    assert abs(r.iterations - int(golden["bern865_plain_t12_iters"])) <= 1
    assert rel(r.u, golden["bern865_plain_t12_u"]) < 1e-10


@pytest.mark.parametrize("coarse", ["dense", "nd"])
@pytest.mark.parametrize("b", [2, 3])
def test_dpcg_golden(tv, golden, b, coarse):
    from paper_2203_15115_b200 import fea

    op = make_op(tv, (8, 6, 5), golden["bern865_occ"], golden["bern865_fixed"])
    d = op.domain
    defl = fea.build_deflation(d, op.topology, golden["bern865_fixed"], b, coarse=coarse)
    assert defl.n_vectors == int(golden[f"bern865_b{b}_nvec"])
    for t in (8, 12):
        r = fea.solve_static(op, golden["bern865_f"], tol=10.0 ** -t, deflation=defl)
        assert abs(r.iterations - int(golden[f"bern865_b{b}_t{t}_iters"])) <= 1
        tol = 1e-10 if t == 12 else 1e-7
        assert rel(r.u, golden[f"bern865_b{b}_t{t}_u"]) < tol


@pytest.mark.parametrize("coarse", ["dense", "nd"])
def test_dpcg_c1_golden(tv, golden, coarse):
    """BASELINE configs[0]: 40x20x20 full-solid cantilever, 4^3 agglomerates."""
    from paper_2203_15115_b200 import fea

    d, case, fixed, f = cantilever(40, 20, 20, (40, 10, 10), (40, 10, 10))
    op = make_op(tv, (40, 20, 20), np.ones(d.n_elems), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, 4, coarse=coarse)
    assert defl.n_vectors == int(golden["c1_nvec"])
    r8 = fea.solve_static(op, f, tol=1e-8, deflation=defl)
    assert abs(r8.iterations - int(golden["c1_t8_iters"])) <= 1
    assert float(f @ r8.u) == pytest.approx(float(golden["c1_t8_J"]), rel=1e-10)
    r12 = fea.solve_static(op, f, tol=1e-12, deflation=defl)
    assert abs(r12.iterations - int(golden["c1_t12_iters"])) <= 1
    assert rel(r12.u, golden["c1_t12_u"]) < 1e-10
    s, st, vm = fea.batch_element_state(op, r12.u)
    assert vm.max() == pytest.approx(float(golden["c1_vm_max"]), rel=1e-8)
    rp = fea.solve_static(op, f, tol=1e-8)
    assert abs(rp.iterations - int(golden["c1_plain_t8_iters"])) <= 1


def test_dpcg_c3_c4_survey_kats(tv):
    """BASELINE configs[2] (C3, 80x40x40, b = 4) and the C4 geometry (160x80x80,
    b = 8), full solid, point load at the x = nx face centre: the reference's
    own measurements (SURVEY.md 8c KAT table / 8a a8 row): C3 J0 =
    2.4345313102 with 253 DPCG and 503 plain-PCG iterations; C4 geometry 447
    DPCG and 991 plain-PCG iterations (tol 1e-8)."""
    from paper_2203_15115_b200 import fea

    for dims, b, J0, it_d, it_p in (((80, 40, 40), 4, 2.4345313102, 253, 503), ((160, 80, 80), 8, None, 447, 991)):
        nx, ny, nz = dims
        c = (nx, ny // 2, nz // 2)
        d, case, fixed, f = cantilever(nx, ny, nz, c, c)
        op = make_op(tv, dims, np.ones(d.n_elems), fixed)
        defl = fea.build_deflation(d, op.topology, fixed, b)
        r = fea.solve_static(op, f, tol=1e-8, deflation=defl)
        assert abs(r.iterations - it_d) <= 1, (dims, r.iterations)
        if J0 is not None:
            assert float(f @ r.u) == pytest.approx(J0, rel=1e-9)  # J0 pinned to 11 digits
        rp = fea.solve_static(op, f, tol=1e-8)
        assert abs(rp.iterations - it_p) <= 1, (dims, rp.iterations)


def test_solver_edge_cases(tv, golden):
    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import DimensionMismatch, NoConvergence

    op = make_op(tv, (8, 6, 5), golden["bern865_occ"], golden["bern865_fixed"])
    r = fea.solve_static(op, np.zeros(op.n_dofs))
    assert r.iterations == 0 and np.all(r.u == 0)
    with pytest.raises(ValueError):
        fea.solve_static(op, golden["bern865_f"], tol=0.5)
    with pytest.raises(DimensionMismatch):
        fea.solve_static(op, np.ones(5))
    with pytest.raises(NoConvergence) as ei:
        fea.solve_static(op, golden["bern865_f"], tol=1e-12, max_iters=5)
    assert ei.value.iterations == 5 and ei.value.residual > 1e-12
    bad = golden["bern865_f"].copy()
    bad[7] = np.nan
    with pytest.raises(ValueError):
        fea.solve_static(op, bad)


def test_extract_and_combine_vs_oracle(tv, oracle):
    from paper_2203_15115_b200 import levelset

    rng = np.random.default_rng(11)
    d = tv.Domain(23, 17, 9, 1.0)
    vals = np.round(rng.standard_normal(d.n_elems), 2)  # many exact ties
    vals[::7] = 0.0
    vals[1::11] = -0.0
    for vf in (1.0, 0.975, 0.5, 0.3331, 1.0 / d.n_elems):
        t = levelset.extract(d, vals, vf, ersatz=1e-3)
        occ, _, k = oracle.extract(vals, d.design_mask, vf, 1e-3)
        assert np.array_equal(t.occupancy, occ), vf
        assert int((t.occupancy == 1.0).sum()) == k
    a, b = rng.standard_normal(d.n_elems), rng.standard_normal(d.n_elems) * 1e5
    got, fb = levelset.combine([a, b], [2.0, 3.0])
    ref, rfb = oracle.combine([a, b], [2.0, 3.0])
    assert not fb and rel(got, ref) < 1e-14
    got, fb = levelset.combine([a, b], [0.0, 0.0])
    assert fb and rel(got, oracle.normalize_field(a)) < 1e-15
    assert np.all(levelset.normalize_field(np.zeros(5)) == 0)


def test_extract_with_design_mask(tv, oracle):
    from paper_2203_15115_b200 import levelset

    d = tv.build_domain(10, 6, 4, 1.0, csg=[{"op": "subtract", "shape": "box", "min": (0, 0, 0), "max": (3, 3, 4)}])
    vals = np.random.default_rng(4).random(d.n_elems)
    t = levelset.extract(d, vals, 0.6, ersatz=1e-3)
    occ, _, _ = oracle.extract(vals, d.design_mask, 0.6, 1e-3)
    occ[~d.design_mask] = tv.EPS_VOID
    assert np.array_equal(t.occupancy, occ)


def test_coarse_nd_matches_dense_on_device(tv, golden, oracle):
    """The ND coarse solve equals the dense inverse on a real E (Bernoulli(0.9)
    topology; at 0.7-0.85 even the reference DPCG stalls before 1e-12)."""
    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import NoConvergence

    occ = np.where(np.random.default_rng(3).random(24 * 12 * 12) < 0.9, 1.0, 1e-3)
    d, case, fixed, f = cantilever(24, 12, 12, (24, 0, 0), (24, 12, 12))
    op = make_op(tv, (24, 12, 12), occ, fixed)
    dn = fea.build_deflation(d, op.topology, fixed, 3, coarse="dense")
    nd = fea.build_deflation(d, op.topology, fixed, 3, coarse="nd")
    dn.prepare(op)
    nd.prepare(op)
    y = np.random.default_rng(4).standard_normal(dn.n_vectors)
    a, b = dn.coarse_solve(y), nd.coarse_solve(y)
    assert rel(b, a) < 1e-11
    # dense explicit inverse vs ND factor: the reference's recurrence is
    # sensitive to the coarse solve's rounding at 1e-12 on this problem, so the
    # two coarse solvers are compared under the stabilised projection
    ra = fea.solve_static(op, f, tol=1e-12, deflation=dn, projection="stabilized")
    rb = fea.solve_static(op, f, tol=1e-12, deflation=nd, projection="stabilized")
    assert abs(ra.iterations - rb.iterations) <= 1
    assert rel(rb.u, ra.u) < 1e-10
    ref = oracle.Operator(24, 12, 12, 1.0, occ, dirichlet=fixed)
    uo, ito, _ = oracle.solve_static(ref, f, tol=1e-12, deflation=oracle.Deflation(ref, 3))
    assert abs(rb.iterations - ito) <= 2
    assert rel(rb.u, uo) < 1e-10
    # the reference's own recurrence with the ND factor: at 1e-12 on this
    # problem it depends on rounding alone whether it converges (reported)
    try:
        rr = fea.solve_static(op, f, tol=1e-12, deflation=nd, projection="reference")
        out = f"{rr.iterations} it, rel {rel(rr.u, uo):.1e}"
    except NoConvergence as exc:
        out = f"NoConvergence (residual {exc.residual:.1e})"
    print(f"[coarse nd] reference projection at 1e-12: {out} (oracle {ito} it)")


def test_projection_stabilized_converges_where_reference_drifts(tv):
    """C1 geometry with the load spread over the whole x = 40 face, tol 1e-12:
    the reference's recurrence drifts (the reference itself stops at its
    iteration cap with residual 8.8e3); projection='stabilized' converges. The
    default (reference) recurrence's outcome is reported."""
    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import NoConvergence

    d, case, fixed, f = cantilever(40, 20, 20, (40, 0, 0), (40, 20, 20))
    op = make_op(tv, (40, 20, 20), np.ones(d.n_elems), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, 4)
    r8 = fea.solve_static(op, f, tol=1e-8, deflation=defl)
    assert abs(r8.iterations - 129) <= 1  # the reference: 129 (noise_floor study)
    rs = fea.solve_static(op, f, tol=1e-12, deflation=defl, projection="stabilized")
    assert rs.iterations < 200
    try:
        rr = fea.solve_static(op, f, tol=1e-12, deflation=defl, projection="reference")
        outcome = f"converged in {rr.iterations}"
    except NoConvergence as exc:
        outcome = f"NoConvergence (residual {exc.residual:.2e} at {exc.iterations})"
    print(f"[projection] C1 face load tol 1e-12: stabilized {rs.iterations} it; reference recurrence {outcome} "
          f"(the reference: NoConvergence, residual 8.8e3 at 2329)")


@pytest.mark.parametrize("occ_kind", ["solid", "bernoulli"])
def test_dpcg_c4_size_converges(tv, occ_kind):
    """C4 geometry (160x80x80, 8^3 agglomerates, nested-dissection coarse
    solve): the full-size deflated solve converges, its recursive residual is
    honest (true residual via an independent K.u), its iteration count matches
    the reference protocol's order (457 on the full solid), and it is bitwise
    reproducible. Catches races that only show at full size."""
    import torch

    from paper_2203_15115_b200 import fea

    dims = (160, 80, 80)
    d, case, fixed, f = cantilever(*dims, (160, 39, 39), (160, 41, 41))
    n = d.n_elems
    occ = np.ones(n) if occ_kind == "solid" else np.where(np.random.default_rng(7).random(n) < 0.9, 1.0, 1e-3)
    op = make_op(tv, dims, occ, fixed)
    defl = fea.build_deflation(d, op.topology, fixed, 8)
    fd = torch.from_numpy(f).cuda()
    r1 = fea.solve_static(op, fd, tol=1e-8, deflation=defl)
    r2 = fea.solve_static(op, fd, tol=1e-8, deflation=defl)
    assert torch.equal(r1.u, r2.u) and r1.iterations == r2.iterations
    if occ_kind == "solid":
        assert abs(r1.iterations - 457) <= 2
    else:
        assert r1.iterations < 1500
    res = op.apply_device(r1.u) - fd
    free = torch.from_numpy(op.free_mask).cuda()
    true_rel = float(res[free].norm() / fd[free].norm())
    assert true_rel < 1e-7, true_rel


def test_generic_operator_path_keeps_deflation(tv, golden):
    """solve_static with apply_op / diag (the reference's hook for shifted
    solves, fea.py:218-299) still deflates with the space prepared for op, as
    the reference does: with apply_op = op's own K it reproduces the default
    device solve's iterates (same count +-1, solution 1e-10)."""
    import torch

    from paper_2203_15115_b200 import fea

    d, case, fixed, f = cantilever(24, 12, 12, (24, 0, 0), (24, 12, 12))
    occ = np.where(np.random.default_rng(3).random(d.n_elems) < 0.9, 1.0, 1e-3)
    op = make_op(tv, (24, 12, 12), occ, fixed)
    defl = fea.build_deflation(d, op.topology, fixed, 3)
    fd = torch.from_numpy(f).cuda()
    r0 = fea.solve_static(op, fd, tol=1e-10, deflation=defl, projection="reference")
    rg = fea.solve_static(op, fd, tol=1e-10, deflation=defl, apply_op=op.apply_device)
    rp = fea.solve_static(op, fd, tol=1e-10, apply_op=op.apply_device)
    assert abs(rg.iterations - r0.iterations) <= 1, (rg.iterations, r0.iterations)
    assert rel(rg.u.cpu().numpy(), r0.u.cpu().numpy()) < 1e-9
    assert rp.iterations > rg.iterations  # without the space: plain Jacobi PCG
