"""Multi-RHS batching on the device: fea.solve_static_batch
solves several load vectors against one operator / deflation space. Each RHS
must be BITWISE the single-RHS solve (same kernels, same per-column coarse
arithmetic), keep its own iteration count, and match the oracle like
solve_static does (1e-10 relative at tol 1e-12)."""

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

    return tv


def _problem(tv, dims, p_solid, seed):
    from paper_2203_15115_b200 import fea

    nx, ny, nz = dims
    d, case, fixed, f = cantilever(nx, ny, nz, (nx, 0, 0), (nx, ny, nz))
    occ = np.where(np.random.default_rng(seed).random(d.n_elems) < p_solid, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    return d, fixed, f, occ, op


def _forces(d, fixed, f, m, seed):
    rng = np.random.default_rng(seed)
    out = [f]
    for _ in range(m - 1):
        g = rng.standard_normal(d.n_dofs)
        g[fixed] = 0.0
        out.append(g)
    return out


@pytest.mark.parametrize("coarse,b,m", [("dense", 3, 2), ("nd", 3, 3), ("nd", 2, 5), ("dense", 2, 9)])
def test_batch_bitwise_equals_single(tv, coarse, b, m):
    import torch

    from paper_2203_15115_b200 import fea

    d, fixed, f, occ, op = _problem(tv, (24, 12, 12), 0.9, 3)
    defl = fea.build_deflation(d, op.topology, fixed, b, coarse=coarse)
    F = [torch.from_numpy(v).cuda() for v in _forces(d, fixed, f, m, 11)]
    batch = fea.solve_static_batch(op, F, tol=1e-10, deflation=defl)
    assert len(batch) == m
    for c in range(m):
        single = fea.solve_static(op, F[c], tol=1e-10, deflation=defl)
        assert batch[c].iterations == single.iterations
        assert batch[c].residual == single.residual
        assert torch.equal(batch[c].u, single.u), c


def test_batch_plain_pcg_and_zero_rhs(tv):
    import torch

    from paper_2203_15115_b200 import fea

    d, fixed, f, occ, op = _problem(tv, (12, 6, 6), 0.85, 5)
    F = _forces(d, fixed, f, 3, 2)
    F.insert(1, np.zeros(d.n_dofs))
    batch = fea.solve_static_batch(op, np.stack(F), tol=1e-10)
    assert batch[1].iterations == 0 and np.all(batch[1].u == 0)
    for c in (0, 2, 3):
        single = fea.solve_static(op, F[c], tol=1e-10)
        assert batch[c].iterations == single.iterations
        assert np.array_equal(batch[c].u, single.u)
    # deflated with the zero RHS in the middle of the coarse column range
    defl = fea.build_deflation(d, op.topology, fixed, 3, coarse="nd")
    Fd = [torch.from_numpy(v).cuda() for v in F]
    bd = fea.solve_static_batch(op, Fd, tol=1e-10, deflation=defl)
    assert bd[1].iterations == 0 and not bool(bd[1].u.any())
    for c in (0, 2, 3):
        assert torch.equal(bd[c].u, fea.solve_static(op, Fd[c], tol=1e-10, deflation=defl).u)


def test_batch_vs_oracle(tv, oracle):
    """Every column against the CPU restatement of the reference DPCG."""
    from paper_2203_15115_b200 import fea

    d, fixed, f, occ, op = _problem(tv, (24, 12, 12), 0.9, 3)
    defl = fea.build_deflation(d, op.topology, fixed, 3, coarse="nd")
    F = _forces(d, fixed, f, 2, 21)
    batch = fea.solve_static_batch(op, F, tol=1e-12, deflation=defl)
    ref = oracle.Operator(24, 12, 12, 1.0, occ, dirichlet=fixed)
    od = oracle.Deflation(ref, 3)
    for c in range(2):
        uo, ito, _ = oracle.solve_static(ref, F[c], tol=1e-12, deflation=od)
        assert abs(batch[c].iterations - ito) <= 2
        assert rel(batch[c].u, uo) < 1e-10


def test_batch_errors(tv):
    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import DimensionMismatch, NoConvergence

    d, fixed, f, occ, op = _problem(tv, (12, 6, 6), 0.85, 5)
    assert fea.solve_static_batch(op, []) == []
    with pytest.raises(DimensionMismatch):
        fea.solve_static_batch(op, [f, np.ones(7)])
    with pytest.raises(DimensionMismatch):
        fea.solve_static_batch(op, np.ones(d.n_dofs))
    bad = f.copy()
    bad[3] = np.inf
    with pytest.raises(ValueError):
        fea.solve_static_batch(op, [f, bad])
    # the easy RHS converges, the other hits the cap: NoConvergence names it
    with pytest.raises(NoConvergence) as ei:
        fea.solve_static_batch(op, [np.zeros(d.n_dofs), f], tol=1e-12, max_iters=4)
    assert "right-hand side 1" in str(ei.value) and ei.value.residual > 1e-12


def test_batch_c4_two_load_cases(tv):
    """C4 geometry, both load cases of BASELINE configs[3] in one batch:
    bitwise equal to the two single solves (full-size race guard)."""
    import torch

    from paper_2203_15115_b200 import fea

    dims = (160, 80, 80)
    d, case, fixed, f1 = cantilever(*dims, (160, 39, 39), (160, 41, 41))
    case2 = tv.LoadCase("c2", dirichlet=case.dirichlet,
                        loads=((tv.RegionSelector("box", min=(160, 39, 39), max=(160, 41, 41)), (0, -1, 0),
                                "total"),))
    f2 = tv.assemble_force(d, case2)
    occ = np.where(np.random.default_rng(7).random(d.n_elems) < 0.9, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    defl = fea.build_deflation(d, op.topology, fixed, 8)
    F = [torch.from_numpy(v).cuda() for v in (f1, f2)]
    batch = fea.solve_static_batch(op, F, tol=1e-8, deflation=defl)
    for c in range(2):
        single = fea.solve_static(op, F[c], tol=1e-8, deflation=defl)
        assert batch[c].iterations == single.iterations
        assert torch.equal(batch[c].u, single.u)


@pytest.mark.parametrize("flow", ["1", "0"])
def test_batch_nd_tree_schedules(tv, flow, monkeypatch):
    """Multi-column coarse solve through a real bottom tree (small dense top),
    with the persistent dataflow kernel (flow = 1, used from 48k coarse DOFs
    at full size) and with the per-level launches + packed top tiles: every
    column bitwise equals its single solve, and the ND solution matches the
    dense coarse inverse's."""
    import torch

    import paper_2203_15115_b200.coarse as C
    from paper_2203_15115_b200 import fea

    monkeypatch.setattr(C, "FLOW", flow)
    monkeypatch.setattr(C, "TOP_MAX", 200)
    monkeypatch.setattr(C, "LEAF_MAX", 8)
    d, fixed, f, occ, op = _problem(tv, (32, 16, 16), 0.9, 9)
    defl = fea.build_deflation(d, op.topology, fixed, 4, coarse="nd")
    defl.prepare(op)
    assert defl.nd.H0 >= 1 and defl.nd.n_top > 0
    assert (defl.nd.top_tiles > 0) == (flow == "0")
    F = [torch.from_numpy(v).cuda() for v in _forces(d, fixed, f, 3, 5)]
    batch = fea.solve_static_batch(op, F, tol=1e-12, deflation=defl)
    for c in range(3):
        single = fea.solve_static(op, F[c], tol=1e-12, deflation=defl)
        assert batch[c].iterations == single.iterations
        assert torch.equal(batch[c].u, single.u)
    dense = fea.build_deflation(d, op.topology, fixed, 4, coarse="dense")
    rd = fea.solve_static(op, F[0], tol=1e-12, deflation=dense)
    assert abs(rd.iterations - batch[0].iterations) <= 1
    assert rel(batch[0].u.cpu().numpy(), rd.u.cpu().numpy()) < 1e-10
