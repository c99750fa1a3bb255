"""K6 on the device (csrc/dense.cu): the nested-dissection front factorisation
and the dense small-space inverse, against numpy on the same E
(reference: scipy.linalg.cho_factor of the symmetrised E, topovox/fea.py:197-205)."""

import numpy as np
import pytest

from test_coarse_nd import dense_of, random_block_stencil


def _nd_solve(nd, y):
    import torch

    ndi = nd.nd_index()
    yn = np.empty_like(y)
    yn[ndi] = y
    xd = torch.empty(y.size, dtype=torch.float64, device="cuda")
    nd.solve_device(torch.from_numpy(yn).cuda(), xd)
    return xd.cpu().numpy()[ndi]


@pytest.mark.gpu
@pytest.mark.parametrize("grid,leaf,top_max", [((5, 5, 10), 27, 0), ((5, 5, 10), 27, 60), ((9, 8, 7), 8, 600),
                                               ((4, 3, 2), 2, 4608), ((7, 1, 3), 4, 60), ((12, 10, 9), 27, 2000)])
def test_device_front_factor_matches_dense(grid, leaf, top_max):
    import torch

    from paper_2203_15115_b200.coarse import NDCoarseSolver

    mx, my, mz = grid
    Es = random_block_stencil(mx, my, mz, seed=sum(grid) + leaf)
    E = dense_of(Es, mx, my, mz)
    nd = NDCoarseSolver(grid, torch.from_numpy(Es.reshape(-1)).cuda(), leaf_max=leaf, top_max=top_max)
    y = np.random.default_rng(2).standard_normal(E.shape[0])
    x = _nd_solve(nd, y)
    ref = np.linalg.solve(E, y)
    err = np.abs(x - ref).max() / np.abs(ref).max()
    print(f"[front factor] grid {grid} leaf {leaf} top {top_max}: H0 {nd.H0}, top {nd.n_top}, rel {err:.1e}")
    assert err <= 1e-12


@pytest.mark.gpu
def test_device_dense_inverse_and_spd_check():
    import torch

    from paper_2203_15115_b200.coarse import dense_inverse

    grid = (6, 5, 4)
    Es = random_block_stencil(*grid, seed=9)
    E = dense_of(Es, *grid)
    Zi = dense_inverse(grid, torch.from_numpy(Es.reshape(-1)).cuda()).cpu().numpy()
    ref = np.linalg.inv(E)
    assert np.abs(Zi - ref).max() <= 1e-12 * np.abs(ref).max()
    # symmetrisation 0.5 (E + E^T) (fea.py:198): a perturbed, non-symmetric stencil
    Ep = Es.copy()
    Ep[:, 13] += 1e-3 * np.random.default_rng(1).standard_normal(Ep[:, 13].shape)
    Zp = dense_inverse(grid, torch.from_numpy(Ep.reshape(-1)).cuda()).cpu().numpy()
    Ed = dense_of(Ep, *grid)
    assert np.abs(Zp - np.linalg.inv(0.5 * (Ed + Ed.T))).max() <= 1e-12 * np.abs(ref).max()
    with pytest.raises(np.linalg.LinAlgError):
        dense_inverse(grid, torch.from_numpy(-Es.reshape(-1)).cuda())


@pytest.mark.gpu
def test_deflation_dense_and_nd_on_real_operator():
    """A real E (24x12x12 Bernoulli(0.9) cantilever, b = 3): the device dense
    inverse and the device ND factor both match numpy's inverse of the
    symmetrised E (from the coarse-assembly kernel)."""
    import torch

    import paper_2203_15115_b200 as tv
    from paper_2203_15115_b200 import _lib, fea
    from paper_2203_15115_b200._lib import ptr, stream_ptr
    from conftest import cantilever

    occ = np.where(np.random.default_rng(3).random(24 * 12 * 12) < 0.9, 1.0, 1e-3)
    d, case, fixed, f = cantilever(24, 12, 12, (24, 0, 0), (24, 12, 12))
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    dn = fea.build_deflation(d, op.topology, fixed, 3, coarse="dense")
    dn.prepare(op)
    nc = 6 * dn.n_blocks
    E = torch.empty(nc * nc, dtype=torch.float64, device="cuda")
    _lib.lib().tvb_coarse_dense(d.nx, d.ny, d.nz, 3, ptr(dn.Es), ptr(E), stream_ptr())
    E = E.view(nc, nc).cpu().numpy()  # dropped (rank-deficient) modes carry a unit diagonal
    ref = np.linalg.inv(0.5 * (E + E.T))
    got = dn.coarse_inv.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()
    nd = fea.build_deflation(d, op.topology, fixed, 3, coarse="nd")
    nd.prepare(op)
    y = np.random.default_rng(4).standard_normal(nd.n_vectors)
    assert np.abs(nd.coarse_solve(y) - dn.coarse_solve(y)).max() <= 1e-10 * np.abs(dn.coarse_solve(y)).max()
