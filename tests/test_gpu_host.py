"""Host-buffer matvec entry points (the e2e path): tvb_matvec_host and the
double-buffered stream tvb_matvec_host_batch must return exactly the device
K.u (same kernel, same slab split) for numpy and pinned-tensor buffers, with
and without Dirichlet masking."""

import numpy as np
import pytest

from conftest import cantilever

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tv():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2203_15115_b200 import _build

    _build.build()
    import paper_2203_15115_b200 as tv

    return tv


@pytest.mark.parametrize("dims,slabs", [((16, 9, 11), 0), ((13, 5, 40), 7), ((4, 4, 4), 64)])
def test_host_batch_bitwise(tv, dims, slabs):
    import torch

    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import DimensionMismatch

    d, case, fixed, f = cantilever(*dims, (dims[0], 0, 0), (dims[0], dims[1], dims[2]))
    occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
    op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
    rng = np.random.default_rng(1)
    us = [rng.standard_normal(d.n_dofs) for _ in range(5)]
    ref = [op.apply_device(torch.from_numpy(u).cuda()).cpu().numpy() for u in us]
    out = op.apply_host_batch(us, slabs=slabs)
    for a, b in zip(out, ref):
        assert np.array_equal(a, b)
    raw = op.apply_host_batch(us[:3], raw=True, slabs=slabs)
    for u, a in zip(us, raw):
        assert np.array_equal(a, op.apply_device(torch.from_numpy(u).cuda(), raw=True).cpu().numpy())
    # pinned tensors, one input streamed several times into one output (the bench pattern)
    up = torch.from_numpy(us[0]).pin_memory()
    yp = torch.empty(d.n_dofs, dtype=torch.float64).pin_memory()
    op.apply_host_batch([up] * 4, [yp] * 4, slabs=slabs)
    assert np.array_equal(yp.numpy(), ref[0])
    assert np.array_equal(op.apply_host(us[1]), ref[1])
    assert op.apply_host_batch([]) == []
    with pytest.raises(DimensionMismatch):
        op.apply_host_batch(us[:2], [np.empty(d.n_dofs)])
    with pytest.raises(DimensionMismatch):
        op.apply_host_batch([np.ones(7)])
