"""Casting constraint (PAPER §3.7) on the
device: tvb_casting_project against the oracle's running-minimum restatement
(bitwise: the projection only copies values), extraction of a projected field
with all threshold ties retained (identical masks), the exhaustive undercut
audit, and a casting-constrained optimizer run against the oracle's."""

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


AXES = ["+x", "-x", "+y", "-y", "+z", "-z"]


@pytest.mark.parametrize("dims", [(13, 7, 9), (1, 1, 5), (40, 20, 20)])
def test_casting_project_matches_oracle(tv, oracle, dims):
    import torch

    from paper_2203_15115_b200 import levelset

    d = tv.Domain(*dims, 1.0)
    f = np.random.default_rng(1).standard_normal(d.n_elems)
    for ax in AXES:
        a = "xyz".index(ax[1])
        for plane in (None, 0, dims[a] // 2, dims[a]):
            spec = levelset.CastingSpec(ax, plane)
            axis, parting = spec.resolve(d)
            got = levelset.casting_project(d, f, spec)
            ref = oracle.casting_project(f, dims, axis, parting)
            assert np.array_equal(got, ref), (ax, plane)
            # in place on the device, idempotent
            t = torch.from_numpy(f.copy()).cuda()
            levelset.casting_project_device(d, t, spec, out_d=t)
            assert np.array_equal(t.cpu().numpy(), ref)
            assert np.array_equal(levelset.casting_project(d, ref, spec), ref)


def test_casting_spec_validation(tv):
    from paper_2203_15115_b200 import levelset

    d = tv.Domain(4, 3, 2, 1.0)
    with pytest.raises(ValueError):
        levelset.CastingSpec("x")
    with pytest.raises(ValueError):
        levelset.CastingSpec("+w")
    with pytest.raises(ValueError):
        levelset.CastingSpec("+z", 3).resolve(d)
    assert levelset.CastingSpec("-y").resolve(d) == (1, 3)
    assert levelset.CastingSpec("+y").resolve(d) == (1, 0)


def test_casting_extract_matches_oracle_and_audit(tv, oracle):
    from paper_2203_15115_b200 import levelset

    dims = (16, 9, 11)
    d = tv.Domain(*dims, 1.0)
    rng = np.random.default_rng(2)
    f = np.round(rng.standard_normal(d.n_elems) * 4) / 4  # many ties
    for ax, plane in (("+z", 5), ("-x", None), ("+y", 0)):
        spec = levelset.CastingSpec(ax, plane)
        axis, parting = spec.resolve(d)
        pf = oracle.casting_project(f, dims, axis, parting)
        for vf in list(rng.random(20)) + [1.0]:
            vf = max(float(vf), 0.01)
            topo = levelset.extract(d, f, vf, ersatz=1e-3, casting=spec)
            occ_ref, _, k = oracle.extract(pf, d.design_mask, vf, 1e-3, all_ties=True)
            assert np.array_equal(topo.occupancy, occ_ref), (ax, vf)
            assert np.count_nonzero(topo.occupancy == 1.0) >= k
            assert oracle.undercut_violations(topo.occupancy, dims, axis, parting) == 0


def test_casting_optimizer_run(tv, oracle):
    """Compliance-constrained 12x6x6 cantilever cast along z with the parting
    plane at mid-height: every accepted topology is undercut-free and the run
    follows the oracle's casting run (same stop reason, step count within 2)."""
    from paper_2203_15115_b200 import levelset
    from paper_2203_15115_b200 import optimize as opt

    prob = opt.cantilever_problem(12, 6, 6, (12, 3, 3), (12, 3, 3),
                                  constraints=[opt.ConstraintSpec("compliance", 1.6)])
    prob.casting = levelset.CastingSpec("+z", 3)
    cfg = opt.OptimizerConfig(ersatz=1e-3, block=3, max_outer=12)
    seen = []
    topo, hist, reason = opt.run(prob, cfg, callback=lambda rec: seen.append(rec))
    assert oracle.undercut_violations(topo.occupancy, (12, 6, 6), 2, 3) == 0
    d, case, fixed, f = cantilever(12, 6, 6, (12, 3, 3), (12, 3, 3))
    occ_r, hist_r, reason_r = oracle.run_optimizer(12, 6, 6, [(fixed, f)],
                                                   [{"kind": "compliance", "alpha": 1.6, "case": 0}],
                                                   block=3, ersatz=1e-3, max_outer=12, casting=(2, 3))
    assert reason == reason_r
    assert oracle.undercut_violations(occ_r, (12, 6, 6), 2, 3) == 0
    acc = [h.v for h in hist if h.accepted]
    acc_r = [h["v"] for h in hist_r if h["accepted"]]
    assert abs(len(acc) - len(acc_r)) <= 2
