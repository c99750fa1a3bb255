"""Solution-level DPCG parity at the BASELINE configurations (C3, C4 with both
3x3-patch load cases, full solid and Bernoulli(0.9), C5, C2(b)) against
fixtures of the REAL reference's algorithm (tests/golden/make_large_fixtures.py:
the reference's operator, deflation space and loop; a sparse exact coarse
solve instead of the dense cho_solve).

Per recorded stop of the reference (tolerance 1e-8 / 1e-11, or a fixed
iteration count k), following SURVEY §0.5 / §8(c) ("parity of the solution
must be judged at a tight tolerance or at a fixed iteration count; report
tol 1e-8 differences alongside, as information" -- the reference's own two
backends are 1.2e-10 apart at a 1e-8 stop):
  * every tolerance stop: the device solve at that tolerance stops within +-1
    iteration of the reference, and its compliance f.u matches to 1e-8.
    Both projections are run: ``reference`` is the reference's recurrence
    step for step; ``stabilized`` (the default, solver.cu) re-imposes
    W^T A p = 0 every iteration. At a 1e-11 stop after ~1070 iterations the
    reference recurrence's residual carries ~10 % of accumulated drift that
    the stabilised one does not (device residual at x_1073 of c4_bern_y:
    9.48e-12 with the reference projection, CPU reference 9.54e-12,
    stabilised 8.62e-12), so the stabilised solve may stop up to 0.3 % of the
    iterations EARLIER there (never more than 1 later);
  * tight stops (1e-11) and fixed-iteration iterates: the device iterate after
    the SAME number of iterations (solve_static with that max_iters;
    NoConvergence carries the iterate) matches the reference's within 1e-10
    relative (north-star solution tolerance) at 4096 seeded sample DOFs, in
    norm and in f.u;
  * 1e-8 stops: the same comparison is reported, and bounded by 1e-9 (the
    order of the iterate's own truncation error, 3e-10 .. 1.4e-9 on these
    problems). Measured: <= 2.5e-11 except the two C4 Bernoulli(0.9) cases
    after ~940 iterations (7.5e-11 and 1.2e-10; the reference against itself
    with K.u rounded differently moves 8.5e-12 there, tests/golden/
    noise_floor.py).

(The reference's recurrence diverges at 1e-12 on some of these problems --
e.g. the C1 geometry with a face load reaches residual 8.8e3 at its iteration
cap -- so 1e-11 is the tightest tolerance recorded.)
"""

import os

import numpy as np
import pytest

import large_cases as LC

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "large_dpcg.npz")
SOL_TOL = 1e-10   # north star: PCG solution within 1e-10 relative
LOOSE_TOL = 1e-9  # iterate at a 1e-8 stop (information): order of its truncation error
J_TOL = 1e-8      # north star: compliance within 1e-8 relative


def _fixture():
    return np.load(FIX) if os.path.exists(FIX) else None


def _tags(fx, name):
    tags = sorted({k[len(name) + 1:].rsplit("_", 1)[0] for k in fx.files
                   if k.startswith(name + "_") and k.endswith("_u")})
    return tags


def test_fixture_covers_every_case():
    fx = _fixture()
    assert fx is not None, "tests/golden/large_dpcg.npz missing (run tests/golden/make_large_fixtures.py)"
    for name, spec in LC.CASES.items():
        tags = _tags(fx, name)
        for t in spec["tols"]:
            if f"tol{t:g}" not in tags:
                assert "no convergence" in str(fx[f"{name}_status"]), (name, t)
        for k in spec["iters"]:
            assert f"k{k}" in tags, (name, k)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


_CACHE = {}


def _problem(name):
    """(op, deflation, f on device) of a case, cached for the last case key."""
    import torch

    import paper_2203_15115_b200 as tv
    from paper_2203_15115_b200 import fea, mesh

    spec = LC.CASES[name]
    key = (spec["dims"], spec["occ"], spec["block"], spec["load"])
    if key not in _CACHE:
        _CACHE.clear()
        torch.cuda.empty_cache()
        d, fixed, f, occ = LC.problem(mesh, spec)
        op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
        defl = fea.build_deflation(d, op.topology, fixed, spec["block"])
        _CACHE[key] = (op, defl, torch.from_numpy(f).cuda(), f, fixed)
    return _CACHE[key]


def _iteration_window(projection, tag, it_ref):
    """Allowed (lo, hi) stopping iterations of the device solve."""
    early = 1
    if projection == "stabilized" and tag != "tol1e-08":
        early = max(1, int(np.ceil(0.003 * it_ref)))
    return it_ref - early, it_ref + 1


@pytest.mark.gpu
@pytest.mark.parametrize("projection", ["stabilized", "reference"])
@pytest.mark.parametrize("name", list(LC.CASES))
def test_dpcg_matches_reference_at_full_size(name, projection):
    from paper_2203_15115_b200 import fea
    from paper_2203_15115_b200.errors import NoConvergence

    fx = _fixture()
    assert fx is not None
    op, defl, fd, f, fixed = _problem(name)
    assert len(fixed) == int(fx[f"{name}_nfixed"])
    assert np.abs(f).sum() == pytest.approx(float(fx[f"{name}_fsum"]), rel=1e-14)
    assert defl.n_vectors == int(fx[f"{name}_nvec"])
    idx = fx[f"{name}_idx"]
    report = []
    for tag in _tags(fx, name):
        it_ref = int(fx[f"{name}_{tag}_it"])
        u_ref, J_ref = fx[f"{name}_{tag}_u"], float(fx[f"{name}_{tag}_J"])
        if tag.startswith("tol"):
            tol = float(tag[3:])
            r = fea.solve_static(op, fd, tol=tol, deflation=defl, projection=projection)
            lo, hi = _iteration_window(projection, tag, it_ref)
            assert lo <= r.iterations <= hi, (name, projection, tag, r.iterations, it_ref)
            J = float(fd @ r.u)
            assert abs(J - J_ref) <= J_TOL * abs(J_ref), (name, tag, J, J_ref)
            report.append(f"{tag}: it {r.iterations} (ref {it_ref}) J rel {abs(J - J_ref) / abs(J_ref):.1e}")
        # the iterate after exactly it_ref iterations
        with pytest.raises(NoConvergence) as ei:
            fea.solve_static(op, fd, tol=1e-14, max_iters=it_ref, deflation=defl, projection=projection)
        x = ei.value.u
        assert x is not None and ei.value.iterations == it_ref
        xs = x[idx].cpu().numpy()
        e_u = _rel(xs, u_ref)
        e_n = abs(float(x.norm()) - float(fx[f"{name}_{tag}_norm"])) / float(fx[f"{name}_{tag}_norm"])
        e_j = abs(float(fd @ x) - J_ref) / abs(J_ref)
        bound = LOOSE_TOL if tag == "tol1e-08" else SOL_TOL
        report.append(f"x_{it_ref}: u rel {e_u:.1e} |u| rel {e_n:.1e} J rel {e_j:.1e}")
        assert e_u <= bound and e_n <= bound and e_j <= bound, (name, projection, tag, e_u, e_n, e_j, bound)
    print(f"[large parity] {name} ({projection}): " + "; ".join(report))
