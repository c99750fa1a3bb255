"""Host-side logic (problem setup, element constants, C-ABI library
loading) checked against the reference's golden vectors. CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, cantilever
from paper_2203_15115_b200 import elements, mesh
from paper_2203_15115_b200.errors import BadDimension, EmptyDomain, EmptyLoadRegion, SemanticError


def test_k0_and_modal(golden):
    k0 = elements.hex_stiffness(elements.Material(E=1.0, nu=0.3), 1.0)
    assert np.allclose(k0, golden["k0_unit"], rtol=0, atol=1e-15)
    k1 = elements.hex_stiffness(elements.Material(E=2e11, nu=0.25), 0.5)
    assert np.abs(k1 - golden["k0_steel"]).max() <= 1e-14 * np.abs(k1).max()
    # mode-space factorisation reproduces k0 exactly (to rounding)
    M = elements.modal_coupling(k0)
    H3 = np.kron(elements.hadamard_nodes(), np.eye(3))
    assert np.abs(H3 @ M @ H3.T - k0).max() < 1e-14
    assert np.count_nonzero(M) == 45


def test_modal_pattern_rejects_non_cube():
    k0 = elements.hex_stiffness(elements.Material(E=1.0, nu=0.3), 1.0)
    bad = k0.copy()
    bad[0, 5] += 0.1
    bad[5, 0] += 0.1
    with pytest.raises(ValueError):
        elements.modal_coupling(bad)


def test_modal_codegen_in_sync():
    src = open(os.path.join(ROOT, "paper_2203_15115_b200", "csrc", "modal_entries.inc")).read()
    entries = [tuple(map(int, m)) for m in re.findall(r"\{(\d+), (\d+)\}", src)]
    k0 = elements.hex_stiffness(elements.Material(E=1.0, nu=0.3), 1.0)
    M = elements.modal_coupling(k0)
    vtk_to_bin = [int(o[0] + 2 * o[1] + 4 * o[2]) for o in elements.NODE_OFFSETS]
    perm = np.empty(24, dtype=int)
    for n in range(8):
        for a in range(3):
            perm[3 * vtk_to_bin[n] + a] = 3 * n + a
    Mb = M[np.ix_(perm, perm)]
    assert entries == [(i, j) for i in range(24) for j in range(24) if Mb[i, j] != 0.0]


def test_centroid_b_and_elasticity():
    B = elements.centroid_b_matrix(2.0)
    assert set(np.unique(np.abs(B[B != 0]))) == {0.125}
    D = elements.elasticity_matrix(1.0, 0.3)
    c = 1.0 / (1.3 * 0.4)
    assert D[0, 0] == pytest.approx(c * 0.7) and D[0, 1] == pytest.approx(c * 0.3) and D[3, 3] == pytest.approx(c * 0.2)


def test_elem_dofs_and_counts():
    d = mesh.Domain(2, 1, 1, 1.0)
    assert (d.n_elems, d.n_nodes, d.n_dofs) == (2, 12, 36)
    ed = d.elem_dofs
    assert ed.dtype == np.int32 and ed.shape == (2, 24)
    assert list(ed[1, ::3] // 3) == [1, 2, 5, 4, 7, 8, 11, 10]


def test_load_cases_match_reference(golden):
    d, case, fixed, f = cantilever(40, 20, 20, (40, 10, 10), (40, 10, 10))
    assert fixed.size == int(golden["c1_nfixed"]) == 1323
    assert np.array_equal(np.flatnonzero(f), golden["c1_fnz"])
    for name, dims, lo, hi, force in [
        ("c3", (80, 40, 40), (80, 20, 20), (80, 20, 20), (0, 0, -1)),
        ("c4a", (160, 80, 80), (160, 39, 39), (160, 41, 41), (0, 0, -1)),
        ("c4b", (160, 80, 80), (160, 39, 39), (160, 41, 41), (0, -1, 0)),
    ]:
        d, case, fixed, f = cantilever(*dims, lo, hi, force)
        assert fixed.size == int(golden[name + "_nfixed"])
        assert int(fixed.sum()) == int(golden[name + "_fixed_sum"])
        nz = np.flatnonzero(f)
        assert np.array_equal(nz, golden[name + "_f_idx"])
        assert np.array_equal(f[nz], golden[name + "_f_val"])


def test_selectors_and_errors():
    d = mesh.Domain(2, 1, 1, 1.0)
    face = mesh.select(d, mesh.RegionSelector("box", min=(0, 0, 0), max=(0, 1, 1)))
    assert list(face) == [0, 3, 6, 9]
    one = mesh.select(d, mesh.RegionSelector("sphere", center=(1.0, 1.0, 1.0), radius=0.0))
    assert list(one) == [10]
    with pytest.raises(SemanticError):
        mesh.select(d, mesh.RegionSelector("ids", ids=(0, 99)))
    with pytest.raises(BadDimension):
        mesh.Domain(0, 1, 1, 1.0)
    with pytest.raises(EmptyDomain):
        mesh.build_domain(2, 2, 2, 1.0, csg=[{"op": "subtract", "shape": "box", "min": (0, 0, 0), "max": (2, 2, 2)}])
    case = mesh.LoadCase("x", loads=((mesh.RegionSelector("box", min=(9, 9, 9), max=(9, 9, 9)), (1, 0, 0), "total"),))
    with pytest.raises(EmptyLoadRegion):
        mesh.assemble_force(d, case)
    with pytest.raises(SemanticError):
        mesh.validate_case(d, mesh.LoadCase("y"))
    f = mesh.assemble_force(d, mesh.LoadCase("t", loads=(
        (mesh.RegionSelector("box", min=(0, 0, 0), max=(0, 1, 1)), (0, 0, -100), "total"),)))
    assert np.allclose(f[2::3][[0, 3, 6, 9]], -25.0)


def test_topology_semantics():
    d = mesh.build_domain(4, 2, 1, 1.0, csg=[{"op": "subtract", "shape": "box", "min": (0, 0, 0), "max": (1, 2, 1)}])
    t = mesh.Topology(d)
    assert np.all(t.occupancy[~d.design_mask] == mesh.EPS_VOID)
    assert t.volume_fraction == 1.0
    t2 = t.set_void(np.flatnonzero(d.design_mask)[:1])
    assert t2.volume_fraction == pytest.approx(1 - 1 / d.n_design)
    assert t2 != t and t.copy() == t


def test_library_exports_header_symbols():
    """The built C-ABI library loads (no GPU needed) and exports every symbol
    declared in include/topovox_b200.h; the ctypes table covers them all."""
    from paper_2203_15115_b200 import _build, _lib

    if _build.needs_build():
        _build.build()
    hdr = open(os.path.join(ROOT, "include", "topovox_b200.h")).read()
    declared = set(re.findall(r"\b(tvb_[a-z0-9_]+)\s*\(", hdr))
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.exported_symbols())
    assert L.tvb_version() == 1


def test_host_modal_matches_library():
    from paper_2203_15115_b200 import _lib

    k0 = np.ascontiguousarray(elements.hex_stiffness(elements.Material(E=3.0, nu=0.2), 0.7))
    mh = np.empty(45)
    assert _lib.lib().tvb_modal_from_k0(k0.ctypes.data, mh.ctypes.data) == 0
    src = open(os.path.join(ROOT, "paper_2203_15115_b200", "csrc", "modal_entries.inc")).read()
    entries = [tuple(map(int, m)) for m in re.findall(r"\{(\d+), (\d+)\}", src)]
    M = elements.modal_coupling(k0)
    vtk_to_bin = [int(o[0] + 2 * o[1] + 4 * o[2]) for o in elements.NODE_OFFSETS]
    perm = np.empty(24, dtype=int)
    for n in range(8):
        for a in range(3):
            perm[3 * vtk_to_bin[n] + a] = 3 * n + a
    Mb = M[np.ix_(perm, perm)]
    assert np.allclose(mh, [Mb[i, j] for i, j in entries], rtol=1e-13, atol=0)
    bad = k0.copy()
    bad[0, 7] += 1.0
    bad[7, 0] += 1.0
    assert _lib.lib().tvb_modal_from_k0(np.ascontiguousarray(bad).ctypes.data, mh.ctypes.data) != 0
