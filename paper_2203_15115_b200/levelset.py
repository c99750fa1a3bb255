"""Augmented topological level set on the GPU (SPEC ``level_set_topology``).

No reference code exists; semantics follow
``/root/reference/SPEC.md:360-439``:

* ``normalize_field``  T / max|T| (zero field unchanged)
* ``combine``          T_L = sum_i w_i T^_i, T_phi = 0; all-zero weights
                       fall back to the compliance field, weight 1
* ``extract``          order-statistic threshold over design elements,
                       ties by ascending element index
* ``fixed_point``      FEA -> fields -> combine -> extract loop
* ``casting_project``  running minimum away from the parting plane    SPEC.md:402-410 (PAPER §3.7)

The retained count for a target fraction v is ``k = floor(v * n_design + 1/2)``
(the SPEC only requires the fraction to be within 1/n_design; this rounding
is the documented builder decision, mirrored by the oracle).
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib, ptr, stream_ptr
from .mesh import EPS_VOID, Domain, Topology

log = logging.getLogger(__name__)


def _t():
    from ._lib import require_cuda

    return require_cuda()


def _dev(x):
    torch = _t()
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda(), True


def maxabs_device(t_d):
    torch = _t()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(1184 * 8, dtype=torch.uint8, device="cuda")
    check(lib().tvb_maxabs(ptr(t_d), t_d.numel(), ptr(out), ptr(ws), ws.numel(), stream_ptr()), "maxabs")
    return out


def normalize_field(field):
    """values / max|values|; an all-zero field is returned unchanged."""
    t, np_in = _dev(field)
    out = combine_device([t], [1.0])
    return out.cpu().numpy() if np_in else out


def combine_device(fields, weights, maxabs=None):
    """sum_i w_i * t_i / max|t_i| on device tensors (one fused pass)."""
    torch = _t()
    k = len(fields)
    if not 1 <= k <= 8:
        raise ValueError("combine supports 1..8 fields")
    n = fields[0].numel()
    if maxabs is None:
        maxabs = torch.cat([maxabs_device(f) for f in fields])
    ptrs = (ctypes.c_void_p * k)(*[f.data_ptr() for f in fields])
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    check(lib().tvb_combine(k, ctypes.cast(ptrs, ctypes.c_void_p), w.ctypes.data, ptr(maxabs), n, ptr(out),
                            stream_ptr()), "combine")
    return out


def combine(fields, weights, fallback: int = 0):
    """(T_L, used_fallback). Weights are the Eq 3.18 values max(mu + gamma g, 0);
    when every weight is zero the field ``fallback`` (compliance) is used with
    unit weight and the event is logged (SPEC AllWeightsZero)."""
    ts = [_dev(f) for f in fields]
    np_in = ts[0][1]
    tens = [t for t, _ in ts]
    weights = [float(w) for w in weights]
    used_fallback = all(w == 0.0 for w in weights)
    if used_fallback:
        log.info("all augmented-Lagrangian weights are zero: falling back to the compliance field")
        out = combine_device([tens[fallback]], [1.0])
    else:
        out = combine_device(tens, weights)
    return (out.cpu().numpy() if np_in else out), used_fallback


_AXES = {"x": 0, "y": 1, "z": 2}


@dataclass(frozen=True)
class CastingSpec:
    """Casting constraint (PAPER §3.7).

    ``axis``: one of ``+x -x +y -y +z -z``. ``parting_plane``: node-plane index
    along the axis where two mold halves separate (element layers at or above
    it pull towards +axis, those below towards -axis; the sign is then
    irrelevant), or None for single-direction mode: one mold half pulled along
    the signed axis, its parting plane the grid face the pull starts from
    (index 0 for +, n_axis for -)."""

    axis: str
    parting_plane: int | None = None

    def __post_init__(self):
        if len(self.axis) != 2 or self.axis[0] not in "+-" or self.axis[1] not in _AXES:
            raise ValueError(f"casting axis must be one of +x -x +y -y +z -z, got {self.axis!r}")

    def resolve(self, domain: Domain) -> tuple[int, int]:
        """(axis index, first element layer of the +axis half)."""
        a = _AXES[self.axis[1]]
        n = (domain.nx, domain.ny, domain.nz)[a]
        if self.parting_plane is None:
            return a, (0 if self.axis[0] == "+" else n)
        p = int(self.parting_plane)
        if not 0 <= p <= n:
            raise ValueError(f"parting plane {p} outside the grid (0..{n}) along {self.axis[1]}")
        return a, p


def casting_project_device(domain: Domain, field_d, spec: CastingSpec, out_d=None):
    """Device casting projection (``tvb_casting_project``); in place if out_d is field_d."""
    torch = _t()
    a, p = spec.resolve(domain)
    if out_d is None:
        out_d = torch.empty_like(field_d)
    check(lib().tvb_casting_project(domain.nx, domain.ny, domain.nz, a, p, ptr(field_d), ptr(out_d), stream_ptr()),
          "casting projection")
    return out_d


def casting_project(domain: Domain, field, spec: CastingSpec):
    """SPEC ``casting_project``: along each element column
    parallel to the casting axis and on each side of the parting plane, the
    running minimum moving away from the plane; every superlevel set is then a
    run touching the plane (no undercuts). Idempotent."""
    t, np_in = _dev(field)
    if t.numel() != domain.n_elems:
        raise ValueError("field length does not match the element count")
    out = casting_project_device(domain, t, spec)
    return out.cpu().numpy() if np_in else out


def retained_count(target_vf: float, n_design: int) -> int:
    return int(min(max(np.floor(target_vf * n_design + 0.5), 0), n_design))


def extract_device(domain: Domain, levelset_d, target_vf: float, ersatz: float = EPS_VOID, design_d=None,
                   casting: CastingSpec | None = None):
    """Device occupancy for the target fraction; returns (occ_d, k, state4).
    With ``casting`` the level set is casting-projected first and every
    design element tied with the threshold is retained (the
    fraction may exceed the target; the retained set stays undercut-free)."""
    torch = _t()
    if casting is not None:
        levelset_d = casting_project_device(domain, levelset_d, casting)
    n = domain.n_elems
    if design_d is None:
        design_d = torch.from_numpy(domain.design_mask.astype(np.uint8)).cuda()
    k = retained_count(target_vf, domain.n_design)
    occ = torch.empty(n, dtype=torch.float64, device="cuda")
    nws = lib().tvb_select_ws_bytes(n)
    ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
    state = (ctypes.c_ulonglong * 4)()
    check(lib().tvb_threshold_select_ex(ptr(levelset_d), ptr(design_d), n, k, float(ersatz), float(EPS_VOID),
                                        1 if casting is not None else 0, ptr(occ), ptr(ws), nws,
                                        ctypes.cast(state, ctypes.c_void_p), stream_ptr()), "extract")
    return occ, k, tuple(state)


def extract(domain: Domain, levelset, target_vf: float, ersatz: float = EPS_VOID,
            casting: CastingSpec | None = None) -> Topology:
    """Topology keeping the ``k`` largest level-set values among design
    elements; with ``casting``, of the casting-projected
    level set, ties at the threshold all retained."""
    if not 0.0 < target_vf <= 1.0:
        raise ValueError(f"target volume fraction must lie in (0, 1], got {target_vf}")
    t, _ = _dev(levelset)
    if t.numel() != domain.n_elems:
        raise ValueError("level set length does not match the element count")
    occ, _, _ = extract_device(domain, t, target_vf, ersatz, casting=casting)
    return Topology(domain, occ.cpu().numpy())


def key_to_double(key: int) -> float:
    """Inverse of the kernel's order-preserving key (for reporting tau)."""
    if key >> 63:
        bits = key & 0x7FFFFFFFFFFFFFFF
    else:
        bits = (~key) & 0xFFFFFFFFFFFFFFFF
    return float(np.array([bits], dtype=np.uint64).view(np.float64)[0])
