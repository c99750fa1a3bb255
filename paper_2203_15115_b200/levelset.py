"""Augmented topological level set on the GPU (SPEC ``level_set_topology``).

No reference code exists; semantics follow
``/root/reference/SPEC.md:360-439``:

* ``normalize_field``  T / max|T| (zero field unchanged)
* ``combine``          T_L = sum_i w_i T^_i, T_phi = 0; all-zero weights
                       fall back to the compliance field, weight 1
* ``extract``          order-statistic threshold over design elements,
                       ties by ascending element index
* ``fixed_point``      FEA -> fields -> combine -> extract loop

The retained count for a target fraction v is ``k = floor(v * n_design + 1/2)``
(the SPEC only requires the fraction to be within 1/n_design; this rounding
is the documented builder decision, mirrored by the oracle).
"""

from __future__ import annotations

import ctypes
import logging

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


def retained_count(target_vf: float, n_design: int) -> int:
    return int(min(max(np.floor(target_vf * n_design + 0.5), 0), n_design))


def extract_device(domain: Domain, levelset_d, target_vf: float, ersatz: float = EPS_VOID, design_d=None):
    """Device occupancy for the target fraction; returns (occ_d, k, state4)."""
    torch = _t()
    n = domain.n_elems
    if design_d is None:
        design_d = torch.from_numpy(domain.design_mask.astype(np.uint8)).cuda()
    k = retained_count(target_vf, domain.n_design)
    occ = torch.empty(n, dtype=torch.float64, device="cuda")
    nws = lib().tvb_select_ws_bytes(n)
    ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
    state = (ctypes.c_ulonglong * 4)()
    check(lib().tvb_threshold_select(ptr(levelset_d), ptr(design_d), n, k, float(ersatz), float(EPS_VOID), ptr(occ),
                                     ptr(ws), nws, ctypes.cast(state, ctypes.c_void_p), stream_ptr()), "extract")
    return occ, k, tuple(state)


def extract(domain: Domain, levelset, target_vf: float, ersatz: float = EPS_VOID) -> Topology:
    """Topology keeping the ``k`` largest level-set values among design
    elements."""
    if not 0.0 < target_vf <= 1.0:
        raise ValueError(f"target volume fraction must lie in (0, 1], got {target_vf}")
    t, _ = _dev(levelset)
    if t.numel() != domain.n_elems:
        raise ValueError("level set length does not match the element count")
    occ, _, _ = extract_device(domain, t, target_vf, ersatz)
    return Topology(domain, occ.cpu().numpy())


def key_to_double(key: int) -> float:
    """Inverse of the kernel's order-preserving key (for reporting tau)."""
    if key >> 63:
        bits = key & 0x7FFFFFFFFFFFFFFF
    else:
        bits = (~key) & 0xFFFFFFFFFFFFFFFF
    return float(np.array([bits], dtype=np.uint64).view(np.float64)[0])
