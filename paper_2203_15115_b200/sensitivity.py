"""Per-element topological sensitivities on the GPU (SPEC ``sensitivity_fields``).

The reference package has no code for this module; the
semantics follow ``/root/reference/SPEC.md:268-358`` and the paper's Eqs
3.2-3.3 (``PAPER.md:162,172``):

* ``compliance_sensitivity`` T_J = 4/(1+nu) s:e - (1-3nu)/(1-nu^2) tr s tr e
* ``pnorm_stress``            sigma_PN = (sum_e w_e vm_e^p)^(1/p), w = occ/sum occ
* ``stress_adjoint``          K lambda = d sigma_PN / du, same DPCG
* ``stress_sensitivity``      T_sigma with sigma(u) and eps(lambda)

Functions take the ``StiffnessOperator`` (which carries domain, topology and
material) plus device or numpy vectors; results mirror the input kind.
"""

from __future__ import annotations

import numpy as np

from ._lib import check, lib, ptr, stream_ptr
from .errors import SemanticError
from .fea import solve_static, to_device, to_host_if


def _t():
    from ._lib import require_cuda

    return require_cuda()


def _args(op):
    d, m = op.domain, op.material
    return d.nx, d.ny, d.nz, d.h, m.E, m.nu


def element_state_device(op, u_d, want=("strains", "stresses", "vm")):
    """(strains, stresses, vm) device tensors for every element."""
    torch = _t()
    ne = op.domain.n_elems
    strains = torch.empty((ne, 6), dtype=torch.float64, device="cuda") if "strains" in want else None
    stresses = torch.empty((ne, 6), dtype=torch.float64, device="cuda") if "stresses" in want else None
    vm = torch.empty(ne, dtype=torch.float64, device="cuda") if "vm" in want else None
    check(lib().tvb_element_state(*_args(op), ptr(u_d), ptr(op.occ_d), ptr(strains), ptr(stresses), ptr(vm), None, 0,
                                  None, None, 0, stream_ptr()), "element state")
    return strains, stresses, vm


def element_fields_device(op, u_d, p: int = 8):
    """One pass: (vm, T_J, (sum occ vm^p, sum occ)) as device tensors."""
    torch = _t()
    d = op.domain
    vm = torch.empty(d.n_elems, dtype=torch.float64, device="cuda")
    tj = torch.empty(d.n_elems, dtype=torch.float64, device="cuda")
    sums = torch.empty(2, dtype=torch.float64, device="cuda")
    nws = lib().tvb_elem_ws_bytes(d.nx, d.ny, d.nz)
    ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
    check(lib().tvb_element_state(*_args(op), ptr(u_d), ptr(op.occ_d), None, None, ptr(vm), ptr(tj), int(p), ptr(sums),
                                  ptr(ws), nws, stream_ptr()), "element fields")
    return vm, tj, sums


def compliance_sensitivity(op, u):
    """T_J per element, evaluated at the centroid with the
    occupancy-scaled stress (void elements get their ersatz values)."""
    torch = _t()
    u_d, np_in = to_device(u, op.n_dofs, "displacement vector")
    d = op.domain
    tj = torch.empty(d.n_elems, dtype=torch.float64, device="cuda")
    check(lib().tvb_element_state(*_args(op), ptr(u_d), ptr(op.occ_d), None, None, None, ptr(tj), 0, None, None, 0,
                                  stream_ptr()), "compliance sensitivity")
    return to_host_if(tj, np_in)


def pnorm_sums(op, u_d, p: int):
    _, _, sums = element_fields_device(op, u_d, p)
    return sums


def pnorm_stress(op, u, p: int = 6) -> float:
    """sigma_PN: volume-normalised p-mean of von Mises."""
    if p < 2 or p % 2:
        raise SemanticError(f"p-norm exponent must be an even integer >= 2, got {p}")
    u_d, _ = to_device(u, op.n_dofs, "displacement vector")
    s = pnorm_sums(op, u_d, p).cpu().numpy()
    return float((s[0] / s[1]) ** (1.0 / p))


def adjoint_rhs_device(op, u_d, p: int, sums=None):
    torch = _t()
    if sums is None:
        sums = pnorm_sums(op, u_d, p)
    d = op.domain
    rhs = torch.empty(d.n_dofs, dtype=torch.float64, device="cuda")
    ws = torch.empty(48 * d.n_elems + 8, dtype=torch.uint8, device="cuda")
    check(lib().tvb_adjoint_rhs(*_args(op), ptr(u_d), ptr(op.occ_d), ptr(op.nflags), int(p), ptr(sums), ptr(rhs),
                                ptr(ws), ws.numel(), stream_ptr()), "adjoint rhs")
    return rhs


def adjoint_rhs(op, u, p: int = 6):
    """d sigma_PN / du with fixed DOFs zeroed."""
    u_d, np_in = to_device(u, op.n_dofs, "displacement vector")
    sums = pnorm_sums(op, u_d, p)
    if not float(sums[0]) > 0.0:
        raise SemanticError("sigma_PN is zero (zero displacement): the stress adjoint is undefined")
    return to_host_if(adjoint_rhs_device(op, u_d, p, sums), np_in)


def stress_adjoint(op, u, p: int = 6, tol: float = 1e-8, deflation=None, max_iters=None):
    """Adjoint field lambda: K lambda = +d sigma_PN / du, solved with the same
    (deflated) PCG and tolerance as the primal."""
    u_d, np_in = to_device(u, op.n_dofs, "displacement vector")
    rhs = adjoint_rhs(op, u_d, p)
    res = solve_static(op, rhs, tol=tol, deflation=deflation, max_iters=max_iters)
    return to_host_if(res.u, np_in)


def stress_sensitivity(op, u, lam):
    """T_sigma = 4/(1+nu) sigma(u):eps(lambda) - (1-3nu)/(1-nu^2) tr sigma(u) tr eps(lambda)."""
    torch = _t()
    u_d, np_in = to_device(u, op.n_dofs, "displacement vector")
    l_d, _ = to_device(lam, op.n_dofs, "adjoint vector")
    ts = torch.empty(op.domain.n_elems, dtype=torch.float64, device="cuda")
    check(lib().tvb_sens_stress(*_args(op), ptr(u_d), ptr(l_d), ptr(op.occ_d), ptr(ts), stream_ptr()),
          "stress sensitivity")
    return to_host_if(ts, np_in)


__all__ = [
    "compliance_sensitivity", "pnorm_stress", "adjoint_rhs", "stress_adjoint", "stress_sensitivity",
    "element_state_device", "element_fields_device",
]


