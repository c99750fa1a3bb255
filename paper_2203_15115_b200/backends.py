"""The kernel seam of the reference (``topovox/backends/__init__.py:49-52``),
re-implemented on the GPU with the reference's positional signatures.

``apply_block24(u, out, elem_dofs, scale, k0, color_perm, color_ptr)``
accumulates ``out += sum_e scale_e * scatter(k0 @ gather(u, e))`` like the
numba kernel. The element->DOF table is only checked for the structured
voxel numbering (the GPU derives indices from the grid dimensions, which are
recovered from the table); colouring arguments are accepted and ignored
(the CUDA kernel is race-free by node ownership). Arrays may be numpy
(copied to the device and back into ``out`` in place) or CUDA tensors.
"""

from __future__ import annotations

import numpy as np

from ._lib import ACCUMULATE, check, lib, ptr, require_cuda, stream_ptr
from .errors import DimensionMismatch

BACKEND = "cuda-sm100a"


def backend_name() -> str:
    return BACKEND


def grid_from_elem_dofs(elem_dofs) -> tuple[int, int, int]:
    """Recover (nx, ny, nz) from a reference-numbered element->DOF table."""
    ed = np.asarray(elem_dofs[:1].cpu() if hasattr(elem_dofs, "cpu") else elem_dofs[:1])
    ne = int(elem_dofs.shape[0])
    n = ed[0, ::3] // 3  # 8 node ids of element 0
    nx = int(n[2] - n[1])  # node (1,1,0) - node (1,0,0) = nx + 1 ... minus 1
    nx -= 1
    pxy = int(n[4])
    ny = pxy // (nx + 1) - 1
    if nx < 1 or ny < 1 or ne % (nx * ny):
        raise DimensionMismatch("element->DOF table is not a structured voxel numbering")
    nz = ne // (nx * ny)
    return nx, ny, nz


def _check_table(elem_dofs, dims):
    from .mesh import Domain

    ref = Domain(*dims, 1.0).elem_dofs
    ed = elem_dofs.cpu().numpy() if hasattr(elem_dofs, "cpu") else np.asarray(elem_dofs)
    probe = np.unique(np.linspace(0, ed.shape[0] - 1, num=min(ed.shape[0], 64)).astype(np.int64))
    if not np.array_equal(ed[probe], ref[probe]):
        raise DimensionMismatch("element->DOF table is not a structured voxel numbering")


def _modal(k0):
    k0 = np.ascontiguousarray(np.asarray(k0.cpu() if hasattr(k0, "cpu") else k0, dtype=np.float64))
    mh = np.empty(45)
    check(lib().tvb_modal_from_k0(k0.ctypes.data, mh.ctypes.data), "modal coefficients")
    return mh


def _dev(a, dtype=None):
    torch = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype or a.dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _writeback(out, out_d):
    torch = require_cuda()
    if isinstance(out, torch.Tensor):
        if out.data_ptr() != out_d.data_ptr():
            out.copy_(out_d)
    else:
        out[...] = out_d.cpu().numpy()


def apply_block24(u, out, elem_dofs, scale, k0, color_perm=None, color_ptr=None):
    torch = require_cuda()
    dims = grid_from_elem_dofs(elem_dofs)
    _check_table(elem_dofs, dims)
    u_d, out_d, s_d = _dev(u, torch.float64), _dev(out, torch.float64), _dev(scale, torch.float64)
    check(lib().tvb_matvec(*dims, _modal(k0).ctypes.data, ptr(u_d), ptr(out_d), ptr(s_d), None, ACCUMULATE, None, None,
                           0, stream_ptr()), "apply_block24")
    _writeback(out, out_d)


def apply_block24_subset(u, out, elem_ids, elem_dofs, scale, k0):
    torch = require_cuda()
    dims = grid_from_elem_dofs(elem_dofs)
    _check_table(elem_dofs, dims)
    u_d, out_d, s_d = _dev(u, torch.float64), _dev(out, torch.float64), _dev(scale, torch.float64)
    el = _dev(np.asarray(elem_ids, dtype=np.int64) if not isinstance(elem_ids, torch.Tensor) else elem_ids,
              torch.int64)
    ne = dims[0] * dims[1] * dims[2]
    ws = torch.empty(12 * ne + 16, dtype=torch.uint8, device="cuda")
    check(lib().tvb_matvec_subset(*dims, _modal(k0).ctypes.data, ptr(u_d), ptr(out_d), ptr(el), el.numel(), ptr(s_d),
                                  ptr(ws), ws.numel(), stream_ptr()), "apply_block24_subset")
    _writeback(out, out_d)


def diag_block24(out, elem_dofs, scale, k0_diag):
    torch = require_cuda()
    dims = grid_from_elem_dofs(elem_dofs)
    _check_table(elem_dofs, dims)
    kd = np.asarray(k0_diag.cpu() if hasattr(k0_diag, "cpu") else k0_diag, dtype=np.float64)
    if not np.allclose(kd, kd[0], rtol=1e-12, atol=0.0):
        raise ValueError("k0 diagonal is not uniform: not a cube element")
    kd3 = np.ascontiguousarray(kd[:3])
    out_d, s_d = _dev(out, torch.float64), _dev(scale, torch.float64)
    check(lib().tvb_diag(*dims, ptr(s_d), None, kd3.ctypes.data, ptr(out_d), 1, None, None, stream_ptr()),
          "diag_block24")
    _writeback(out, out_d)


def apply_nodal_block8(u, out, elem_dofs, blocks, color_perm=None, color_ptr=None):
    """out += scatter of per-element 8x8 nodal blocks acting on each
    displacement component (reference ``numba_kernels.py:61-76``; geometric
    stiffness). blocks: (Ne, 8, 8) in the element's local node order."""
    torch = require_cuda()
    dims = grid_from_elem_dofs(elem_dofs)
    _check_table(elem_dofs, dims)
    ne = dims[0] * dims[1] * dims[2]
    if tuple(blocks.shape) != (ne, 8, 8):
        raise DimensionMismatch(f"blocks have shape {tuple(blocks.shape)}, expected ({ne}, 8, 8)")
    u_d, out_d, b_d = _dev(u, torch.float64), _dev(out, torch.float64), _dev(blocks, torch.float64)
    check(lib().tvb_nodal_block8(*dims, ptr(u_d), ptr(out_d), ptr(b_d), stream_ptr()), "apply_nodal_block8")
    _writeback(out, out_d)


def element_coloring(ix, iy, iz):
    """Parity colouring (reference ``backends/__init__.py:59-66``); kept for
    API compatibility -- the CUDA kernels do not need it."""
    color = (np.asarray(ix) & 1) + 2 * (np.asarray(iy) & 1) + 4 * (np.asarray(iz) & 1)
    perm = np.argsort(color, kind="stable").astype(np.int64)
    ptr_ = np.concatenate([[0], np.cumsum(np.bincount(color, minlength=8))]).astype(np.int64)
    return perm, ptr_


def set_threads(n: int) -> None:
    """No-op (reference caps the numba pool); the GPU has no thread knob."""
    return None
