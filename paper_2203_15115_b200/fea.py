"""Assembly-free voxel elasticity on the GPU: the drop-in for ``topovox.fea``.

Same classes, functions, signatures and error behaviour as the reference
(``topovox/fea.py:30-342``); every array operation runs in the sm_100a kernels
of ``libtopovox_b200.so``:

* ``StiffnessOperator.apply``   -> ``tvb_matvec``   (K1, node-owner mode-space matvec)
* ``StiffnessOperator.diagonal``-> ``tvb_diag``     (K2)
* ``DeflationSpace``            -> ``tvb_defl_build`` / ``tvb_coarse_assemble`` (+ coarse factor)
* ``solve_static``              -> ``tvb_pcg_solve`` (graph-batched device PCG loop)
* ``batch_element_state``       -> ``tvb_element_state`` (see sensitivity.py)

Arrays: methods accept numpy arrays (copied to the device and the result
copied back, like the reference) or CUDA ``torch.float64`` tensors (zero-copy,
result stays on the device).
"""

from __future__ import annotations

import ctypes
import logging
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib, ptr, require_cuda, stream_ptr
from .elements import Material, centroid_b_matrix, elasticity_matrix, hex_stiffness
from .errors import DimensionMismatch, NoConvergence, SingularSystem, raise_for_status, STATUS_NO_CONVERGENCE
from .mesh import Domain, Topology

log = logging.getLogger(__name__)

DENSE_ORACLE_DOF_LIMIT = 3000
#: coarse spaces up to this many DOFs use an explicit dense inverse (one
#: GEMV per iteration beats the nested-dissection launches); larger ones the
#: nested-dissection block-LDL^T factor (coarse.py)
DENSE_COARSE_AUTO_LIMIT = 3000
DENSE_COARSE_MAX = 24000


def _torch():
    return require_cuda()


def to_device(x, n: int, what: str, dtype=None):
    """(cuda tensor, came_from_numpy). Validates the length."""
    torch = _torch()
    dtype = dtype or torch.float64
    if isinstance(x, torch.Tensor):
        if tuple(x.shape) != (n,):
            raise DimensionMismatch(f"{what} has shape {tuple(x.shape)}, expected ({n},)")
        t = x.to(device="cuda", dtype=dtype)
        return t.contiguous(), False
    a = np.asarray(x, dtype=np.float64 if dtype == torch.float64 else None)
    if a.shape != (n,):
        raise DimensionMismatch(f"{what} has shape {a.shape}, expected ({n},)")
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype), True


def to_host_if(t, numpy_out: bool):
    return t.cpu().numpy() if numpy_out else t


def _node_flags(domain: Domain, occ_d, fixed: np.ndarray):
    torch = _torch()
    fixed_d = torch.from_numpy(np.ascontiguousarray(fixed, dtype=np.int64)).cuda()
    nflags = torch.empty(domain.n_nodes, dtype=torch.uint8, device="cuda")
    check(lib().tvb_node_flags(domain.nx, domain.ny, domain.nz, ptr(fixed_d) if fixed.size else None,
                               int(fixed.size), ptr(occ_d), ptr(nflags), stream_ptr()), "node flags")
    return nflags, fixed_d


class StiffnessOperator:
    """Implicit K = sum_e occupancy_e * k0 with homogeneous Dirichlet DOFs
    (reference ``topovox/fea.py:30-85``)."""

    def __init__(self, domain: Domain, topology: Topology, material: Material, dirichlet=()):
        torch = _torch()
        self.domain = domain
        self.topology = topology
        self.material = material
        self.k0 = hex_stiffness(material, domain.h)
        self._k0c = np.ascontiguousarray(self.k0)
        self._mh = np.empty(45)
        check(lib().tvb_modal_from_k0(self._k0c.ctypes.data, self._mh.ctypes.data), "modal coefficients")
        self._kdiag = np.ascontiguousarray([self.k0[0, 0], self.k0[1, 1], self.k0[2, 2]], dtype=np.float64)
        self.dirichlet = np.asarray(np.unique(np.asarray(dirichlet, dtype=np.int64)), dtype=np.int64)
        if self.dirichlet.size and (self.dirichlet[0] < 0 or self.dirichlet[-1] >= domain.n_dofs):
            raise DimensionMismatch("Dirichlet DOF id out of range")
        self.free_mask = np.ones(domain.n_dofs, dtype=bool)
        self.free_mask[self.dirichlet] = False
        self.occ_d = torch.from_numpy(np.ascontiguousarray(topology.occupancy, dtype=np.float64)).cuda()
        self.nflags, self.fixed_d = _node_flags(domain, self.occ_d, self.dirichlet)
        nbytes = lib().tvb_matvec_ws_bytes(domain.nx, domain.ny, domain.nz)
        self._ws = torch.empty(max(nbytes, 8), dtype=torch.uint8, device="cuda")
        self._diag_d = None
        self._diag = None
        self._inv_d = None
        self._pcg_ws = {}

    @property
    def n_dofs(self) -> int:
        return self.domain.n_dofs

    @property
    def mh(self) -> np.ndarray:
        return self._mh

    def _dims(self):
        d = self.domain
        return d.nx, d.ny, d.nz

    def apply_device(self, u_d, out_d=None, raw: bool = False, accumulate: bool = False, dot_out=None):
        """K @ u on device tensors (no host sync)."""
        torch = _torch()
        if out_d is None:
            out_d = torch.empty_like(u_d)
        flags = 0 if (raw or not self.dirichlet.size) else (_lib.MASK_IN | _lib.MASK_OUT)
        if accumulate:
            flags |= _lib.ACCUMULATE
        check(lib().tvb_matvec(*self._dims(), self._mh.ctypes.data, ptr(u_d), ptr(out_d), ptr(self.occ_d),
                               ptr(self.nflags), flags, ptr(dot_out), ptr(self._ws), self._ws.numel(),
                               stream_ptr()), "matvec")
        return out_d

    def apply(self, u, raw: bool = False):
        """K @ u. With raw=True the Dirichlet rows/columns are kept
        (reference ``topovox/fea.py:49-65``). Host input (numpy / CPU tensor)
        returns host output through the pipelined host path (apply_host)."""
        torch = _torch()
        if isinstance(u, torch.Tensor) and u.is_cuda:
            return self.apply_device(u, raw=raw)
        return self.apply_host(u, raw=raw)

    def apply_host(self, u, out=None, raw: bool = False, slabs: int = 0):
        """K @ u for host vectors (numpy or CPU torch tensor; pinned memory
        lets the copies overlap): z-slab pipeline of host->device copy,
        multiply and device->host copy (``tvb_matvec_host``). Returns ``out``
        (allocated like ``u`` when None)."""
        torch = _torch()
        tensor_in = isinstance(u, torch.Tensor)
        if tensor_in:
            if u.dtype != torch.float64 or u.numel() != self.n_dofs:
                raise DimensionMismatch(f"displacement vector has {tuple(u.shape)}, expected ({self.n_dofs},)")
            u_c = u.contiguous()
            if out is None:
                out = torch.empty(self.n_dofs, dtype=torch.float64, pin_memory=u_c.is_pinned())
            pu, po = u_c.data_ptr(), out.data_ptr()
        else:
            u_c = np.ascontiguousarray(u, dtype=np.float64)
            if u_c.shape != (self.n_dofs,):
                raise DimensionMismatch(f"displacement vector has {u_c.shape}, expected ({self.n_dofs},)")
            if out is None:
                out = np.empty(self.n_dofs)
            pu, po = u_c.ctypes.data, out.ctypes.data
        need = lib().tvb_matvec_host_ws_bytes(*self._dims())
        if getattr(self, "_host_ws", None) is None or self._host_ws.numel() < need:
            self._host_ws = torch.empty(need, dtype=torch.uint8, device="cuda")
        flags = 0 if (raw or not self.dirichlet.size) else (_lib.MASK_IN | _lib.MASK_OUT)
        check(lib().tvb_matvec_host(*self._dims(), self._mh.ctypes.data, pu, po, ptr(self.occ_d), ptr(self.nflags),
                                    flags, int(slabs), ptr(self._host_ws), self._host_ws.numel(), stream_ptr()),
              "matvec (host buffers)")
        return out

    def apply_host_batch(self, us, outs=None, raw: bool = False, slabs: int = 0):
        """K @ u for a sequence of host vectors (numpy arrays or CPU float64
        tensors, pinned for full overlap), streamed through the double-buffered
        slab pipeline (``tvb_matvec_host_batch``): vector v+1's host->device
        copies overlap vector v's device->host copies. Returns ``outs``
        (allocated like the inputs when None); results are bitwise those of
        ``apply_host``."""
        torch = _torch()
        us = list(us)
        if outs is None:
            outs = [torch.empty(self.n_dofs, dtype=torch.float64, pin_memory=u.is_pinned())
                    if isinstance(u, torch.Tensor) else np.empty(self.n_dofs) for u in us]
        outs = list(outs)
        if len(outs) != len(us):
            raise DimensionMismatch(f"{len(us)} input vectors but {len(outs)} outputs")
        keep, pin, pout = [], [], []
        for u, o in zip(us, outs):
            for a, lst in ((u, pin), (o, pout)):
                if isinstance(a, torch.Tensor):
                    if a.dtype != torch.float64 or a.numel() != self.n_dofs or a.is_cuda or not a.is_contiguous():
                        raise DimensionMismatch("host vectors must be contiguous CPU float64 of n_dofs entries")
                    lst.append(a.data_ptr())
                else:
                    arr = a if lst is pout else np.ascontiguousarray(a, dtype=np.float64)
                    if arr.shape != (self.n_dofs,) or arr.dtype != np.float64 or not arr.flags.c_contiguous:
                        raise DimensionMismatch("host vectors must be contiguous float64 of n_dofs entries")
                    keep.append(arr)
                    lst.append(arr.ctypes.data)
        need = lib().tvb_matvec_host_batch_ws_bytes(*self._dims())
        if getattr(self, "_host_bws", None) is None or self._host_bws.numel() < need:
            self._host_bws = torch.empty(need, dtype=torch.uint8, device="cuda")
        flags = 0 if (raw or not self.dirichlet.size) else (_lib.MASK_IN | _lib.MASK_OUT)
        n = len(us)
        hu = (ctypes.c_void_p * max(n, 1))(*pin)
        ho = (ctypes.c_void_p * max(n, 1))(*pout)
        check(lib().tvb_matvec_host_batch(*self._dims(), self._mh.ctypes.data, n, ctypes.cast(hu, ctypes.c_void_p),
                                          ctypes.cast(ho, ctypes.c_void_p), ptr(self.occ_d), ptr(self.nflags), flags,
                                          int(slabs), ptr(self._host_bws), self._host_bws.numel(), stream_ptr()),
              "matvec (host buffer batch)")
        return outs

    def apply_subset(self, u, elems):
        """K @ u using only the listed elements (reference ``fea.py:67-76``)."""
        torch = _torch()
        u_d, np_in = to_device(u, self.n_dofs, "displacement vector")
        el = torch.as_tensor(np.ascontiguousarray(np.asarray(elems, dtype=np.int64).ravel()), device="cuda")
        out = torch.zeros(self.n_dofs, dtype=torch.float64, device="cuda")
        ws = torch.empty(self.domain.n_elems * 12 + 16, dtype=torch.uint8, device="cuda")
        check(lib().tvb_matvec_subset(*self._dims(), self._mh.ctypes.data, ptr(u_d), ptr(out), ptr(el), el.numel(),
                                      ptr(self.occ_d), ptr(ws), ws.numel(), stream_ptr()), "matvec subset")
        if self.dirichlet.size:
            out.index_fill_(0, self.fixed_d, 0.0)
        return to_host_if(out, np_in)

    def diagonal_device(self):
        torch = _torch()
        if self._diag_d is None:
            d = torch.empty(self.n_dofs, dtype=torch.float64, device="cuda")
            check(lib().tvb_diag(*self._dims(), ptr(self.occ_d), ptr(self.nflags), self._kdiag.ctypes.data, ptr(d), 0,
                                 None, None, stream_ptr()), "diagonal")
            self._diag_d = d
        return self._diag_d

    def diagonal(self) -> np.ndarray:
        """diag(K), assembly-free; cached (reference ``fea.py:78-85``)."""
        if self._diag is None:
            self._diag = self.diagonal_device().cpu().numpy()
        return self._diag

    def pcg_workspace(self, block: int, nrhs: int = 1):
        torch = _torch()
        key = (int(block), int(nrhs))
        if key not in self._pcg_ws:
            n = lib().tvb_pcg_batch_ws_bytes(*self._dims(), int(block), int(nrhs))
            self._pcg_ws[key] = torch.empty(n, dtype=torch.uint8, device="cuda")
        return self._pcg_ws[key]


@dataclass
class SolveResult:
    u: object
    iterations: int
    residual: float


class DeflationSpace:
    """Per-agglomerate rigid-body deflation basis (reference ``fea.py:95-211``).

    The basis W is implicit on the device (per-block centroid + 6x6
    orthonormalising transform); ``W`` / ``block_elems`` are materialised on
    the host only when accessed (API compatibility).
    """

    def __init__(self, domain: Domain, topology: Topology, dirichlet=(), block: int = 4, coarse: str = "auto"):
        if block < 2:
            raise ValueError(f"agglomerate side must be >= 2, got {block}")
        if coarse not in ("auto", "dense", "nd"):
            raise ValueError(f"coarse must be auto|dense|nd, got {coarse!r}")
        torch = _torch()
        self.coarse = coarse
        self.domain = domain
        self.topology = topology
        self.block = int(block)
        self.dirichlet = np.asarray(np.unique(np.asarray(dirichlet, dtype=np.int64)), dtype=np.int64)
        b = self.block
        self.grid = ((domain.nx - 1) // b + 1, (domain.ny - 1) // b + 1, (domain.nz - 1) // b + 1)
        self.n_blocks = self.grid[0] * self.grid[1] * self.grid[2]
        self.occ_d = torch.from_numpy(np.ascontiguousarray(topology.occupancy, dtype=np.float64)).cuda()
        self.nflags, _ = _node_flags(domain, self.occ_d, self.dirichlet)
        nb = self.n_blocks
        self.cen = torch.empty(3 * nb, dtype=torch.float64, device="cuda")
        self.S = torch.empty(36 * nb, dtype=torch.float64, device="cuda")
        self.keep = torch.empty(nb, dtype=torch.int32, device="cuda")
        check(lib().tvb_defl_build(domain.nx, domain.ny, domain.nz, b, domain.h, ptr(self.occ_d), ptr(self.nflags),
                                   ptr(self.cen), ptr(self.S), ptr(self.keep), stream_ptr()), "deflation basis")
        keep = self.keep.cpu().numpy()
        self.kept_mask = ((keep[:, None] >> np.arange(6)[None, :]) & 1).astype(bool)
        self.n_vectors = int(self.kept_mask.sum())
        self._prepared_for = None
        self.Es = None
        self.coarse_inv = None
        self.nd = None
        self._W = None

    # --- coarse operator -----------------------------------------------------
    def prepare(self, op: StiffnessOperator) -> None:
        """Assemble E = W^T K W on the device and factor it (reference
        ``fea.py:185-206``)."""
        if self.n_vectors == 0 or self._prepared_for is op:
            return
        torch = _torch()
        d = self.domain
        nb = self.n_blocks
        self.Es = torch.empty(nb * 27 * 36, dtype=torch.float64, device="cuda")
        nws = lib().tvb_coarse_assemble_ws_bytes(d.nx, d.ny, d.nz, self.block)
        ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
        check(lib().tvb_coarse_assemble(d.nx, d.ny, d.nz, self.block, d.h, op.mh.ctypes.data, ptr(op.occ_d),
                                        ptr(self.nflags), ptr(self.cen), ptr(self.S), ptr(self.keep), ptr(self.Es),
                                        ptr(ws), nws, stream_ptr()), "coarse operator")
        del ws
        nc = 6 * nb
        kind = self.coarse
        if kind == "auto":
            kind = "dense" if nc <= DENSE_COARSE_AUTO_LIMIT else "nd"
        self.coarse_inv = None
        self.nd = None
        if kind == "nd":
            from .coarse import NDCoarseSolver

            try:
                self.nd = NDCoarseSolver(self.grid, self.Es)
            except np.linalg.LinAlgError:
                if nc > DENSE_COARSE_MAX:
                    raise
                log.warning("deflation coarse matrix not SPD; falling back to pseudo-inverse")
                kind = "dense"
        if kind == "dense":
            if nc > DENSE_COARSE_MAX:
                raise ValueError(f"dense coarse inverse limited to {DENSE_COARSE_MAX} DOFs, got {nc}")
            from .coarse import dense_inverse

            try:  # E swept on the device as one front (csrc/dense.cu)
                self.coarse_inv = dense_inverse(self.grid, self.Es)
            except np.linalg.LinAlgError:
                # the reference's fallback (fea.py:201-205): pseudo-inverse of the symmetrised E
                log.warning("deflation coarse matrix not SPD; falling back to pseudo-inverse")
                E = torch.empty(nc * nc, dtype=torch.float64, device="cuda")
                check(lib().tvb_coarse_dense(d.nx, d.ny, d.nz, self.block, ptr(self.Es), ptr(E), stream_ptr()),
                      "coarse dense")
                E = E.view(nc, nc)
                self.coarse_inv = torch.linalg.pinv(0.5 * (E + E.T), hermitian=True).contiguous()
                del E
        self._prepared_for = op

    def coarse_solve(self, rhs):
        """E^-1 rhs in this space's (kept-column) coarse basis."""
        torch = _torch()
        if self.coarse_inv is None and self.nd is None:
            raise RuntimeError("DeflationSpace.prepare(op) must run first")
        np_in = not isinstance(rhs, torch.Tensor)
        r = torch.as_tensor(np.asarray(rhs, dtype=np.float64) if np_in else rhs, device="cuda", dtype=torch.float64)
        mask = torch.from_numpy(self.kept_mask.ravel()).cuda()
        full = torch.zeros(6 * self.n_blocks, dtype=torch.float64, device="cuda")
        full[mask] = r
        if self.nd is not None:
            ndi = torch.from_numpy(self.nd.nd_index()).cuda()
            y = torch.empty_like(full)
            y[ndi] = full                                   # natural -> ND order
            sol = self.nd.solve_device(y, torch.empty_like(full))[ndi]
        else:
            sol = self.coarse_inv @ full
        return to_host_if(sol[mask], np_in)

    def project_device(self, v):
        """W E^-1 W^T v on device vectors (restriction, exact coarse solve,
        prolongation kernels); the deflated-PCG projection of the reference's
        ``project_out`` (fea.py:258-259) when v = K z."""
        torch = _torch()
        if self.coarse_inv is None and self.nd is None:
            raise RuntimeError("DeflationSpace.prepare(op) must run first")
        d = self.domain
        nc = 6 * self.n_blocks
        yc = torch.empty(nc, dtype=torch.float64, device="cuda")
        check(lib().tvb_restrict(d.nx, d.ny, d.nz, self.block, d.h, ptr(self.nflags), ptr(self.cen), ptr(self.S),
                                 ptr(self.keep), ptr(v), ptr(yc), stream_ptr()), "restrict")
        if self.nd is not None:
            ndi = torch.from_numpy(self.nd.nd_index()).cuda()
            y = torch.empty_like(yc)
            y[ndi] = yc
            mu = self.nd.solve_device(y, torch.empty_like(yc))[ndi].contiguous()
        else:
            mu = (self.coarse_inv @ yc).contiguous()
        out = torch.empty_like(v)
        ws = torch.empty(nc, dtype=torch.float64, device="cuda")
        check(lib().tvb_prolong(d.nx, d.ny, d.nz, self.block, d.h, ptr(self.nflags), ptr(self.cen), ptr(self.S),
                                ptr(self.keep), ptr(mu), ptr(out), ptr(ws), stream_ptr()), "prolong")
        return out

    # --- host views (compatibility / tests) ------------------------------------
    @property
    def W(self):
        """scipy CSC (n_dofs, n_vectors) view of the basis (host, lazily built)."""
        if self.n_vectors == 0:
            return None
        if self._W is None:
            self._W = _materialize_w(self)
        return self._W

    @property
    def block_elems(self):
        d, b = self.domain, self.block
        ix, iy, iz = d.elem_grid_coords()
        out = []
        for B in range(self.n_blocks):
            nk = int(self.kept_mask[B].sum())
            if nk == 0:
                continue
            bx, by, bz = B % self.grid[0], (B // self.grid[0]) % self.grid[1], B // (self.grid[0] * self.grid[1])
            lo = [max(b * c - 1, 0) for c in (bx, by, bz)]
            hi = [min(b * c + b, n - 1) for c, n in zip((bx, by, bz), (d.nx, d.ny, d.nz))]
            near = np.flatnonzero((ix >= lo[0]) & (ix <= hi[0]) & (iy >= lo[1]) & (iy <= hi[1]) & (iz >= lo[2])
                                  & (iz <= hi[2]))
            out.extend([near] * nk)
        return out


def _materialize_w(space: DeflationSpace):
    import scipy.sparse

    d, b = space.domain, space.block
    cen = space.cen.cpu().numpy().reshape(-1, 3)
    S = space.S.cpu().numpy().reshape(-1, 6, 6).transpose(0, 2, 1)  # S[B][j][i] -> [B][i][j]
    flags = space.nflags.cpu().numpy()
    rows, cols, vals = [], [], []
    col0 = 0
    for B in range(space.n_blocks):
        kept = np.flatnonzero(space.kept_mask[B])
        if kept.size == 0:
            continue
        bx, by, bz = B % space.grid[0], (B // space.grid[0]) % space.grid[1], B // (space.grid[0] * space.grid[1])
        xs = np.arange(b * bx, min(b * bx + b, d.nx) + 1)
        ys = np.arange(b * by, min(b * by + b, d.ny) + 1)
        zs = np.arange(b * bz, min(b * bz + b, d.nz) + 1)
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        nodes = (X + (d.nx + 1) * (Y + (d.ny + 1) * Z)).ravel()
        st = (flags[nodes] & 8) != 0
        nodes = nodes[st]
        rel = d.h * (np.stack([X.ravel()[st] - b * bx, Y.ravel()[st] - b * by, Z.ravel()[st] - b * bz], 1) - cen[B])
        raw = np.zeros((3 * nodes.size, 6))
        raw[0::3, 0] = raw[1::3, 1] = raw[2::3, 2] = 1.0
        raw[1::3, 3], raw[2::3, 3] = -rel[:, 2], rel[:, 1]
        raw[0::3, 4], raw[2::3, 4] = rel[:, 2], -rel[:, 0]
        raw[0::3, 5], raw[1::3, 5] = -rel[:, 1], rel[:, 0]
        fx = ((flags[nodes][:, None] >> np.arange(3)) & 1).astype(bool).ravel()
        raw[fx] = 0.0
        q = raw @ S[B][:, kept]
        dofs = (3 * nodes[:, None] + np.arange(3)).ravel()
        for k in range(kept.size):
            rows.append(dofs)
            cols.append(np.full(dofs.size, col0 + k))
            vals.append(q[:, k])
        col0 += kept.size
    return scipy.sparse.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                   shape=(d.n_dofs, col0))


def build_deflation(domain: Domain, topology: Topology, dirichlet=(), block: int = 4,
                    coarse: str = "auto") -> DeflationSpace:
    return DeflationSpace(domain, topology, dirichlet, block, coarse)


def default_max_iters(n_dofs: int) -> int:
    return max(200, int(10 * math.sqrt(n_dofs)))


#: deflated search-direction recurrence: "stabilized" (the default: projects
#: z + beta p, equal to the reference's in exact arithmetic, re-imposes
#: W^T A p = 0 every iteration) or "reference" (fea.py:289 verbatim). Both
#: match the reference's iterates equally closely where it is well behaved
#: (tests/test_gpu_large_parity.py); at tol ~1e-12 the reference's recurrence
#: can diverge depending on rounding alone (the reference itself on the C1
#: geometry with a face load; this library on a 24x12x12 Bernoulli case the
#: reference happens to solve), the stabilised one converges.
#: TVB_PROJECTION overrides the default.
PROJECTIONS = {"reference": 0, "stabilized": 1}


def _projection(projection: str | None) -> int:
    name = projection or os.environ.get("TVB_PROJECTION", "stabilized")
    if name not in PROJECTIONS:
        raise ValueError(f"projection must be one of {sorted(PROJECTIONS)}, got {name!r}")
    return PROJECTIONS[name]


def solve_static(op: StiffnessOperator, f, tol: float = 1.0e-8, max_iters: int | None = None,
                 deflation: DeflationSpace | None = None, apply_op=None, diag=None,
                 check_every: int = 8, projection: str | None = None) -> SolveResult:
    """Solve K u = f to a relative residual on the free DOFs (reference
    ``topovox/fea.py:218-299``): Jacobi PCG, deflated when ``deflation``
    carries vectors, run entirely on the device. ``projection``: see
    ``PROJECTIONS``."""
    torch = _torch()
    if not 0.0 < tol <= 1.0e-2:
        raise ValueError(f"tolerance must lie in (0, 1e-2], got {tol}")
    f_d, np_in = to_device(f, op.n_dofs, "force vector")
    if not bool(torch.isfinite(f_d).all()):
        raise ValueError("force vector is not finite")
    if max_iters is None:
        max_iters = default_max_iters(op.n_dofs)
    if apply_op is not None or diag is not None:
        defl = deflation if (deflation is not None and deflation.n_vectors > 0) else None
        res = _solve_generic(op, f_d, tol, max_iters, apply_op, diag, defl)
        return SolveResult(to_host_if(res.u, np_in), res.iterations, res.residual)
    defl = deflation if (deflation is not None and deflation.n_vectors > 0) else None
    if defl is not None:
        defl.prepare(op)
    x = torch.empty(op.n_dofs, dtype=torch.float64, device="cuda")
    ws = op.pcg_workspace(defl.block if defl is not None else 0)
    desc = _pcg_desc(op, defl, tol, max_iters, check_every, ws, projection)
    desc.d_f, desc.d_x = ptr(f_d), ptr(x)
    st = lib().tvb_pcg_solve(ctypes.byref(desc), stream_ptr())
    if st == STATUS_NO_CONVERGENCE:
        raise NoConvergence(f"CG did not reach {tol:g} in {max_iters} iterations (residual {desc.residual:.3e})",
                            residual=desc.residual, iterations=max_iters, u=to_host_if(x, np_in))
    if st != 0:
        raise_for_status(st, "solve_static", _lib.last_error())
    return SolveResult(to_host_if(x, np_in), int(desc.iterations), float(desc.residual))


def _pcg_desc(op: StiffnessOperator, defl, tol: float, max_iters: int, check_every: int, ws, projection=None):
    """tvb_pcg_desc of the operator / deflation space (RHS pointers unset)."""
    d = op.domain
    desc = _lib.PcgDesc()
    desc.nx, desc.ny, desc.nz, desc.h = d.nx, d.ny, d.nz, d.h
    desc.h_mh45 = op.mh.ctypes.data
    desc.h_kdiag3 = op._kdiag.ctypes.data
    desc.d_occ, desc.d_nflags = ptr(op.occ_d), ptr(op.nflags)
    desc.d_ws, desc.ws_bytes = ptr(ws), ws.numel()
    desc.tol, desc.max_iters, desc.check_every = float(tol), int(max_iters), int(check_every)
    desc.projection = _projection(projection)
    if defl is not None:
        desc.block = defl.block
        desc.d_cen, desc.d_S, desc.d_keep = ptr(defl.cen), ptr(defl.S), ptr(defl.keep)
        desc.d_defl_nflags = ptr(defl.nflags)  # W is the space's (its Dirichlet set / topology)
        if defl.nd is not None:
            desc.coarse_kind = 1
            desc.coarse_nd = ctypes.pointer(defl.nd.desc)
        else:
            desc.d_coarse = ptr(defl.coarse_inv)
            desc.coarse_kind = 0
    return desc


#: right-hand sides per batched device solve (solver.cuh kPcgMaxRhs)
MAX_BATCH_RHS = 8


def solve_static_batch(op: StiffnessOperator, forces, tol: float = 1.0e-8, max_iters: int | None = None,
                       deflation: DeflationSpace | None = None, check_every: int = 8,
                       projection: str | None = None) -> list:
    """Multi-RHS batching: solve K u_c = f_c for several load
    vectors against ONE operator and deflation space -- every load case and
    adjoint of a topology. Each RHS follows ``solve_static`` exactly (own
    stopping test, iteration count and errors; its result is bitwise the one
    ``solve_static`` returns for it alone); per iteration the coarse solve
    reads the factor once for all RHS and one CUDA graph launch / host check
    serves them all.

    ``forces``: a sequence of vectors or an (m, n_dofs) array / tensor.
    Returns a list of ``SolveResult``. Raises like ``solve_static`` for the
    first failing RHS (``NoConvergence`` carries that RHS's residual)."""
    torch = _torch()
    if not 0.0 < tol <= 1.0e-2:
        raise ValueError(f"tolerance must lie in (0, 1e-2], got {tol}")
    if isinstance(forces, torch.Tensor) or isinstance(forces, np.ndarray):
        if forces.ndim != 2:
            raise DimensionMismatch(f"force batch must be 2-D (m, n_dofs), got shape {tuple(forces.shape)}")
        forces = [forces[i] for i in range(forces.shape[0])]
    forces = list(forces)
    if not forces:
        return []
    if max_iters is None:
        max_iters = default_max_iters(op.n_dofs)
    fds, np_flags = [], []
    for i, f in enumerate(forces):
        f_d, np_in = to_device(f, op.n_dofs, f"force vector {i}")
        if not bool(torch.isfinite(f_d).all()):
            raise ValueError(f"force vector {i} is not finite")
        fds.append(f_d.contiguous())
        np_flags.append(np_in)
    defl = deflation if (deflation is not None and deflation.n_vectors > 0) else None
    if defl is not None:
        defl.prepare(op)
    out = []
    for g0 in range(0, len(fds), MAX_BATCH_RHS):
        grp = fds[g0:g0 + MAX_BATCH_RHS]
        m = len(grp)
        xs = [torch.empty(op.n_dofs, dtype=torch.float64, device="cuda") for _ in range(m)]
        ws = op.pcg_workspace(defl.block if defl is not None else 0, m)
        desc = _pcg_desc(op, defl, tol, max_iters, check_every, ws, projection)
        fptr = (ctypes.c_void_p * m)(*[ptr(t) for t in grp])
        xptr = (ctypes.c_void_p * m)(*[ptr(t) for t in xs])
        its = (ctypes.c_int * m)()
        res = (ctypes.c_double * m)()
        sts = (ctypes.c_int * m)()
        st = lib().tvb_pcg_solve_batch(ctypes.byref(desc), m, ctypes.cast(fptr, ctypes.c_void_p),
                                       ctypes.cast(xptr, ctypes.c_void_p), ctypes.cast(its, ctypes.c_void_p),
                                       ctypes.cast(res, ctypes.c_void_p), ctypes.cast(sts, ctypes.c_void_p),
                                       stream_ptr())
        # The call's own status is authoritative: a failure before or after the
        # per-RHS loop (bad problem, workspace, CUDA / graph error) leaves the
        # per-RHS array meaningless, so it is never read as success.
        if st not in (0, STATUS_NO_CONVERGENCE):
            raise_for_status(st, "solve_static_batch", _lib.last_error())
        for c in range(m):
            if sts[c] == STATUS_NO_CONVERGENCE:
                raise NoConvergence(f"CG did not reach {tol:g} in {max_iters} iterations for right-hand side "
                                    f"{g0 + c} (residual {res[c]:.3e})", residual=res[c], iterations=max_iters,
                                    u=to_host_if(xs[c], np_flags[g0 + c]))
            if sts[c] != 0:
                raise_for_status(sts[c], f"solve_static_batch (right-hand side {g0 + c})", _lib.last_error())
        if st == STATUS_NO_CONVERGENCE:
            raise NoConvergence(f"CG did not reach {tol:g} in {max_iters} iterations", iterations=max_iters)
        out.extend(SolveResult(to_host_if(xs[c], np_flags[g0 + c]), int(its[c]), float(res[c])) for c in range(m))
    return out


def _solve_generic(op, f_d, tol, max_iters, apply_op, diag, defl=None):
    """PCG with a caller-supplied operator / diagonal (reference hook used for
    shifted solves, fea.py:218-299 with ``apply_op`` / ``diag``). Vector
    algebra on the device. As in the reference, a deflation space still
    deflates: it is prepared for ``op`` and projects with op's K (KW of
    ``op``, fea.py:256-262), whatever ``apply_op`` is."""
    torch = _torch()
    free = torch.from_numpy(op.free_mask).cuda()
    A = apply_op if apply_op is not None else (lambda v: op.apply_device(v))
    dd = diag if diag is not None else op.diagonal_device()
    dd = torch.as_tensor(dd, dtype=torch.float64, device="cuda")
    fnorm = float(torch.linalg.norm(f_d[free]))
    if fnorm == 0.0:
        return SolveResult(torch.zeros_like(f_d), 0, 0.0)
    if bool((dd[free] == 0.0).any()):
        raise SingularSystem("zero stiffness diagonal on a loaded free DOF")
    inv_d = torch.zeros_like(f_d)
    inv_d[free] = 1.0 / dd[free]
    if defl is not None:
        defl.prepare(op)
        x = defl.project_device(f_d.contiguous())  # W E^-1 W^T f
        r = f_d - torch.as_tensor(A(x), device="cuda", dtype=torch.float64)

        def project_out(v):
            return defl.project_device(op.apply_device(v.contiguous()))
    else:
        x = torch.zeros_like(f_d)
        r = f_d.clone()
    r[~free] = 0.0
    res = float(torch.linalg.norm(r)) / fnorm
    if res <= tol:
        return SolveResult(x, 0, res)
    z = inv_d * r
    p = z - project_out(z) if defl is not None else z.clone()
    rz = float(r @ z)
    for it in range(1, max_iters + 1):
        q = torch.as_tensor(A(p), device="cuda", dtype=torch.float64)
        alpha = rz / float(p @ q)
        x += alpha * p
        r -= alpha * q
        res = float(torch.linalg.norm(r)) / fnorm
        if res <= tol:
            break
        z = inv_d * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        if defl is not None:
            p = p - project_out(z)
        rz = rz_new
    else:
        raise NoConvergence(f"CG did not reach {tol:g} in {max_iters} iterations (residual {res:.3e})",
                            residual=res, iterations=max_iters)
    x[~free] = 0.0
    return SolveResult(x, it, res)


def dense_stiffness(op: StiffnessOperator) -> np.ndarray:
    """Assembled raw K (small systems; reference ``fea.py:324-332``), built by
    applying the device operator to unit vectors."""
    torch = _torch()
    if op.n_dofs > DENSE_ORACLE_DOF_LIMIT:
        raise ValueError(f"dense oracle limited to {DENSE_ORACLE_DOF_LIMIT} DOFs")
    eye = torch.eye(op.n_dofs, dtype=torch.float64, device="cuda")
    cols = [op.apply_device(eye[j].contiguous(), raw=True) for j in range(op.n_dofs)]
    return torch.stack(cols, dim=1).cpu().numpy()


def dense_solve(op: StiffnessOperator, f) -> np.ndarray:
    """Direct solve on the free DOFs via Cholesky (reference ``fea.py:335-342``)."""
    torch = _torch()
    K = torch.from_numpy(dense_stiffness(op)).cuda()
    free = torch.from_numpy(op.free_mask).cuda()
    fd = torch.as_tensor(np.asarray(f, dtype=np.float64), device="cuda")
    Kf = K[free][:, free]
    L = torch.linalg.cholesky(Kf)
    u = torch.zeros(op.n_dofs, dtype=torch.float64, device="cuda")
    u[free] = torch.cholesky_solve(fd[free].unsqueeze(1), L).squeeze(1)
    return u.cpu().numpy()


def batch_element_state(op: StiffnessOperator, u):
    """Centroid strain / stress / von Mises per element (reference
    ``fea.py:302-309``), computed by the device kernel."""
    from .sensitivity import element_state_device

    u_d, np_in = to_device(u, op.n_dofs, "displacement vector")
    strains, stresses, vm = element_state_device(op, u_d)
    if np_in:
        return strains.cpu().numpy(), stresses.cpu().numpy(), vm.cpu().numpy()
    return strains, stresses, vm


def element_state(op: StiffnessOperator, u, e: int):
    """(strain tensor, stress tensor, von Mises) of element ``e``."""
    from .elements import voigt_to_tensor

    strains, stresses, vm = batch_element_state(op, np.asarray(u.cpu() if hasattr(u, "cpu") else u))
    s = strains[e]
    eps = voigt_to_tensor(s)
    eps[0, 1] = eps[1, 0] = s[3] / 2.0
    eps[1, 2] = eps[2, 1] = s[4] / 2.0
    eps[0, 2] = eps[2, 0] = s[5] / 2.0
    return eps, voigt_to_tensor(stresses[e]), float(vm[e])
