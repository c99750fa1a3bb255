"""Sparse direct solver for the deflation coarse system E mu = y (a6/a7).

The reference factors E = W^T K W densely (``scipy.linalg.cho_factor``,
``topovox/fea.py:197-200``) and runs a dense ``cho_solve`` every CG iteration
(``fea.py:208-211``); at C4 that is a 1.15 GB factor and at C2(b) a 309 GB one
(SURVEY §0.4). E is a 27-point stencil of 6x6 blocks on the agglomerate grid,
so it is factored here by geometric nested dissection:

* symbolic (host, once per block grid): recursive bisection of the block box
  along its longest axis by one-block-thick separator planes down to small
  leaf boxes; for each tree node its separator S and update set U (the
  ancestor-separator blocks adjacent to the node's box);
* numeric (device, once per operator): multifrontal block-LDL^T. For each node
  in postorder the front F = [[F_SS, F_SU], [F_US, F_UU]] is assembled from the
  stencil and the children's update matrices, then
      Z = F_SS^-1,  G = F_US Z,  update = F_UU - G F_SU  (passed to the parent);
* solve (device, every CG iteration, hand-written kernels in coarse.cu):
      forward, leaves -> root:  f_S = y_S + sum(children), c_U = f_U - G f_S
      backward, root -> leaves: x_S = Z f_S - G^T x_U
  i.e. exactly one kernel per tree height and direction, reading G, G^T and Z
  once each. The exact coarse solve keeps the DPCG iterates identical (up to
  rounding) to the reference's dense Cholesky.

The dense per-front linear algebra of the factorisation uses torch on the
device (cuSOLVER/cuBLAS); it runs once per topology, not per iteration.
"""

from __future__ import annotations

import ctypes
import logging
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr, stream_ptr

log = logging.getLogger(__name__)

#: fronts larger than this (DOFs) get a separate assembly pass in the forward solve
SPLIT_FRONT = int(__import__("os").environ.get("TVB_ND_SPLIT_FRONT", "2048"))


@dataclass
class NDNode:
    sep: np.ndarray          # separator block ids (sorted)
    upd: np.ndarray          # update-set block ids (ordered as in the parent's front)
    children: list = field(default_factory=list)
    height: int = 0
    box: tuple = ()


def nested_dissection(mx: int, my: int, mz: int, leaf_max: int = 27) -> list[NDNode]:
    """Geometric ND of the mx x my x mz block grid; nodes in postorder."""
    nodes: list[NDNode] = []

    def bid(x, y, z):
        return x + mx * (y + my * z)

    def box_ids(x0, x1, y0, y1, z0, z1):
        zz, yy, xx = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
        return bid(xx, yy, zz).ravel()

    def adjacent(ids, box):
        x0, x1, y0, y1, z0, z1 = box
        x, y, z = ids % mx, (ids // mx) % my, ids // (mx * my)
        m = (x >= x0 - 1) & (x <= x1) & (y >= y0 - 1) & (y <= y1) & (z >= z0 - 1) & (z <= z1)
        return ids[m]

    def rec(box, front_above):
        x0, x1, y0, y1, z0, z1 = box
        ext = (x1 - x0, y1 - y0, z1 - z0)
        if min(ext) <= 0:
            return None
        upd = adjacent(front_above, box)
        if ext[0] * ext[1] * ext[2] <= leaf_max:
            node = NDNode(sep=np.sort(box_ids(*box)), upd=upd, box=box)
        else:
            ax = int(np.argmax(ext))
            lo, hi = box[2 * ax], box[2 * ax + 1]
            mid = (lo + hi) // 2
            sb, b1, b2 = list(box), list(box), list(box)
            sb[2 * ax], sb[2 * ax + 1] = mid, mid + 1
            b1[2 * ax + 1] = mid
            b2[2 * ax] = mid + 1
            sep = np.sort(box_ids(*sb))
            node = NDNode(sep=sep, upd=upd, box=box)
            here = np.concatenate([sep, upd])
            kids = [k for k in (rec(tuple(b1), here), rec(tuple(b2), here)) if k is not None]
            node.children = kids
            node.height = 1 + max(nodes[k].height for k in kids) if kids else 0
        nodes.append(node)
        return len(nodes) - 1

    rec((0, mx, 0, my, 0, mz), np.empty(0, dtype=np.int64))
    return nodes


class NDCoarseSolver:
    """Factor E (block stencil Es on the device) and hold the device data of
    the per-iteration solve kernels (see ``tvb_coarse_nd_*`` in the C-ABI)."""

    def __init__(self, grid: tuple[int, int, int], Es, leaf_max: int = 27, make_desc: bool = True):
        import torch

        mx, my, mz = grid
        self.grid = grid
        self.nb = mx * my * mz
        self.nodes = nested_dissection(mx, my, mz, leaf_max)
        nodes = self.nodes
        self.height = max(n.height for n in nodes)
        # ---- host index structures ------------------------------------
        s_blocks = [n.sep.size for n in nodes]
        u_blocks = [n.upd.size for n in nodes]
        s = np.array(s_blocks, dtype=np.int64) * 6
        u = np.array(u_blocks, dtype=np.int64) * 6
        self.s, self.u = s, u

        def dofs(blocks):
            return (6 * blocks[:, None] + np.arange(6)[None, :]).ravel().astype(np.int32)

        s_dof = [dofs(n.sep) for n in nodes]
        u_dof = [dofs(n.upd) for n in nodes]
        # child maps: child's U position -> parent's front position
        cmaps = []
        child_ptr = [0]
        child_list = []
        for n in nodes:
            pos = {int(b): i for i, b in enumerate(np.concatenate([n.sep, n.upd]))}
            for c in n.children:
                cb = nodes[c].upd
                m = np.array([pos[int(b)] for b in cb], dtype=np.int64)
                cmaps.append((6 * m[:, None] + np.arange(6)[None, :]).ravel().astype(np.int32))
                child_list.append(c)
            child_ptr.append(len(child_list))
        self._make = make_desc
        self._factor(torch, Es, nodes, s, u, s_dof, u_dof, cmaps, child_ptr, child_list)

    # ------------------------------------------------------------------
    def _factor(self, torch, Es, nodes, s, u, s_dof, u_dof, cmaps, child_ptr, child_list):
        mx, my, mz = self.grid
        dev = Es.device
        E6 = Es.view(self.nb, 27, 6, 6)
        upd_mats = {}
        G_list, Z_list = [], []
        cm_iter = 0
        for ni, n in enumerate(nodes):
            blocks = np.concatenate([n.sep, n.upd])
            ns, nu = n.sep.size, n.upd.size
            f = 6 * (ns + nu)
            F = torch.zeros((f, f), dtype=torch.float64, device=dev)
            # original entries E[S, S u U]: neighbour offsets of every separator block
            pos = -np.ones(self.nb, dtype=np.int64)
            pos[blocks] = np.arange(blocks.size)
            sb = n.sep
            x, y, z = sb % mx, (sb // mx) % my, sb // (mx * my)
            rows, cols, srcB, srcD = [], [], [], []
            for d in range(27):
                dx, dy, dz = d % 3 - 1, (d // 3) % 3 - 1, d // 9 - 1
                cx, cy, cz = x + dx, y + dy, z + dz
                ok = (cx >= 0) & (cx < mx) & (cy >= 0) & (cy < my) & (cz >= 0) & (cz < mz)
                cb = cx + mx * (cy + my * cz)
                pc = np.where(ok, pos[np.where(ok, cb, 0)], -1)
                keep = ok & (pc >= 0)
                rows.append(np.arange(ns)[keep])
                cols.append(pc[keep])
                srcB.append(sb[keep])
                srcD.append(np.full(int(keep.sum()), d))
            rows, cols = np.concatenate(rows), np.concatenate(cols)
            srcB, srcD = np.concatenate(srcB), np.concatenate(srcD)
            blk = E6[torch.from_numpy(srcB).to(dev), torch.from_numpy(srcD).to(dev)]  # (k, 6, 6)
            r6 = torch.from_numpy(6 * rows).to(dev)[:, None, None] + torch.arange(6, device=dev)[None, :, None]
            c6 = torch.from_numpy(6 * cols).to(dev)[:, None, None] + torch.arange(6, device=dev)[None, None, :]
            F[r6.expand(-1, 6, 6), c6.expand(-1, 6, 6)] = blk
            # U x S part = transpose of S x U (entries with a column in U)
            inU = cols >= ns
            if inU.any():
                F[c6[inU].expand(-1, 6, 6).transpose(1, 2), r6[inU].expand(-1, 6, 6).transpose(1, 2)] = \
                    blk[torch.from_numpy(inU).to(dev)].transpose(1, 2)
            # extend-add children's update matrices (fixed order: deterministic)
            for c in n.children:
                m = torch.from_numpy(cmaps[cm_iter].astype(np.int64)).to(dev)
                cm_iter += 1
                Uc = upd_mats.pop(c)
                F[m[:, None], m[None, :]] += Uc
            S = 6 * ns
            Fss = 0.5 * (F[:S, :S] + F[:S, :S].T)
            L, info = torch.linalg.cholesky_ex(Fss)
            if int(info.item()) != 0:
                raise np.linalg.LinAlgError(f"coarse front {ni} not SPD")
            Z = torch.cholesky_inverse(L)
            G = F[S:, :S] @ Z
            if nu:
                upd_mats[ni] = F[S:, S:] - G @ F[:S, S:]
            Z_list.append(Z.contiguous())
            G_list.append(G.contiguous())
            del F
        self._pack(torch, dev, G_list, Z_list, s, u, s_dof, u_dof, cmaps, child_ptr, child_list)

    def _pack(self, torch, dev, G_list, Z_list, s, u, s_dof, u_dof, cmaps, child_ptr, child_list):
        nn = len(self.nodes)
        g_off = np.zeros(nn + 1, dtype=np.int64)
        z_off = np.zeros(nn + 1, dtype=np.int64)
        g_off[1:] = np.cumsum(s * u)
        z_off[1:] = np.cumsum(s * s)
        # G, G^T and Z live in ONE allocation so the solver can pin it in L2
        # with a single access-policy window (tvb_pcg_solve, coarse_kind 1).
        ng, nz = int(g_off[-1]), int(z_off[-1])
        self.factor = torch.empty(2 * ng + nz + 2, dtype=torch.float64, device=dev)
        self.G = self.factor[:ng + 1]
        self.Gt = self.factor[ng + 1:2 * ng + 2]
        self.Z = self.factor[2 * ng + 2:]
        if ng:
            self.G[:ng] = torch.cat([g.reshape(-1) for g in G_list])
            self.Gt[:ng] = torch.cat([g.T.contiguous().reshape(-1) for g in G_list])
        self.Z[:] = torch.cat([z.reshape(-1) for z in Z_list])
        sd_off = np.zeros(nn + 1, dtype=np.int64)
        ud_off = np.zeros(nn + 1, dtype=np.int64)
        sd_off[1:] = np.cumsum(s)
        ud_off[1:] = np.cumsum(u)
        self.s_dof = torch.from_numpy(np.concatenate(s_dof)).to(dev)
        self.u_dof = torch.from_numpy(np.concatenate(u_dof + [np.zeros(1, np.int32)])).to(dev)
        cm_off = np.zeros(len(cmaps) + 1, dtype=np.int64)
        cm_off[1:] = np.cumsum([c.size for c in cmaps])
        self.cmap = torch.from_numpy(np.concatenate(cmaps + [np.zeros(1, np.int32)])).to(dev)
        # per-node meta (int64): s, u, g_off, z_off, sd_off, ud_off, child_begin, child_end
        meta = np.stack([s, u, g_off[:-1], z_off[:-1], sd_off[:-1], ud_off[:-1],
                         np.array(child_ptr[:-1]), np.array(child_ptr[1:])], axis=1).astype(np.int64)
        self.meta = torch.from_numpy(np.ascontiguousarray(meta)).to(dev)
        # child list entries: (child node, cmap offset)
        ch = np.stack([np.array(child_list, dtype=np.int64), cm_off[:-1]], axis=1) if child_list else \
            np.zeros((1, 2), dtype=np.int64)
        self.children = torch.from_numpy(np.ascontiguousarray(ch)).to(dev)
        # per-node scratch: f_S (s) and c_U (u); offsets sd_off / ud_off
        self.fS = torch.zeros(int(sd_off[-1]) + 1, dtype=torch.float64, device=dev)
        self.cU = torch.zeros(int(ud_off[-1]) + 1, dtype=torch.float64, device=dev)
        # work items per height: (node, row0, row1); forward rows = u, backward rows = s.
        # 8 rows = one row per warp: longer chunks (to amortise the per-item
        # front assembly) measured slower at C2(b), C4 and C5 (less parallelism).
        def rows_per_item(front):
            return 8

        fwd, bwd, fptr, bptr = [], [], [0], [0]
        heights = np.array([n.height for n in self.nodes])
        for h in range(self.height + 1):
            for ni in np.flatnonzero(heights == h):
                nr, step = int(u[ni]), rows_per_item(int(s[ni] + u[ni]))
                for r0 in range(0, max(nr, 1), step):
                    fwd.append((ni, r0, min(nr, r0 + step)))
            fptr.append(len(fwd))
        for h in range(self.height, -1, -1):
            for ni in np.flatnonzero(heights == h):
                nr, step = int(s[ni]), rows_per_item(int(s[ni] + u[ni]))
                for r0 in range(0, nr, step):
                    bwd.append((ni, r0, min(nr, r0 + step)))
            bptr.append(len(bwd))
        self.fwd_items = torch.from_numpy(np.array(fwd, dtype=np.int32).reshape(-1, 3)).to(dev)
        self.bwd_items = torch.from_numpy(np.array(bwd, dtype=np.int32).reshape(-1, 3)).to(dev)
        self.fwd_ptr = np.array(fptr, dtype=np.int64)
        self.bwd_ptr = np.array(bptr, dtype=np.int64)
        self.max_front = int((s + u).max())
        self.max_sep = int(s.max())
        # heights whose largest front exceeds SPLIT_FRONT use a separate
        # per-node assembly launch (the fused item would re-assemble the whole
        # front for every 8-row chunk)
        self.split = np.array([int(max(int(s[i] + u[i]) for i in np.flatnonzero(heights == h)) > SPLIT_FRONT)
                               for h in range(self.height + 1)], dtype=np.int32)
        asm, aptr = [], [0]
        for h in range(self.height + 1):
            asm.extend(np.flatnonzero(heights == h).tolist())
            aptr.append(len(asm))
        self.asm_nodes = torch.from_numpy(np.array(asm, dtype=np.int32)).to(dev)
        self.asm_ptr = np.array(aptr, dtype=np.int64)
        self.bytes = self.factor.numel() * 8
        self.desc = self._make_desc() if self._make else None

    def _make_desc(self):
        from ._lib import CoarseND

        d = CoarseND()
        d.n_nodes = len(self.nodes)
        d.height = self.height
        d.max_front = self.max_front
        d.d_meta, d.d_children, d.d_cmap = ptr(self.meta), ptr(self.children), ptr(self.cmap)
        d.d_G, d.d_Gt, d.d_Z = ptr(self.G), ptr(self.Gt), ptr(self.Z)
        d.d_sdof, d.d_udof = ptr(self.s_dof), ptr(self.u_dof)
        d.d_fS, d.d_cU = ptr(self.fS), ptr(self.cU)
        d.d_fwd_items, d.d_bwd_items = ptr(self.fwd_items), ptr(self.bwd_items)
        d.d_factor, d.factor_bytes = ptr(self.factor), self.bytes
        self._fptr = (ctypes.c_longlong * len(self.fwd_ptr))(*self.fwd_ptr.tolist())
        self._bptr = (ctypes.c_longlong * len(self.bwd_ptr))(*self.bwd_ptr.tolist())
        d.h_fwd_ptr = ctypes.cast(self._fptr, ctypes.c_void_p)
        d.h_bwd_ptr = ctypes.cast(self._bptr, ctypes.c_void_p)
        self._split = (ctypes.c_int * len(self.split))(*self.split.tolist())
        self._aptr = (ctypes.c_longlong * len(self.asm_ptr))(*self.asm_ptr.tolist())
        d.h_split = ctypes.cast(self._split, ctypes.c_void_p)
        d.d_asm_nodes = ptr(self.asm_nodes)
        d.h_asm_ptr = ctypes.cast(self._aptr, ctypes.c_void_p)
        d.max_sep = self.max_sep
        return d

    def solve_device(self, y, x):
        """x = E^-1 y on device tensors (length 6 * n_blocks)."""
        check(lib().tvb_coarse_nd_solve(ctypes.byref(self.desc), ptr(y), ptr(x), stream_ptr()), "coarse solve")
        return x
