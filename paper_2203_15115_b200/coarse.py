"""Sparse direct solver for the deflation coarse system E mu = y (a6/a7).

The reference factors E = W^T K W densely (``scipy.linalg.cho_factor``,
``topovox/fea.py:197-200``) and runs a dense ``cho_solve`` every CG iteration
(``fea.py:208-211``); at C4 that is a 1.15 GB factor and at C2(b) a 309 GB one
(SURVEY §0.4). E is a 27-point stencil of 6x6 blocks on the agglomerate grid,
so it is factored here by geometric nested dissection:

* symbolic (host, once per block grid): recursive bisection of the block box
  along its longest axis by one-block-thick separator planes down to small
  leaf boxes; for each tree node its separator S and update set U (the
  ancestor-separator blocks adjacent to the node's box). Coarse DOFs are
  renumbered in ND order (separators by increasing tree height), so every
  separator is a contiguous DOF range and the top levels form the tail.
* numeric (device, once per operator): multifrontal elimination of the
  "bottom" nodes (height < H0): per node, in order of height (block sweep of
  the separator, csrc/dense.cu),
      Z = F_SS^-1,  G = F_US Z,  update = F_UU - G F_SU  (to the parent front);
  the "top" nodes (height >= H0, at most TOP_MAX DOFs in total) are not
  factored node by node: their Schur complement S_T (original entries among
  top DOFs plus the updates of the bottom nodes whose parent is a top node) is
  inverted densely. H0 = 0 gives a pure dense inverse (small coarse spaces).
* solve (device, every CG iteration, hand-written kernels in coarse.cu):
      forward, bottom heights 0..H0-1:  f_S = y_S + sum(children c|S), c_U = f_U - G f_S
      top:                              x_T = S_T^-1 (y_T + sum(children c|T))
      backward, heights H0-1..0:        x_S = [Z | -G^T] [f_S ; x_U]   (one stored s x (s+u) row block)
  Front vectors are gathered (each front position lists its children's
  update-vector entries), so assembly needs no barriers or atomics, and long
  matrix rows are split across several warps (the solve is latency-bound).
  The exact coarse solve keeps the DPCG iterates identical (up to rounding) to
  the reference's dense Cholesky.

The numeric factorisation (once per topology) runs in hand-written kernels
too (csrc/dense.cu, ``front_plan``): every front of a tree height is
assembled and swept in one launch sequence; no cuSOLVER / cuBLAS.
"""

from __future__ import annotations

import ctypes
import functools
import logging
import os
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr, stream_ptr

log = logging.getLogger(__name__)

#: fronts larger than this (DOFs) get a separate assembly pass in the forward solve
SPLIT_FRONT = int(os.environ.get("TVB_ND_SPLIT_FRONT", "2048"))
#: largest top set inverted densely (DOFs); the top tree levels it replaces
#: would otherwise cost two latency-bound launches each. 6200 admits the
#: 6144-DOF top separator of C2(b) (2247 -> 2200 us per iteration); C4 (3738)
#: and C5 (2400) are unchanged; 13000 was slower at C2(b), 2500 at C4 (+5 %)
TOP_MAX = int(os.environ.get("TVB_ND_TOP_MAX", "6200"))
#: largest leaf box of the dissection (blocks); default by size: 125 for
#: coarse systems up to FLOW_MIN_DOFS (fewer, fatter tree levels: C4 coarse
#: solve 86 -> 66 us in the iteration), 64 above (C5 / C2(b) are bandwidth-bound)
LEAF_MAX = int(os.environ["TVB_ND_LEAF"]) if os.environ.get("TVB_ND_LEAF") else None
#: schedule of the per-iteration solve: "1" = one persistent dataflow launch,
#: "0" = one launch per tree level, unset = by size: the level schedule is
#: 15-20 % faster for 12k coarse DOFs (C3/C4: inside a CUDA graph the per-level
#: launch gap is smaller than the dataflow items' counter traffic), the
#: dataflow one ~5 % faster from ~50k (C5: many items per level overlap)
FLOW = os.environ.get("TVB_ND_FLOW")
FLOW_MIN_DOFS = 48000
#: target warps per solve launch (148 SMs x 16)
WARPS_IN_FLIGHT = int(os.environ.get("TVB_ND_WARPS", "2368"))
#: dynamic shared memory per CTA (B200: 227 KB opt-in)
SMEM_MAX = 227 * 1024
#: right-hand sides per coarse-solve launch (coarse.cu kCoarseMaxCols); the
#: scratch vectors fS / cU / fT carry this many columns
MAX_COLS = 4
#: symmetric top inverse stored as its lower 64x64 tiles (half the bytes read
#: per solve; coarse.cu k_top_tiles / k_top_reduce); TVB_ND_PACK_TOP=0 -> dense rows
TOP_TILE = 64
PACK_TOP = os.environ.get("TVB_ND_PACK_TOP", "1") != "0"
#: resident 256-thread CTAs on the GPU (148 SMs x 8): one wave of solve items
CTA_SLOTS = int(os.environ.get("TVB_ND_SLOTS", "1184"))
#: index plans of the numeric factorisation, keyed by (block grid, leaf, top, device)
_PLAN_CACHE: dict = {}


def mode_step(mode: int) -> int:
    """rows per work item for a row schedule ``mode`` = WPR | RPW << 4."""
    return 8 * max(1, mode >> 4) // (mode & 15)


@dataclass
class NDNode:
    sep: np.ndarray          # separator block ids (sorted)
    upd: np.ndarray          # update-set block ids (ordered as in the parent's front)
    children: list = field(default_factory=list)
    height: int = 0
    box: tuple = ()
    parent: int = -1


@functools.lru_cache(maxsize=4)
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
        me = len(nodes) - 1
        for k in node.children:
            nodes[k].parent = me
        return me

    rec((0, mx, 0, my, 0, mz), np.empty(0, dtype=np.int64))
    return nodes


def _dofs(first_block_pos: np.ndarray) -> np.ndarray:
    return (6 * first_block_pos[:, None] + np.arange(6)[None, :]).ravel()


FT = 64  # tile order of the device front factorisation (csrc/dense.cuh kFT)


def _roundup(x: int, m: int = FT) -> int:
    return -(-int(x) // m) * m


def front_plan(torch, dev, specs):
    """Device records of the front factorisation (csrc/dense.cu).

    ``specs``: per front (natural block ids -- separator then update set --,
    separator DOFs s, update DOFs u, [(child front index, child update block
    ids in the child's order)], level). A child's update block list maps into
    the parent front through the parent's block positions. Returns the
    records, pool / scratch sizes and per-level launch lists."""
    n = len(specs)
    rec = np.zeros((n, 12), dtype=np.int64)
    blocks, children, gmap = [], [], []
    blk_off = gm_off = child_cnt = 0
    a_off = 0
    levels = {}
    for f, (blk, s, u, kids, level) in enumerate(specs):
        s_pad, nf = _roundup(s), _roundup(s) + _roundup(u)
        pos = {int(b): i for i, b in enumerate(blk)}
        rec[f, :10] = (a_off, nf, s, s_pad, u, blk_off, len(kids), child_cnt, 0, nf // FT)
        for cf, cupd in kids:
            g = -np.ones(s + u, dtype=np.int32)
            ppos = np.array([pos[int(b)] for b in cupd], dtype=np.int64)
            g[_dofs(ppos)] = np.arange(6 * cupd.size, dtype=np.int32)
            children.append((cf, gm_off))
            gmap.append(g)
            gm_off += g.size
            child_cnt += 1
        blocks.append(np.asarray(blk, dtype=np.int32))
        blk_off += len(blk)
        a_off += nf * nf
        levels.setdefault(level, []).append(f)
    out_levels, scratch = [], 0
    for level in sorted(levels):
        fr = levels[level]
        off = 0
        tiles, cols = [], []
        for f in fr:
            ntf = int(rec[f, 9])
            rec[f, 8] = off
            off += (1 + 2 * ntf) * FT * FT
            I, J = np.tril_indices(ntf)
            tiles.append(np.stack([np.full(I.size, f), I, J], axis=1))
            cols.append(np.stack([np.full(ntf, f), np.arange(ntf)], axis=1))
        scratch = max(scratch, off)
        tiles = np.concatenate(tiles).astype(np.int32)
        cols = np.concatenate(cols).astype(np.int32)
        out_levels.append({"fronts": torch.from_numpy(np.array(fr, dtype=np.int32)).to(dev), "n": len(fr),
                           "tiles": torch.from_numpy(np.ascontiguousarray(tiles)).to(dev), "nt": tiles.shape[0],
                           "cols": torch.from_numpy(np.ascontiguousarray(cols)).to(dev), "nc": cols.shape[0],
                           "steps": int(max(rec[f, 3] for f in fr)) // FT})
    return {"rec": torch.from_numpy(rec).to(dev),
            "blocks": torch.from_numpy(np.concatenate(blocks)).to(dev),
            "children": torch.from_numpy(np.array(children or [(0, 0)], dtype=np.int64)).to(dev),
            "gmap": torch.from_numpy(np.concatenate(gmap) if gmap else np.zeros(1, np.int32)).to(dev),
            "levels": out_levels, "pool": max(a_off, 1), "scratch": max(scratch, 1)}


def front_set(fp, pool, scratch, Es, grid, err):
    """tvb_front_set of a front plan; keeps its tensors alive on the struct."""
    from ._lib import FrontSet

    fs = FrontSet()
    fs.d_fronts, fs.d_pool, fs.d_scratch = ptr(fp["rec"]), ptr(pool), ptr(scratch)
    fs.d_blocks, fs.d_children, fs.d_gmap = ptr(fp["blocks"]), ptr(fp["children"]), ptr(fp["gmap"])
    fs.d_Es = ptr(Es)
    fs.mx, fs.my, fs.mz = grid
    fs.d_err = ptr(err)
    fs._keep = (fp, pool, scratch, Es, err)
    return fs


def run_front_levels(fs, levels):
    for L in levels:
        check(lib().tvb_front_level(ctypes.byref(fs), L["n"], ptr(L["fronts"]), L["nt"], ptr(L["tiles"]), L["nc"],
                                    ptr(L["cols"]), L["steps"], stream_ptr()), "front factorisation")


def dense_inverse(grid, Es):
    """E^-1 (natural block order, dense rows) of a small coarse space: E as one
    front with no update set, swept on the device. Raises LinAlgError when E
    is not SPD."""
    import torch

    nb = grid[0] * grid[1] * grid[2]
    fp = front_plan(torch, Es.device, [(np.arange(nb), 6 * nb, 0, [], 0)])
    pool = torch.empty(fp["pool"], dtype=torch.float64, device=Es.device)
    scratch = torch.empty(fp["scratch"], dtype=torch.float64, device=Es.device)
    err = torch.zeros(1, dtype=torch.int32, device=Es.device)
    fs = front_set(fp, pool, scratch, Es, grid, err)
    run_front_levels(fs, fp["levels"])
    out = torch.empty((6 * nb, 6 * nb), dtype=torch.float64, device=Es.device)
    check(lib().tvb_front_pack_top(ctypes.byref(fs), 0, 6 * nb, 0, ptr(out), stream_ptr()), "front pack")
    if int(err.item()) != 0:
        raise np.linalg.LinAlgError("coarse matrix not SPD")
    return out


class NDCoarseSolver:
    """Factor E (block stencil ``Es`` on the device, natural block order) and
    hold the device data of the per-iteration solve (``tvb_coarse_nd_solve``).
    Solve vectors are in ND order: natural block B sits at ND block ``perm[B]``."""

    def __init__(self, grid: tuple[int, int, int], Es, leaf_max: int | None = None, top_max: int | None = None,
                 make_desc: bool = True, numeric: bool = True):
        import torch

        mx, my, mz = grid
        self.grid = grid
        self.nb = nb = mx * my * mz
        if leaf_max is None:
            leaf_max = LEAF_MAX if LEAF_MAX is not None else (125 if 6 * nb <= FLOW_MIN_DOFS else 64)
        nodes = nested_dissection(mx, my, mz, leaf_max)
        self.nodes = nodes
        H = max(n.height for n in nodes)
        top_max = TOP_MAX if top_max is None else top_max
        self.leaf_max, self.top_max = leaf_max, top_max
        seps_by_h = np.zeros(H + 2, dtype=np.int64)
        for n in nodes:
            seps_by_h[n.height] += 6 * n.sep.size
        tail = np.cumsum(seps_by_h[::-1])[::-1]  # DOFs at heights >= h
        self.H0 = next(h for h in range(H + 2) if tail[h] <= top_max)
        order = sorted(range(len(nodes)), key=lambda i: (nodes[i].height, i))
        bottom = [i for i in order if nodes[i].height < self.H0]
        top = [i for i in order if nodes[i].height >= self.H0]
        self.n_bottom_levels = self.H0
        # ND block order: bottom separators by height, then the top set
        blk_order = np.concatenate([nodes[i].sep for i in bottom + top]).astype(np.int64)
        perm = np.empty(nb, dtype=np.int64)
        perm[blk_order] = np.arange(nb)
        self.perm_host = perm
        self.n_top = 6 * int(sum(nodes[i].sep.size for i in top))
        self.top_off = 6 * nb - self.n_top
        bidx = {ni: k for k, ni in enumerate(bottom)}
        # bottom-tree links for the dataflow schedule
        self._bparent = np.full(len(bottom), -1, dtype=np.int64)     # bottom parent (-1: top parent / root)
        self._bkids = [[] for _ in bottom]
        self._top_parent = np.zeros(len(bottom), dtype=bool)
        for k, ni in enumerate(bottom):
            p = nodes[ni].parent
            if p >= 0 and nodes[p].height < self.H0:
                self._bparent[k] = bidx[p]
                self._bkids[bidx[p]].append(k)
            elif p >= 0:
                self._top_parent[k] = True
        self.flow = FLOW != "0" if FLOW is not None else 6 * nb >= FLOW_MIN_DOFS
        #: packed symmetric top tiles (per-level schedule; the dataflow kernel reads dense rows)
        self.top_tiles = (self.n_top + TOP_TILE - 1) // TOP_TILE if (self.n_top and not self.flow and PACK_TOP) else 0
        self.bottom_nodes, self.top_nodes = bottom, top
        # numeric=False (CPU tests of the symbolic layout and the solve
        # schedule only): the factor arrays are allocated but left for the
        # caller to fill; nothing on the product path passes it
        self._factor(torch, Es, nodes, bottom, top, bidx, perm, numeric)
        self._make = make_desc
        self.desc = self._make_desc() if make_desc else None

    def _plan(self, torch, dev, nodes, bottom, top, perm):
        """Index plan (depends on the block grid only, so it is cached across
        topologies): the solve's per-node layout (separator / update sizes,
        update-DOF maps, gathered front positions) and the device front
        records of the numeric factorisation (``front_plan``)."""
        nb = self.nb
        P = {}
        bidx_of = {ni: k for k, ni in enumerate(bottom)}
        tblocks = np.concatenate([nodes[i].sep for i in top]).astype(np.int64) if top else np.zeros(0, np.int64)
        ud_off = {}
        ud_cursor = 0
        blk_cursor = 0
        s_list, u_list, sd_list, udof_list, gmaps = [], [], [], [], []
        for ni in bottom:
            n = nodes[ni]
            ns, nu = n.sep.size, n.upd.size
            front = np.concatenate([n.sep, n.upd])
            nf = 6 * front.size
            pos = -np.ones(nb, dtype=np.int64)
            pos[front] = np.arange(front.size)
            gm = -np.ones((nf, 2), dtype=np.int64)
            assert len(n.children) <= 2
            for k, c in enumerate(n.children):
                m = _dofs(pos[nodes[c].upd])
                gm[m, k] = ud_off[c] + np.arange(m.size)
            gmaps.append(gm.astype(np.int32).ravel())
            s_list.append(6 * ns)
            u_list.append(6 * nu)
            sd_list.append(6 * blk_cursor)
            ud_off[ni] = ud_cursor
            ud_cursor += 6 * nu
            blk_cursor += ns
            udof_list.append(_dofs(perm[n.upd]).astype(np.int32))
        t_pos, t_idx = [], []
        if self.n_top:
            tpos = -np.ones(nb, dtype=np.int64)
            tpos[tblocks] = perm[tblocks] - (nb - tblocks.size)
            for ni in bottom:
                if nodes[ni].parent >= 0 and nodes[nodes[ni].parent].height >= self.H0:
                    m = _dofs(tpos[nodes[ni].upd])
                    t_pos.append(m)
                    t_idx.append(ud_off[ni] + np.arange(m.size))
        P["pack"] = (np.array(s_list, np.int64), np.array(u_list, np.int64), np.array(sd_list, np.int64),
                     udof_list, gmaps, t_pos, t_idx, ud_cursor, [nodes[i].height for i in bottom])
        specs = []
        for ni in bottom:
            n = nodes[ni]
            specs.append((np.concatenate([n.sep, n.upd]), 6 * n.sep.size, 6 * n.upd.size,
                          [(bidx_of[c], nodes[c].upd) for c in n.children], n.height))
        if self.n_top:
            tchild = [(bidx_of[ni], nodes[ni].upd) for ni in bottom
                      if nodes[ni].parent >= 0 and nodes[nodes[ni].parent].height >= self.H0]
            specs.append((tblocks, self.n_top, 0, tchild, self.H0))
        P["front"] = front_plan(torch, dev, specs)
        return P

    def _factor(self, torch, Es, nodes, bottom, top, bidx, perm, numeric=True):
        """Numeric factorisation on the device (csrc/dense.cu, one launch
        sequence per tree height: assemble the fronts, sweep their separators),
        then the per-iteration layouts written by the pack kernels."""
        dev = Es.device
        key = (self.grid, self.leaf_max, self.top_max, str(dev))
        plan = _PLAN_CACHE.get(key)
        if plan is None:
            plan = self._plan(torch, dev, nodes, bottom, top, perm)
            _PLAN_CACHE.clear()  # keep one plan (one block grid per optimisation run)
            _PLAN_CACHE[key] = plan
        fp = plan["front"]
        if not numeric:
            self._pack(torch, dev, None, len(bottom), *plan["pack"])
            return
        pool = torch.empty(fp["pool"], dtype=torch.float64, device=dev)
        scratch = torch.empty(fp["scratch"], dtype=torch.float64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        fs = front_set(fp, pool, scratch, Es, self.grid, err)
        run_front_levels(fs, fp["levels"])
        self._pack(torch, dev, fs, len(bottom), *plan["pack"])
        if int(err.item()) != 0:  # one host sync for all fronts
            raise np.linalg.LinAlgError("coarse front not SPD")
        del pool, scratch

    @staticmethod
    def _wpr(rowlen: int, rows: int) -> int:
        """warps per matrix row (1, 2, 4, 8) for a launch of ``rows`` rows of
        length ``rowlen``: rows are split across warps only until the launch
        has enough warps in flight (small levels are latency-bound); every
        split costs one more shared-memory copy of the right-hand vector per
        row, which dominates once the level is bandwidth-bound."""
        forced = os.environ.get("TVB_ND_WPR")
        if forced:
            return int(forced)
        w = 1
        while w < 8 and rows * w < WARPS_IN_FLIGHT and rowlen >= 256 * w:
            w *= 2
        return w

    @classmethod
    def _mode(cls, rowlen: int, rows_per_node: np.ndarray) -> int:
        """Row schedule of one launch (coarse.cu ``mode``: WPR | RPW << 4).
        WPR > 1 splits long rows over warps; with WPR = 1 a warp takes RPW = 2
        or 4 rows when that brings the launch down to about one wave of CTAs
        (the per-CTA front/vector load is then amortised over more rows)."""
        w = cls._wpr(rowlen, int(rows_per_node.sum()))
        if w > 1:
            return w
        forced = os.environ.get("TVB_ND_RPW")
        if forced:
            r = int(forced)
            return 1 if r <= 1 else 1 | (r << 4)
        rpw = 1
        while rpw < 4 and int(np.ceil(rows_per_node / (8 * rpw)).sum()) > CTA_SLOTS:
            rpw *= 2
        return 1 if rpw == 1 else 1 | (rpw << 4)

    def _pack(self, torch, dev, fs, nbot, s, u, sd, udof_list, gmaps, t_pos, t_idx, n_cu, heights):
        self.n_bottom = nbot
        self.s, self.u = s, u
        g_off = np.zeros(nbot + 1, dtype=np.int64)
        b_off = np.zeros(nbot + 1, dtype=np.int64)
        if nbot:
            g_off[1:] = np.cumsum(s * u)
            b_off[1:] = np.cumsum(s * (s + u))
        ng, nbb = int(g_off[-1]), int(b_off[-1])
        nt = self.top_tiles
        ntop2 = nt * (nt + 1) // 2 * TOP_TILE * TOP_TILE if nt else self.n_top * self.n_top
        # G, [Z | -G^T] and the dense top inverse in ONE allocation
        self.factor = torch.zeros(ng + nbb + ntop2 + 3, dtype=torch.float64, device=dev)
        self.G = self.factor[:ng + 1]
        self.B = self.factor[ng + 1:ng + nbb + 2]
        self.ZT = self.factor[ng + nbb + 2:]
        self.g_off, self.b_off = g_off, b_off
        base = self.factor.data_ptr()
        for k in range(nbot if fs is not None else 0):  # G (u x s) and B = [Z | -G^T] (s x (s + u)) of every bottom front
            check(lib().tvb_front_pack(ctypes.byref(fs), k, base + 8 * int(g_off[k]), base + 8 * (ng + 1 + int(b_off[k])),
                                       int(s[k]), int(u[k]), stream_ptr()), "front pack")
        if ntop2 and fs is not None:  # the top inverse: lower 64x64 tiles or dense rows
            check(lib().tvb_front_pack_top(ctypes.byref(fs), nbot, self.n_top, nt, base + 8 * (ng + nbb + 2),
                                           stream_ptr()), "front pack top")
        if nt:
            self.tpart = torch.zeros(MAX_COLS, nt * nt * TOP_TILE, dtype=torch.float64, device=dev)
        else:
            self.tpart = None
        ud_off = np.zeros(nbot + 1, dtype=np.int64)
        if nbot:
            ud_off[1:] = np.cumsum(u)
        assert int(ud_off[-1]) == n_cu
        self.udof = torch.from_numpy(np.concatenate(udof_list + [np.zeros(1, np.int32)])).to(dev)
        gm_off = np.zeros(nbot + 1, dtype=np.int64)
        gm_off[1:] = np.cumsum([g.size for g in gmaps])
        self.gmap = torch.from_numpy(np.concatenate(gmaps + [np.zeros(1, np.int32)])).to(dev)
        meta = np.zeros((max(nbot, 1), 8), dtype=np.int64)
        if nbot:
            meta[:, :7] = np.stack([s, u, g_off[:-1], b_off[:-1], sd, ud_off[:-1], gm_off[:-1]], axis=1)
        self.meta = torch.from_numpy(np.ascontiguousarray(meta)).to(dev)
        # top gather (CSR over top positions, contributions in child order)
        if t_pos:
            tp, ti = np.concatenate(t_pos), np.concatenate(t_idx)
            o = np.argsort(tp, kind="stable")
            tp, ti = tp[o], ti[o]
        else:
            tp, ti = np.zeros(0, np.int64), np.zeros(0, np.int64)
        tptr = np.zeros(self.n_top + 1, dtype=np.int64)
        np.add.at(tptr, tp + 1, 1)
        tptr = np.cumsum(tptr)
        self.tptr = torch.from_numpy(tptr.astype(np.int32)).to(dev)
        self.tidx = torch.from_numpy(np.concatenate([ti, [0]]).astype(np.int32)).to(dev)
        n_c = 6 * self.nb
        # per-RHS scratch columns (multi-RHS solves, coarse.cu ColSet)
        self.max_cols = MAX_COLS
        self.fS = torch.zeros(MAX_COLS, n_c + 1, dtype=torch.float64, device=dev)   # indexed by ND dof
        self.cU = torch.zeros(MAX_COLS, n_cu + 1, dtype=torch.float64, device=dev)
        self.fT = torch.zeros(MAX_COLS, self.n_top + 1, dtype=torch.float64, device=dev)
        self.perm = torch.from_numpy(self.perm_host.astype(np.int32)).to(dev)
        # work items per bottom height: (node, row0, row1); fwd rows = u (length s),
        # bwd rows = s (length s + u); 8 / wpr rows per 256-thread CTA
        heights = np.array(heights, dtype=np.int64)
        fwd, bwd, fptr, bptr, fw, bw = [], [], [0], [0], [], []
        for h in range(self.H0):
            at = np.flatnonzero(heights == h)
            w = self._mode(int(s[at].max()) if at.size else 1, u[at])
            fw.append(w)
            step = mode_step(w)
            for ni in at:
                nr = int(u[ni])
                for r0 in range(0, max(nr, 1), step):
                    fwd.append((ni, r0, min(nr, r0 + step)))
            fptr.append(len(fwd))
        for h in range(self.H0 - 1, -1, -1):
            at = np.flatnonzero(heights == h)
            w = self._mode(int((s[at] + u[at]).max()) if at.size else 1, s[at])
            bw.append(w)
            step = mode_step(w)
            for ni in at:
                nr = int(s[ni])
                for r0 in range(0, nr, step):
                    bwd.append((ni, r0, min(nr, r0 + step)))
            bptr.append(len(bwd))
        self.top_wpr = (int(os.environ["TVB_ND_TOP_MODE"]) if os.environ.get("TVB_ND_TOP_MODE")
                        else self._mode(self.n_top, np.array([self.n_top])))
        self.fwd_items = torch.from_numpy(np.array(fwd or [(0, 0, 0)], dtype=np.int32).reshape(-1, 3)).to(dev)
        self.bwd_items = torch.from_numpy(np.array(bwd or [(0, 0, 0)], dtype=np.int32).reshape(-1, 3)).to(dev)
        # device item records of the level schedule: the node's meta row, 0, row0, row1
        # (one round trip per CTA instead of item -> node -> meta)
        def records(lst):
            a = np.array(lst or [(0, 0, 0)], dtype=np.int64).reshape(-1, 3)
            rec = np.zeros((a.shape[0], 10), dtype=np.int64)
            rec[:, :8] = meta[a[:, 0]]
            rec[:, 8:] = a[:, 1:]
            return torch.from_numpy(rec).to(dev)

        self.fwd_rec = records(fwd)
        self.bwd_rec = records(bwd)
        self.fwd_ptr = np.array(fptr, dtype=np.int64)
        self.bwd_ptr = np.array(bptr, dtype=np.int64)
        self.fwd_wpr = np.array(fw or [1], dtype=np.int32)
        self.bwd_wpr = np.array(bw or [1], dtype=np.int32)
        self.max_front = int((s + u).max()) if nbot else 1
        self.max_sep = int(s.max()) if nbot else 1
        if 8 * max(self.max_front, self.n_top + 1) > SMEM_MAX:
            raise ValueError(f"coarse front of {max(self.max_front, self.n_top)} DOFs exceeds shared memory")
        self.split = np.array([int(max(int(s[i] + u[i]) for i in np.flatnonzero(heights == h)) > SPLIT_FRONT)
                               for h in range(self.H0)] or [0], dtype=np.int32)
        asm, aptr = [], [0]
        for h in range(self.H0):
            asm.extend(np.flatnonzero(heights == h).tolist())
            aptr.append(len(asm))
        self.asm_nodes = torch.from_numpy(np.array(asm or [0], dtype=np.int32)).to(dev)
        self.asm_ptr = np.array(aptr, dtype=np.int64)
        self.bytes = self.factor.numel() * 8
        # dataflow items: structural, cached with the index plan
        flow_key = ("flow", self.grid, self.leaf_max, self.top_max, str(dev))
        if flow_key not in _PLAN_CACHE:
            items, rel, ncnt = self._flow_items(s, u, heights)
            _PLAN_CACHE[flow_key] = (len(items) // 12,
                                     torch.from_numpy(np.array(items, dtype=np.int32).reshape(-1, 12)).to(dev),
                                     torch.from_numpy(np.array(rel + [0], dtype=np.int32)).to(dev), ncnt)
        self.n_items, self.items, self.rel, ncnt = _PLAN_CACHE[flow_key]
        self.cnt = torch.zeros(ncnt + 1, dtype=torch.int64, device=dev)
        self.ctl = torch.zeros(4, dtype=torch.int64, device=dev)

    # item types of the dataflow schedule (coarse.cu: CoarseItem)
    FWD, ASM, ROWS, TOP_GATHER, TOP_ROWS, BWD = range(6)

    def _flow_items(self, s, u, heights):
        """Work items of the persistent dataflow solve in topological order.

        Counters (one int64 each): per bottom node k: fwd_ready[k] (children
        finished), fwd_done[k], asm_done[k], bwd_ready[k] (parent finished),
        bwd_done[k]; then top_ready, gather_done, top_done. An item waits for
        cnt[wait] >= epoch * need and bumps cnt[done]; the item that brings
        cnt[done] to epoch * need releases its dependants (bumps ``rel``)."""
        nb = self.n_bottom
        F_READY, F_DONE, A_DONE, B_READY, B_DONE = (k * nb for k in range(5))
        TOP_READY, G_DONE, T_DONE = 5 * nb, 5 * nb + 1, 5 * nb + 2
        items, rel = [], []
        tchildren = [k for k in range(nb) if self._top_parent[k]]

        def add(typ, wpr, node, r0, r1, wait, wneed, done, dneed, releases):
            items.extend([typ, wpr, node, r0, r1, wait, wneed, done, dneed, len(rel), len(rel) + len(releases), 0])
            rel.extend(releases)

        def fwd_release(k):
            if self._bparent[k] >= 0:
                return [F_READY + int(self._bparent[k])]
            if self._top_parent[k]:
                return [TOP_READY]
            return [B_READY + k]  # root of a pure-ND tree: its own backward pass may start

        for h in range(self.H0):
            at = np.flatnonzero(heights == h)
            w = int(self.fwd_wpr[h])
            split = bool(self.split[h])
            step = mode_step(w)
            for k in at if split else []:
                nk = len(self._bkids[k])
                add(self.ASM, 1, k, 0, 0, F_READY + k if nk else -1, nk, A_DONE + k, 1, [])
            for k in at:
                nr = int(u[k])
                chunks = list(range(0, max(nr, 1), step))
                nk = len(self._bkids[k])
                wait, wneed = (A_DONE + k, 1) if split else ((F_READY + k, nk) if nk else (-1, 0))
                rl = fwd_release(k)
                for r0 in chunks:
                    add(self.ROWS if split else self.FWD, w, k, r0, min(nr, r0 + step), wait, wneed,
                        F_DONE + k, len(chunks), rl)
        if self.n_top:
            n_g = (self.n_top + 255) // 256
            for c in range(n_g):
                add(self.TOP_GATHER, 1, 0, 256 * c, min(self.n_top, 256 * (c + 1)),
                    TOP_READY if tchildren else -1, len(tchildren), G_DONE, n_g, [])
            step = mode_step(self.top_wpr)
            chunks = list(range(0, self.n_top, step))
            for r0 in chunks:
                add(self.TOP_ROWS, self.top_wpr, 0, r0, min(self.n_top, r0 + step), G_DONE, n_g, T_DONE,
                    len(chunks), [B_READY + k for k in tchildren])
        for gi, h in enumerate(range(self.H0 - 1, -1, -1)):
            at = np.flatnonzero(heights == h)
            w = int(self.bwd_wpr[gi])
            step = mode_step(w)
            for k in at:
                nr = int(s[k])
                chunks = list(range(0, nr, step))
                for r0 in chunks:
                    add(self.BWD, w, k, r0, min(nr, r0 + step), B_READY + k, 1, B_DONE + k, len(chunks),
                        [B_READY + c for c in self._bkids[k]])
        return items, rel, 5 * nb + 3

    def _host_array(self, ctype, values):
        arr = (ctype * len(values))(*values)
        self._keep.append(arr)
        return ctypes.cast(arr, ctypes.c_void_p)

    def _make_desc(self):
        from ._lib import CoarseND

        self._keep = []
        d = CoarseND()
        d.n_levels = self.H0
        d.max_front, d.max_sep = self.max_front, self.max_sep
        d.d_meta, d.d_gmap = ptr(self.meta), ptr(self.gmap)
        d.d_G, d.d_B = ptr(self.G), ptr(self.B)
        d.d_udof, d.d_fS, d.d_cU = ptr(self.udof), ptr(self.fS), ptr(self.cU)
        d.d_fwd_items, d.d_bwd_items = ptr(self.fwd_rec), ptr(self.bwd_rec)
        d.h_fwd_ptr = self._host_array(ctypes.c_longlong, self.fwd_ptr.tolist())
        d.h_bwd_ptr = self._host_array(ctypes.c_longlong, self.bwd_ptr.tolist())
        d.h_fwd_wpr = self._host_array(ctypes.c_int, self.fwd_wpr.tolist())
        d.h_bwd_wpr = self._host_array(ctypes.c_int, self.bwd_wpr.tolist())
        d.h_split = self._host_array(ctypes.c_int, self.split.tolist())
        d.d_asm_nodes = ptr(self.asm_nodes)
        d.h_asm_ptr = self._host_array(ctypes.c_longlong, self.asm_ptr.tolist())
        d.n_top, d.top_off, d.top_wpr = self.n_top, self.top_off, self.top_wpr
        d.d_ZT, d.d_fT = ptr(self.ZT), ptr(self.fT)
        d.d_tptr, d.d_tidx = ptr(self.tptr), ptr(self.tidx)
        d.d_perm = ptr(self.perm)
        if self.flow:
            d.d_items, d.n_items, d.d_rel = ptr(self.items), self.n_items, ptr(self.rel)
            d.d_cnt, d.d_ctl = ptr(self.cnt), ptr(self.ctl)
        d.d_factor, d.factor_bytes = ptr(self.factor), self.bytes
        d.fs_ld, d.cu_ld, d.ft_ld = self.fS.shape[1], self.cU.shape[1], self.fT.shape[1]
        d.max_cols = self.max_cols
        if self.top_tiles:
            d.top_tiles, d.d_tpart, d.tpart_ld = self.top_tiles, ptr(self.tpart), self.tpart.shape[1]
        return d

    def solve_device(self, y, x):
        """x = E^-1 y on device tensors in ND order (length 6 * n_blocks)."""
        check(lib().tvb_coarse_nd_solve(ctypes.byref(self.desc), ptr(y), ptr(x), stream_ptr()), "coarse solve")
        return x

    def nd_index(self):
        """ND DOF position of every natural coarse DOF 6B + j (host array)."""
        return _dofs(self.perm_host)
