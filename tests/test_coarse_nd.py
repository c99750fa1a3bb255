"""Nested-dissection coarse solver: the host symbolic layout and the device
solve schedules (k_coarse_fwd / k_coarse_bwd / top tiles, the dataflow
items), emulated in numpy over the packed arrays, checked against a dense
solve. The packed factor is filled by a numpy front elimination
(``host_factor``); the device factorisation itself is tested on the GPU
(tests/test_gpu_front_factor.py). CPU only."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def random_block_stencil(mx, my, mz, seed=0):
    """Symmetric, diagonally dominant 27-neighbour 6x6 block stencil."""
    rng = np.random.default_rng(seed)
    nb = mx * my * mz
    Es = np.zeros((nb, 27, 6, 6))
    for B in range(nb):
        bx, by, bz = B % mx, (B // mx) % my, B // (mx * my)
        for d in range(27):
            dx, dy, dz = d % 3 - 1, (d // 3) % 3 - 1, d // 9 - 1
            cx, cy, cz = bx + dx, by + dy, bz + dz
            if not (0 <= cx < mx and 0 <= cy < my and 0 <= cz < mz):
                continue
            C = cx + mx * (cy + my * cz)
            if (C, 26 - d) < (B, d):
                Es[B, d] = Es[C, 26 - d].T
            elif d == 13:
                a = rng.standard_normal((6, 6))
                Es[B, d] = a @ a.T + 60.0 * np.eye(6)
            else:
                Es[B, d] = rng.standard_normal((6, 6))
    return Es


def dense_of(Es, mx, my, mz):
    nb = mx * my * mz
    E = np.zeros((6 * nb, 6 * nb))
    for B in range(nb):
        bx, by, bz = B % mx, (B // mx) % my, B // (mx * my)
        for d in range(27):
            dx, dy, dz = d % 3 - 1, (d // 3) % 3 - 1, d // 9 - 1
            cx, cy, cz = bx + dx, by + dy, bz + dz
            if 0 <= cx < mx and 0 <= cy < my and 0 <= cz < mz:
                C = cx + mx * (cy + my * cz)
                E[6 * B:6 * B + 6, 6 * C:6 * C + 6] = Es[B, d]
    return E


def host_factor(nd, E):
    """numpy twin of the device front factorisation (csrc/dense.cu) writing
    the solver's packed layout: per bottom node Z = F_SS^-1, G = F_US Z,
    update F_UU - G F_SU to the parent; the top Schur complement inverted
    densely (test infrastructure: the product factors on the device only)."""
    nodes = nd.nodes
    perm = nd.perm_host
    Gv, Bv, ZTv = nd.G.numpy(), nd.B.numpy(), nd.ZT.numpy()
    upd = {}
    fronts = {}
    for k, ni in enumerate(nd.bottom_nodes):
        n = nodes[ni]
        front = np.concatenate([n.sep, n.upd])
        dofs = (6 * front[:, None] + np.arange(6)).ravel()
        F = np.zeros((dofs.size, dofs.size))
        S = 6 * n.sep.size
        # original entries with the row or the column in the separator
        F[:S, :] = E[np.ix_(dofs[:S], dofs)]
        F[S:, :S] = E[np.ix_(dofs[S:], dofs[:S])]
        pos = {int(b): i for i, b in enumerate(front)}
        for c in n.children:
            cu, U = upd.pop(c)
            m = (6 * np.array([pos[int(b)] for b in cu])[:, None] + np.arange(6)).ravel()
            F[np.ix_(m, m)] += U
        Z = np.linalg.inv(F[:S, :S])
        G = F[S:, :S] @ Z
        if n.upd.size:
            upd[ni] = (n.upd, F[S:, S:] - G @ F[:S, S:])
        s, u = S, 6 * n.upd.size
        Gv[nd.g_off[k]:nd.g_off[k] + s * u] = G.ravel()
        Bv[nd.b_off[k]:nd.b_off[k] + s * (s + u)] = np.concatenate([Z, -G.T], axis=1).ravel()
    if nd.n_top:
        tblocks = np.concatenate([nodes[i].sep for i in nd.top_nodes])
        tdofs = (6 * tblocks[:, None] + np.arange(6)).ravel()
        ST = E[np.ix_(tdofs, tdofs)].copy()
        tpos = {int(b): i for i, b in enumerate(tblocks)}
        for ni, (cu, U) in list(upd.items()):
            m = (6 * np.array([tpos[int(b)] for b in cu])[:, None] + np.arange(6)).ravel()
            ST[np.ix_(m, m)] += U
            upd.pop(ni)
        Zt = np.linalg.inv(ST)
        n = nd.n_top
        if nd.top_tiles:
            nt, ts = nd.top_tiles, 64
            Zp = np.zeros((nt * ts, nt * ts))
            Zp[:n, :n] = Zt
            I, J = np.tril_indices(nt)
            tiles = Zp.reshape(nt, ts, nt, ts).transpose(0, 2, 1, 3)[I, J]
            ZTv[:tiles.size] = tiles.ravel()
        else:
            ZTv[:n * n] = Zt.ravel()
    assert not upd


def emulate_solve(nd, y):
    """numpy twin of the device solve (coarse.cu) over the packed data; y and
    the result are in ND order."""
    meta = nd.meta.numpy()
    gmap = nd.gmap.numpy()
    G, B, ZT = nd.G.numpy(), nd.B.numpy(), nd.ZT.numpy()
    udof = nd.udof.numpy()
    fS = np.zeros(nd.fS.numel())
    cU = np.zeros(nd.cU.numel())
    fwd, bwd = nd.fwd_items.numpy(), nd.bwd_items.numpy()

    def gather(gm, p, base):
        g = gmap[gm + 2 * p:gm + 2 * p + 2].reshape(-1, 2) if np.ndim(p) == 0 else \
            np.stack([gmap[gm + 2 * p], gmap[gm + 2 * p + 1]], axis=1)
        c0 = np.where(g[:, 0] >= 0, cU[np.maximum(g[:, 0], 0)], 0.0)
        c1 = np.where(g[:, 1] >= 0, cU[np.maximum(g[:, 1], 0)], 0.0)
        return base + c0 + c1

    for h in range(nd.H0):  # k_coarse_fwd (or k_coarse_asm + assembled rows)
        for node, r0, r1 in fwd[nd.fwd_ptr[h]:nd.fwd_ptr[h + 1]]:
            s, u, g, b, so, uo, gm, _ = meta[node]
            fs = gather(gm, np.arange(s), y[so:so + s])
            fS[so:so + s] = fs
            fu = gather(gm, s + np.arange(r0, r1), 0.0)
            Gm = G[g:g + s * u].reshape(u, s)
            cU[uo + r0:uo + r1] = fu - Gm[r0:r1] @ fs
    x = np.zeros_like(y)
    if nd.n_top:  # k_coarse_top_gather + k_coarse_top_rows
        n = nd.n_top
        tptr, tidx = nd.tptr.numpy(), nd.tidx.numpy()
        fT = np.array([y[nd.top_off + i] + cU[tidx[tptr[i]:tptr[i + 1]]].sum() for i in range(n)])
        if nd.top_tiles:  # k_top_tiles + k_top_reduce over the packed lower tiles
            nt, ts = nd.top_tiles, 64
            fp = np.zeros(nt * ts)
            fp[:n] = fT
            tiles = ZT[:nt * (nt + 1) // 2 * ts * ts].reshape(-1, ts, ts)
            P = np.zeros((nt, nt, ts))
            for t, (I, J) in enumerate(zip(*np.tril_indices(nt))):
                P[I, J] = tiles[t] @ fp[J * ts:(J + 1) * ts]
                if I != J:
                    P[J, I] = tiles[t].T @ fp[I * ts:(I + 1) * ts]
            x[nd.top_off:] = P.sum(axis=1).reshape(-1)[:n]
        else:
            x[nd.top_off:] = ZT[:n * n].reshape(n, n) @ fT
    for node, r0, r1 in bwd:  # k_coarse_bwd, top-most bottom level first
        s, u, g, b, so, uo, gm, _ = meta[node]
        Bm = B[b:b + s * (s + u)].reshape(s, s + u)
        v = np.concatenate([fS[so:so + s], x[udof[uo:uo + u]]])
        x[so + r0:so + r1] = Bm[r0:r1] @ v
    return x


@pytest.mark.parametrize("top_max", [0, 60, 4608])
@pytest.mark.parametrize("grid,leaf", [((5, 5, 10), 27), ((4, 3, 2), 2), ((7, 1, 3), 4), ((1, 1, 1), 27),
                                       ((9, 8, 7), 8)])
def test_nd_factor_matches_dense(grid, leaf, top_max):
    from paper_2203_15115_b200.coarse import NDCoarseSolver, nested_dissection

    mx, my, mz = grid
    Es = random_block_stencil(mx, my, mz, seed=sum(grid))
    E = dense_of(Es, mx, my, mz)
    assert np.allclose(E, E.T)
    nodes = nested_dissection(mx, my, mz, leaf)
    # every block is in exactly one separator
    allsep = np.concatenate([n.sep for n in nodes])
    assert np.array_equal(np.sort(allsep), np.arange(mx * my * mz))
    nd = NDCoarseSolver(grid, torch.from_numpy(Es.reshape(-1)), leaf_max=leaf, top_max=top_max,
                        make_desc=False, numeric=False)
    host_factor(nd, E)
    assert nd.n_top <= max(top_max, 0) or nd.H0 == max(n.height for n in nodes) + 1
    # the ND order is a permutation; separators are contiguous
    assert np.array_equal(np.sort(nd.perm_host), np.arange(mx * my * mz))
    y = np.random.default_rng(1).standard_normal(E.shape[0])
    ndi = nd.nd_index()
    yn = np.empty_like(y)
    yn[ndi] = y
    x = emulate_solve(nd, yn)[ndi]
    ref = np.linalg.solve(E, y)
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()


def run_flow(nd, y, epochs=2, workers=7, seed=0):
    """numpy twin of k_coarse_flow: `workers` persistent CTAs pull items in
    index order and finish them in random order once their dependency counter
    is satisfied; checks the schedule never deadlocks over several epochs."""
    rng = np.random.default_rng(seed)
    meta = nd.meta.numpy()
    gmap = nd.gmap.numpy()
    G, B, ZT = nd.G.numpy(), nd.B.numpy(), nd.ZT.numpy()
    udof, items, rel = nd.udof.numpy(), nd.items.numpy(), nd.rel.numpy()
    tptr, tidx = nd.tptr.numpy(), nd.tidx.numpy()
    cnt = np.zeros(nd.cnt.numel(), dtype=np.int64)

    def gather(gm, p, base):
        c0 = np.where(gmap[gm + 2 * p] >= 0, cU[np.maximum(gmap[gm + 2 * p], 0)], 0.0)
        c1 = np.where(gmap[gm + 2 * p + 1] >= 0, cU[np.maximum(gmap[gm + 2 * p + 1], 0)], 0.0)
        return base + c0 + c1

    for E in range(1, epochs + 1):
        fS = np.full(nd.fS.numel(), np.nan)
        cU = np.full(nd.cU.numel(), np.nan)
        fT = np.full(nd.fT.numel(), np.nan)
        x = np.full_like(y, np.nan)
        nxt, running = 0, []
        while nxt < len(items) or running:
            while len(running) < workers and nxt < len(items):
                running.append(nxt)
                nxt += 1
            ready = [k for k in running if items[k][5] < 0 or cnt[items[k][5]] >= E * items[k][6]]
            assert ready, "dataflow schedule deadlocked"
            k = ready[rng.integers(len(ready))]
            running.remove(k)
            typ, wpr, node, r0, r1 = items[k][:5]
            if typ in (0, 1, 2):
                s, u, g, b, so, uo, gm, _ = meta[node]
                if typ == 1:
                    fS[so:so + s] = gather(gm, np.arange(s), y[so:so + s])
                    cU[uo:uo + u] = gather(gm, s + np.arange(u), 0.0)
                else:
                    if typ == 0:
                        fs = gather(gm, np.arange(s), y[so:so + s])
                        if r0 == 0:
                            fS[so:so + s] = fs
                        fu = gather(gm, s + np.arange(r0, r1), 0.0)
                    else:
                        fs = fS[so:so + s]
                        fu = cU[uo + r0:uo + r1]
                    assert np.isfinite(fs).all() and np.isfinite(fu).all()
                    cU[uo + r0:uo + r1] = fu - G[g:g + s * u].reshape(u, s)[r0:r1] @ fs
            elif typ == 3:
                for i in range(r0, r1):
                    fT[i] = y[nd.top_off + i] + cU[tidx[tptr[i]:tptr[i + 1]]].sum()
            elif typ == 4:
                n = nd.n_top
                assert np.isfinite(fT[:n]).all()
                x[nd.top_off + r0:nd.top_off + r1] = ZT[:n * n].reshape(n, n)[r0:r1] @ fT[:n]
            else:
                s, u, g, b, so, uo, gm, _ = meta[node]
                v = np.concatenate([fS[so:so + s], x[udof[uo:uo + u]]])
                assert np.isfinite(v).all()
                x[so + r0:so + r1] = B[b:b + s * (s + u)].reshape(s, s + u)[r0:r1] @ v
            cnt[items[k][7]] += 1
            if cnt[items[k][7]] == E * items[k][8]:
                for j in range(items[k][9], items[k][10]):
                    cnt[rel[j]] += 1
    return x


@pytest.mark.parametrize("top_max", [0, 60, 4608])
@pytest.mark.parametrize("grid,leaf", [((5, 5, 10), 27), ((4, 3, 2), 2), ((9, 8, 7), 8), ((1, 1, 1), 27)])
def test_nd_dataflow_schedule(grid, leaf, top_max, monkeypatch):
    import paper_2203_15115_b200.coarse as C

    monkeypatch.setattr(C, "SPLIT_FRONT", 200)  # exercise the assembly items too
    monkeypatch.setattr(C, "FLOW", "1")  # the dataflow kernel reads the dense top rows (no packed tiles)
    mx, my, mz = grid
    Es = random_block_stencil(mx, my, mz, seed=sum(grid) + 1)
    E = dense_of(Es, mx, my, mz)
    nd = C.NDCoarseSolver(grid, torch.from_numpy(Es.reshape(-1)), leaf_max=leaf, top_max=top_max, make_desc=False,
                          numeric=False)
    host_factor(nd, E)
    y = np.random.default_rng(3).standard_normal(E.shape[0])
    ndi = nd.nd_index()
    yn = np.empty_like(y)
    yn[ndi] = y
    x = run_flow(nd, yn)[ndi]
    ref = np.linalg.solve(E, y)
    assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()
