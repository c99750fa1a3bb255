import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import cantilever
import paper_2203_15115_b200 as tv
from paper_2203_15115_b200 import fea
from oracle import topovox_oracle as O

p = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
dims = (24, 12, 12)
occ = np.where(np.random.default_rng(3).random(np.prod(dims)) < p, 1.0, 1e-3)
d, case, fixed, f = cantilever(*dims, (dims[0], 0, 0), dims)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), fixed)
defl = fea.build_deflation(d, op.topology, fixed, 3, coarse="dense")
defl.prepare(op)
W = defl.W.toarray()
ref = O.Operator(*dims, 1.0, occ, dirichlet=fixed)
KW = np.stack([ref.apply(W[:, j]) for j in range(W.shape[1])], axis=1)
E_host = W.T @ KW
nb = defl.n_blocks
Es = defl.Es.view(nb, 27, 6, 6).cpu().numpy()
# dense from Es over kept columns
mask = defl.kept_mask.ravel()
mx, my, mz = defl.grid
Ed = np.zeros((6 * nb, 6 * nb))
for B in range(nb):
    bx, by, bz = B % mx, (B // mx) % my, B // (mx * my)
    for dd in range(27):
        cx, cy, cz = bx + dd % 3 - 1, by + (dd // 3) % 3 - 1, bz + dd // 9 - 1
        if 0 <= cx < mx and 0 <= cy < my and 0 <= cz < mz:
            C = cx + mx * (cy + my * cz)
            Ed[6*B:6*B+6, 6*C:6*C+6] = Es[B, dd]
Ek = Ed[np.ix_(mask, mask)]
print("E probe vs host W^T K W:", np.abs(Ek - E_host).max(), np.abs(E_host).max())
print("W orthonormal per block:", np.abs(W.T @ W - np.eye(W.shape[1])).max())
od = O.Deflation(ref, 3)
# span check: projection of oracle W onto my W
Wo = od.W.toarray()
res = Wo - W @ np.linalg.lstsq(W, Wo, rcond=None)[0]
print("span residual:", np.abs(res).max(), "nvec", W.shape[1], od.n_vectors)
y = np.random.default_rng(0).standard_normal(d.n_dofs)
yd = torch.from_numpy(y).cuda()
yc = torch.empty(6 * nb, dtype=torch.float64, device="cuda")
from paper_2203_15115_b200._lib import lib, ptr, stream_ptr
lib().tvb_restrict(d.nx, d.ny, d.nz, 3, d.h, ptr(defl.nflags), ptr(defl.cen), ptr(defl.S), ptr(defl.keep), ptr(yd), ptr(yc), stream_ptr())
print("restrict vs W^T y:", np.abs(yc.cpu().numpy()[mask] - W.T @ y).max())
mu = np.random.default_rng(1).standard_normal(6 * nb)
mud = torch.from_numpy(mu).cuda()
out = torch.empty(d.n_dofs, dtype=torch.float64, device="cuda")
nuw = torch.empty(6 * nb, dtype=torch.float64, device="cuda")
lib().tvb_prolong(d.nx, d.ny, d.nz, 3, d.h, ptr(defl.nflags), ptr(defl.cen), ptr(defl.S), ptr(defl.keep), ptr(mud), ptr(out), ptr(nuw), stream_ptr())
print("prolong vs W mu:", np.abs(out.cpu().numpy() - W @ mu[mask]).max())
try:
    r = fea.solve_static(op, f, tol=1e-12, deflation=defl)
    print("dpcg iters", r.iterations)
except Exception as e:
    print("dpcg failed", e)
r = fea.solve_static(op, f, tol=1e-12)
print("pcg iters", r.iterations)

# ---- replay DPCG in Python with the device pieces ----
Einv = defl.coarse_inv
nc = 6 * nb
free = torch.from_numpy(op.free_mask).cuda()
def restrict(v):
    out = torch.empty(nc, dtype=torch.float64, device="cuda")
    lib().tvb_restrict(d.nx, d.ny, d.nz, 3, d.h, ptr(defl.nflags), ptr(defl.cen), ptr(defl.S), ptr(defl.keep), ptr(v), ptr(out), stream_ptr())
    return out
def prolong(mu):
    out = torch.empty(d.n_dofs, dtype=torch.float64, device="cuda")
    nuw = torch.empty(nc, dtype=torch.float64, device="cuda")
    lib().tvb_prolong(d.nx, d.ny, d.nz, 3, d.h, ptr(defl.nflags), ptr(defl.cen), ptr(defl.S), ptr(defl.keep), ptr(mu.contiguous()), ptr(out), ptr(nuw), stream_ptr())
    return out
A = lambda v: op.apply_device(v.contiguous())
fd = torch.from_numpy(f).cuda()
dg = op.diagonal_device()
inv_d = torch.where(free, 1.0 / dg, torch.zeros_like(dg))
fn = float(torch.linalg.norm(fd[free]))
x = prolong(Einv @ restrict(fd))
r = fd - A(x); r[~free] = 0
z = inv_d * r
p = z - prolong(Einv @ restrict(A(z)))
rz = float(r @ z)
hist = []
for it in range(1, 400):
    q = A(p); al = rz / float(p @ q); x += al * p; r -= al * q
    res = float(torch.linalg.norm(r)) / fn; hist.append(res)
    if res <= 1e-12: break
    z = inv_d * r; rzn = float(r @ z); be = rzn / rz; rz = rzn
    p = z + be * p - prolong(Einv @ restrict(A(z)))
print("python-replay DPCG:", it, "iters, res", hist[-1], "hist[0:5]", [f"{h:.2e}" for h in hist[:5]])
# also the driver's residual history with small caps
for cap in (1, 2, 3, 5, 10, 20):
    try:
        fea.solve_static(op, f, tol=1e-12, deflation=defl, max_iters=cap, check_every=1)
    except Exception as e:
        print("driver cap", cap, "residual", e.residual)
import scipy.sparse
os.makedirs("gpurun_out", exist_ok=True)
scipy.sparse.save_npz("gpurun_out/myW.npz", defl.W.tocsc())
y2 = np.random.default_rng(9).standard_normal(d.n_dofs)
np.savez("gpurun_out/myA.npz", y=y2, Ay=op.apply(y2), occ=occ, fixed=fixed, f=f, Ed=Ek)
