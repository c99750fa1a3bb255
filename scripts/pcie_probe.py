"""PCIe copy rates (pinned) and the host-buffer matvec pipeline vs slab count at C2(a)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

n = 128
d = tv.Domain(n, n, n, 1.0)
occ = np.where(np.random.default_rng(0).random(d.n_elems) < 0.7, 1.0, 1e-3)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
u = torch.from_numpy(np.random.default_rng(1).standard_normal(d.n_dofs)).pin_memory()
y = torch.empty_like(u).pin_memory()
ud = u.cuda()
yd = torch.empty_like(ud)
nb = 8 * d.n_dofs


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t_h2d = timeit(lambda: ud.copy_(u, non_blocking=True))
t_d2h = timeit(lambda: y.copy_(yd, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        ud.copy_(u, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(yd, non_blocking=True)


t_both = timeit(both)
print(f"H2D {nb / t_h2d / 1e9:.1f} GB/s  D2H {nb / t_d2h / 1e9:.1f} GB/s  concurrent: {2 * nb / t_both / 1e9:.1f} GB/s "
      f"({t_both * 1e3:.3f} ms for both)")
for slabs in (1, 2, 3, 4, 6, 8):
    t = timeit(lambda: op.apply_host(u, y, slabs=slabs))
    print(f"slabs {slabs}: {t * 1e3:.3f} ms/step  {d.n_dofs / t / 1e9:.2f} GDOF/s")

# pipeline emulation with torch streams/events: H2D chunk k on s1, D2H chunk k on s2 after H2D chunk k
for K in (2, 4, 8, 16):
    ev = [torch.cuda.Event() for _ in range(K)]
    n = u.numel()
    cuts = [n * k // K for k in range(K + 1)]

    def pipe():
        for k in range(K):
            with torch.cuda.stream(s1):
                ud[cuts[k]:cuts[k + 1]].copy_(u[cuts[k]:cuts[k + 1]], non_blocking=True)
                ev[k].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(ev[k])
                y[cuts[k]:cuts[k + 1]].copy_(yd[cuts[k]:cuts[k + 1]], non_blocking=True)

    t = timeit(pipe)
    print(f"torch pipeline K={K}: {t * 1e3:.3f} ms ({2 * nb / t / 1e9:.1f} GB/s)")


def both_chunked(K):
    n = u.numel()
    cuts = [n * k // K for k in range(K + 1)]
    for k in range(K):
        with torch.cuda.stream(s1):
            ud[cuts[k]:cuts[k + 1]].copy_(u[cuts[k]:cuts[k + 1]], non_blocking=True)
        with torch.cuda.stream(s2):
            y[cuts[k]:cuts[k + 1]].copy_(yd[cuts[k]:cuts[k + 1]], non_blocking=True)


for K in (4, 16):
    t = timeit(lambda: both_chunked(K))
    print(f"independent chunked K={K}: {t * 1e3:.3f} ms")
