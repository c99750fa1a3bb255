"""e2e host-buffer matvec at C2 (128^3): apply_host_batch over 50 pinned steps
for several slab counts, device-timed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_15115_b200 as tv  # noqa: E402
from paper_2203_15115_b200 import fea  # noqa: E402

n = 128
occ = np.where(np.random.default_rng(0).random(n ** 3) < 0.7, 1.0, 1e-3)
u = np.random.default_rng(1).standard_normal(3 * (n + 1) ** 3)
d = tv.Domain(n, n, n, 1.0)
op = fea.StiffnessOperator(d, tv.Topology(d, occ), tv.Material(E=1.0, nu=0.3), ())
up = torch.from_numpy(u).pin_memory()
yp = torch.empty(d.n_dofs, dtype=torch.float64).pin_memory()
steps = 50
for slabs in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4,6,8,12,16").split(",")]:
    op.apply_host_batch([up] * 3, [yp] * 3, slabs=slabs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    op.apply_host_batch([up] * steps, [yp] * steps, slabs=slabs)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    print(f"slabs {slabs:3d}: {ms:.3f} ms/step  {d.n_dofs / ms / 1e6:.2f} GDOF/s  "
          f"{2 * 8 * d.n_dofs / ms / 1e6:.1f} GB/s PCIe both ways", flush=True)
# plain copies for reference: H2D and D2H of the same bytes, concurrently, 50x
dev = torch.empty(d.n_dofs, dtype=torch.float64, device="cuda")
dev2 = torch.empty_like(dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    with torch.cuda.stream(s1):
        dev.copy_(up, non_blocking=True)
    with torch.cuda.stream(s2):
        yp.copy_(dev2, non_blocking=True)
torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
print(f"raw concurrent H2D+D2H copies: {ms:.3f} ms/step ({2 * 8 * d.n_dofs / ms / 1e6:.1f} GB/s)")
