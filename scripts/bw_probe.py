"""HBM bandwidth vs transfer size (calibration for the per-kernel roofline
fractions): torch copy_ (read+write bytes) and sum (read bytes) at the
vector / factor sizes of the DPCG iteration, L2 flushed before each rep."""
import json
import torch

dev = torch.device("cuda")
flush = torch.empty(512 * 2**20, dtype=torch.uint8, device=dev)
out = {}
for mb in (8, 25, 58, 100, 200, 1024):
    n = mb * 2**20 // 8
    a = torch.randn(n, dtype=torch.float64, device=dev)
    b = torch.empty_like(a)
    res = {}
    for name, fn, bytes_ in (("copy", lambda: b.copy_(a), 16 * n), ("sum", lambda: a.sum(), 8 * n)):
        ts = []
        for _ in range(12):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        res[name] = {"us": t * 1e6, "GBs": bytes_ / t / 1e9}
    out[f"{mb}MB"] = res
    print(mb, json.dumps(res))
