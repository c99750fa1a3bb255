"""Optimizer throughput on the GPU: a few outer iterations of the BASELINE
configs (C3 single-case compliance, C4 two load cases + p-norm stress),
timed per outer iteration and per FEA solve."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15115_b200 import optimize as opt  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "C3"
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "C3":
    prob = opt.cantilever_problem(80, 40, 40, (80, 20, 20), (80, 20, 20),
                                  constraints=[opt.ConstraintSpec("compliance", 1.6)])
    cfg = opt.OptimizerConfig(ersatz=1e-3, block=4, max_outer=outer)
elif which == "C4":
    prob = opt.cantilever_problem(160, 80, 80, (160, 39, 39), (160, 41, 41), force=(0, 0, -1),
                                  extra_cases=[("case2", (160, 39, 39), (160, 41, 41), (0, -1, 0))],
                                  constraints=[opt.ConstraintSpec("compliance", 2.0, load_case="load"),
                                               opt.ConstraintSpec("compliance", 2.0, load_case="case2"),
                                               opt.ConstraintSpec("pnorm_stress", 1.2, load_case="load", p=8),
                                               opt.ConstraintSpec("pnorm_stress", 1.2, load_case="case2", p=8)])
    cfg = opt.OptimizerConfig(ersatz=1e-3, block=8, max_outer=outer)
else:
    raise SystemExit("C3 | C4")
recs = []
t0 = time.perf_counter()
last = [t0]


def cb(rec):
    now = time.perf_counter()
    recs.append({"k": rec.k, "v": round(rec.v, 4), "accepted": rec.accepted, "inner": rec.inner_iters,
                 "solves": rec.solves, "s": round(now - last[0], 3), "J": rec.J})
    last[0] = now
    print(json.dumps(recs[-1]), flush=True)


topo, hist, reason = opt.run(prob, cfg, callback=cb)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
solves = sum(r["solves"] for r in recs)
print(json.dumps({"config": which, "outer": len(recs), "total_s": round(tot, 2), "solves": solves,
                  "s_per_outer": round(tot / max(len(recs), 1), 3), "reason": reason}))
