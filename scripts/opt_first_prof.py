"""cProfile of the FIRST C4 optimizer outer iteration in a fresh process
(setup, J0 reference solves, graph capture, library initialisation)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15115_b200 import optimize as opt  # noqa: E402

torch.zeros(1, device="cuda")
torch.cuda.synchronize()
prob = opt.cantilever_problem(160, 80, 80, (160, 39, 39), (160, 41, 41), force=(0, 0, -1),
                              extra_cases=[("case2", (160, 39, 39), (160, 41, 41), (0, -1, 0))],
                              constraints=[opt.ConstraintSpec("compliance", 2.0, load_case="load"),
                                           opt.ConstraintSpec("compliance", 2.0, load_case="case2"),
                                           opt.ConstraintSpec("pnorm_stress", 1.2, load_case="load", p=8),
                                           opt.ConstraintSpec("pnorm_stress", 1.2, load_case="case2", p=8)])
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
opt.run(prob, opt.OptimizerConfig(ersatz=1e-3, block=8, max_outer=1))
torch.cuda.synchronize()
pr.disable()
print("first outer iteration incl. setup: %.2f s" % (time.perf_counter() - t0))
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
