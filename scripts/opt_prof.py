"""cProfile of C4 optimizer outer iterations (after a warm-up iteration)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15115_b200 import optimize as opt  # noqa: E402

prob = opt.cantilever_problem(160, 80, 80, (160, 39, 39), (160, 41, 41), force=(0, 0, -1),
                              extra_cases=[("case2", (160, 39, 39), (160, 41, 41), (0, -1, 0))],
                              constraints=[opt.ConstraintSpec("compliance", 2.0, load_case="load"),
                                           opt.ConstraintSpec("compliance", 2.0, load_case="case2"),
                                           opt.ConstraintSpec("pnorm_stress", 1.2, load_case="load", p=8),
                                           opt.ConstraintSpec("pnorm_stress", 1.2, load_case="case2", p=8)])
opt.run(prob, opt.OptimizerConfig(ersatz=1e-3, block=8, max_outer=1))  # warm
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
opt.run(prob, opt.OptimizerConfig(ersatz=1e-3, block=8, max_outer=2))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
