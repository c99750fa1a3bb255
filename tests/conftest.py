import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libtopovox_b200.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def oracle():
    from oracle import topovox_oracle as O

    O.build_lib()
    return O


def cantilever(nx, ny, nz, load_min, load_max, force=(0, 0, -1)):
    from paper_2203_15115_b200.mesh import Domain, LoadCase, RegionSelector, assemble_force, dirichlet_dofs

    d = Domain(nx, ny, nz, 1.0)
    case = LoadCase("c", dirichlet=((RegionSelector("box", min=(0, 0, 0), max=(0, ny, nz)), (1, 1, 1)),),
                    loads=((RegionSelector("box", min=load_min, max=load_max), force, "total"),))
    return d, case, dirichlet_dofs(d, case), assemble_force(d, case)
