"""paper_2203_15115_b200 -- B200-native hot path of voxel topology optimisation.

Drop-in for the reference package ``topovox`` on its hot path (assembly-free
hex FEA, deflated PCG, topological sensitivities, level-set extraction and
the augmented-Lagrangian optimize loop). Same public names as
``topovox/__init__.py:12-25``; the compute runs in sm_100a CUDA kernels
(``libtopovox_b200.so``) and never on the CPU.
"""

__version__ = "0.1.0"

from .elements import Material  # noqa: E402
from .mesh import (EPS_VOID, Domain, LoadCase, RegionSelector, Topology, assemble_force,  # noqa: E402
                   build_domain, dirichlet_dofs, select, validate_case)


def backend_name() -> str:
    """The only backend: hand-written CUDA for sm_100a (reference
    ``backends/__init__.py:55-56`` returns numba|numpy)."""
    return "cuda-sm100a"


__all__ = [
    "Material",
    "Domain",
    "Topology",
    "RegionSelector",
    "LoadCase",
    "build_domain",
    "select",
    "backend_name",
    "assemble_force",
    "dirichlet_dofs",
    "validate_case",
    "EPS_VOID",
    "__version__",
]
