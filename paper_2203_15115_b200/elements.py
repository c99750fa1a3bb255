"""Element constants of the 8-node trilinear voxel (host side, numpy).

Every element of the grid is the same cube of edge ``h``, so the whole
operator is driven by a handful of constants that are computed once on the
host and handed to the CUDA kernels:

* ``hex_stiffness``    the 24x24 element stiffness k0 (reference
  ``topovox/elements.py:117-132``: 2x2x2 Gauss, symmetrised),
* ``modal_coupling``   the same matrix expressed in the element's
  Walsh-Hadamard mode basis, where it has only 45 nonzeros (the kernel
  applies k0 as ``H3 . M . H3^T`` instead of 576 FMAs),
* ``centroid_b_matrix`` / ``elasticity_matrix`` / ``VONMISES_Q`` for the
  per-element state and sensitivity kernels (reference ``:43-52,72-79,135-138``).

Conventions (fixed package-wide, identical to the reference): local node ``i``
sits at grid offset ``NODE_OFFSETS[i]`` (VTK hexahedron order), element DOF
``3*i + axis``, Voigt order (xx, yy, zz, xy, yz, zx) with engineering shear.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# VTK hexahedron: bottom face counter-clockwise, then top face.
NODE_OFFSETS = np.array(
    [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0),
     (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)],
    dtype=np.int64,
)

# sigma_vm^2 = s^T Q s for a Voigt stress row s.
VONMISES_Q = np.diag([1.0, 1.0, 1.0, 3.0, 3.0, 3.0])
VONMISES_Q[:3, :3] -= 0.5 * (1.0 - np.eye(3))


@dataclass(frozen=True)
class Material:
    """Isotropic linear elastic material (reference ``elements.py:57-71``)."""

    E: float = 2.0e11
    nu: float = 0.3
    rho: float = 7800.0

    def __post_init__(self):
        if not self.E > 0.0:
            raise ValueError(f"Young's modulus must be positive, got {self.E}")
        if not (0.0 <= self.nu < 0.5):
            raise ValueError(f"Poisson ratio must lie in [0, 0.5), got {self.nu}")
        if not self.rho > 0.0:
            raise ValueError(f"density must be positive, got {self.rho}")


def elasticity_matrix(E: float, nu: float) -> np.ndarray:
    """Isotropic 6x6 Voigt stiffness (Lame form: lam*tr + 2*mu on normals)."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] = lam + 2.0 * mu
    D[np.arange(3, 6), np.arange(3, 6)] = mu
    return D


def _corner_signs() -> np.ndarray:
    return 2.0 * NODE_OFFSETS.astype(float) - 1.0


def _grad_ref(point) -> np.ndarray:
    """d N_i / d(xi, eta, zeta) of the 8 trilinear shape functions, (8, 3)."""
    s = _corner_signs()
    p = np.asarray(point, dtype=float)
    lin = 1.0 + s * p[None, :]  # (8, 3): (1 + s_a * x_a) per axis
    g = np.empty((8, 3))
    for a in range(3):
        others = [b for b in range(3) if b != a]
        g[:, a] = s[:, a] * lin[:, others[0]] * lin[:, others[1]] / 8.0
    return g


def strain_displacement(grad: np.ndarray) -> np.ndarray:
    """(6, 24) B matrix from physical shape-function gradients (8, 3)."""
    B = np.zeros((6, 24))
    for i in range(8):
        gx, gy, gz = grad[i]
        c = 3 * i
        B[0, c], B[1, c + 1], B[2, c + 2] = gx, gy, gz
        B[3, c], B[3, c + 1] = gy, gx          # gamma_xy
        B[4, c + 1], B[4, c + 2] = gz, gy      # gamma_yz
        B[5, c], B[5, c + 2] = gz, gx          # gamma_zx
    return B


def hex_stiffness(material: Material, h: float) -> np.ndarray:
    """Element stiffness of a cube of edge ``h`` (2x2x2 Gauss, symmetrised).

    Follows reference ``topovox/elements.py:117-132``; linear in E and h.
    """
    if not h > 0.0:
        raise ValueError(f"edge length must be positive, got {h}")
    D = elasticity_matrix(material.E, material.nu)
    jac = (0.5 * h) ** 3
    g = 1.0 / np.sqrt(3.0)
    k = np.zeros((24, 24))
    for sx in (-1.0, 1.0):
        for sy in (-1.0, 1.0):
            for sz in (-1.0, 1.0):
                B = strain_displacement(_grad_ref((sx * g, sy * g, sz * g)) * (2.0 / h))
                k += jac * (B.T @ D @ B)
    return 0.5 * (k + k.T)


def geometric_tensor(h: float) -> np.ndarray:
    """A[p, q, i, j] = sum_gp dNi/dx_p dNj/dx_q detJ over the 2x2x2 rule
    (reference ``topovox/elements.py:141-153``): contracting a constant stress
    tensor against (p, q) gives the 8x8 nodal block of the initial-stress
    matrix (replicated on each displacement component)."""
    if not h > 0.0:
        raise ValueError(f"edge length must be positive, got {h}")
    jac = (0.5 * h) ** 3
    g = 1.0 / np.sqrt(3.0)
    A = np.zeros((3, 3, 8, 8))
    for sx in (-1.0, 1.0):
        for sy in (-1.0, 1.0):
            for sz in (-1.0, 1.0):
                dn = _grad_ref((sx * g, sy * g, sz * g)) * (2.0 / h)  # (8, 3)
                A += jac * np.einsum("ip,jq->pqij", dn, dn)
    return A


#: Voigt component order of element stresses (xx, yy, zz, xy, yz, zx)
_VOIGT_PQ = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (2, 0))


def geometric_voigt_blocks(h: float) -> np.ndarray:
    """(6, 8, 8) blocks Bk with sum_pq sigma_pq A[p, q] = sum_k s_k Bk[k] for a
    Voigt stress row s (off-diagonal components enter A[p,q] + A[q,p])."""
    A = geometric_tensor(h)
    out = np.empty((6, 8, 8))
    for k, (p, q) in enumerate(_VOIGT_PQ):
        out[k] = A[p, q] if p == q else A[p, q] + A[q, p]
    return out


def centroid_b_matrix(h: float) -> np.ndarray:
    """B evaluated at the element centroid (reference ``elements.py:135-138``)."""
    return strain_displacement(_grad_ref((0.0, 0.0, 0.0)) * (2.0 / h))


def von_mises(stress_voigt) -> np.ndarray:
    """sqrt(max(s^T Q s, 0)) row-wise."""
    s = np.asarray(stress_voigt, dtype=float)
    q = np.einsum("...i,ij,...j->...", s, VONMISES_Q, s)
    return np.sqrt(np.maximum(q, 0.0))


def voigt_to_tensor(v) -> np.ndarray:
    xx, yy, zz, xy, yz, zx = (float(t) for t in v)
    return np.array([[xx, xy, zx], [xy, yy, yz], [zx, yz, zz]])


# ---------------------------------------------------------------------------
# Walsh-Hadamard mode basis (used by the CUDA matvec)
# ---------------------------------------------------------------------------

def hadamard_nodes() -> np.ndarray:
    """H[n, m] = value of mode m=(a,b,c) at local node n; modes are indexed
    like nodes (mode m uses the bits of NODE_OFFSETS[m]). H^T H = 8 I."""
    s = _corner_signs()
    bits = NODE_OFFSETS
    H = np.ones((8, 8))
    for m in range(8):
        for a in range(3):
            if bits[m, a]:
                H[:, m] *= s[:, a]
    return H


# The 45 structurally nonzero entries of the modal coupling matrix, as
# (row, col) pairs over the 24 modal DOFs 3*mode + axis. The pattern follows
# from Legendre orthogonality on the cube and is the same for every E, nu, h;
# ``modal_coupling`` verifies it numerically.
def _modal_pattern() -> list[tuple[int, int]]:
    pairs = []
    M = _modal_dense(hex_stiffness(Material(E=1.0, nu=0.3), 1.0))
    scale = np.abs(M).max()
    for i in range(24):
        for j in range(24):
            if abs(M[i, j]) > 1e-12 * scale:
                pairs.append((i, j))
    return pairs


def _modal_dense(k0: np.ndarray) -> np.ndarray:
    H3 = np.kron(hadamard_nodes(), np.eye(3))
    return H3.T @ k0 @ H3 / 64.0


MODAL_PATTERN = None


def modal_coupling(k0: np.ndarray) -> np.ndarray:
    """k0 in mode space: k0 = H3 @ Mh @ H3^T with H3 = kron(H, I3).

    Returns the dense (24, 24) Mh and checks that everything outside the
    45-entry pattern vanishes (to rounding), so the kernel may skip it.
    """
    global MODAL_PATTERN
    if MODAL_PATTERN is None:
        MODAL_PATTERN = _modal_pattern()
    M = _modal_dense(np.asarray(k0, dtype=float))
    mask = np.zeros((24, 24), dtype=bool)
    for i, j in MODAL_PATTERN:
        mask[i, j] = True
    off = np.abs(M[~mask]).max(initial=0.0)
    if off > 1e-13 * max(np.abs(M).max(), 1e-300):
        raise ValueError("element stiffness is not a cube/isotropic k0: modal pattern violated")
    M[~mask] = 0.0
    return M
