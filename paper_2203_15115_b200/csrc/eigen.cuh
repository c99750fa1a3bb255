#pragma once
#include "common.cuh"
#include "fields.cuh"

namespace tvb {

// Geometric (initial-stress) stiffness action, SURVEY §8f #2:
//   y = scale * sum_e P_e^T (B_e (x) I3) P_e u  (+ y if accumulate)
// with the per-element 8x8 nodal block B_e either given explicitly
// ([Ne][8][8], the reference seam apply_nodal_block8,
// topovox/backends/numba_kernels.py:61-76) or contracted on the fly from the
// element's centroid stress: B_e = sum_k s_k Bk[k] with Bk the 6 Voigt
// components of geometric_tensor (topovox/elements.py:141-153).
struct GeoArgs {
  Grid g;
  const double* u;
  double* y;
  const double* blocks;   // [Ne][8][8] (VTK local node order) or nullptr
  const double* stress;   // [Ne][6] Voigt xx,yy,zz,xy,yz,zx (used when blocks == nullptr)
  const double* Bk;       // device [6][8][8]
  const uint8_t* nflags;  // fixed-axis bits (mask_in / mask_out), or nullptr
  int mask_in, mask_out, accumulate;
  double scale;
};

cudaError_t launch_geo_matvec(const GeoArgs& A, cudaStream_t s);
// mass[3n+a] = coef * sum_{e ∋ n} occ_e   (coef = rho h^3 / 8)
cudaError_t launch_lumped_mass(const Grid& G, double coef, const double* occ, double* mass, cudaStream_t s);
// T_lambda = sigma(u):eps(u) - omega2rho * occ_e * |u_centroid|^2
cudaError_t launch_eigen_sens(const ElemArgs& A, double omega2rho, double* out, cudaStream_t s);
// T_p = occ_e u_e^T k0 u_e + lambda * sum_a u_ea^T B_e u_ea  (SPEC.md:328-336 with K_sigma = -K_G)
cudaError_t launch_buckling_sens(const Grid& G, const double* k0, const double* Bk, const double* stress,
                                 const double* u, const double* occ, double lambda, double* out, cudaStream_t s);

}  // namespace tvb
