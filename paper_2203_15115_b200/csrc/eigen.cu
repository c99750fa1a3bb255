// eigen / buckling analyses:
//
//   k_geo_matvec       geometric-stiffness action; explicit blocks = the
//                      reference seam apply_nodal_block8
//                      (topovox/backends/numba_kernels.py:61-76), or blocks
//                      contracted from the element stress with the 6 Voigt
//                      components of geometric_tensor (elements.py:141-153)
//   k_lumped_mass      MassOperator: rho h^3 / 8 * occupancy to each corner
//   k_eigen_sens       T_lambda
//   k_buckling_sens    T_p
//
// Node-owner gathers like k_inv_diag: each output node sums its <= 8
// elements in a fixed order (dz, dy, dx), so results are deterministic and
// atomic-free. These are not on the per-iteration path of the static solve
// (the DPCG solves inside the eigen iteration are), so they are written for
// clarity: one thread per node / element, constants staged in shared memory.
#include "eigen.cuh"

namespace tvb {

// local node index (VTK hexahedron order, topovox/elements.py NODE_OFFSETS)
__device__ __forceinline__ int vtk_local(int ox, int oy, int oz) {
  return 4 * oz + (oy ? (ox ? 2 : 3) : (ox ? 1 : 0));
}
__device__ __forceinline__ void vtk_offset(int i, int& ox, int& oy, int& oz) {
  oz = i >> 2;
  const int r = i & 3;
  ox = (r == 1 || r == 2) ? 1 : 0;
  oy = (r >= 2) ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_geo_matvec(GeoArgs A) {
  __shared__ double sB[6 * 64];
  if (A.blocks == nullptr)
    for (int i = threadIdx.x; i < 6 * 64; i += blockDim.x) sB[i] = A.Bk[i];
  __syncthreads();
  const Grid& G = A.g;
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= G.nn) return;
  const int x = (int)(n % G.px), y = (int)((n / G.px) % G.py), z = (int)(n / ((long long)G.px * G.py));
  double acc[3] = {0.0, 0.0, 0.0};
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy, ez = z + dz;
        if (ex < 0 || ex >= G.nx || ey < 0 || ey >= G.ny || ez < 0 || ez >= G.nz) continue;
        const long long e = G.elem(ex, ey, ez);
        const int i = vtk_local(-dx, -dy, -dz);
        double row[8];
        if (A.blocks != nullptr) {
#pragma unroll
          for (int j = 0; j < 8; ++j) row[j] = __ldg(A.blocks + 64 * e + 8 * i + j);
        } else {
          double s[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) s[k] = __ldg(A.stress + 6 * e + k);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double r = 0.0;
#pragma unroll
            for (int k = 0; k < 6; ++k) r = fma(s[k], sB[64 * k + 8 * i + j], r);
            row[j] = r;
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          int ox, oy, oz;
          vtk_offset(j, ox, oy, oz);
          const long long m = G.node(ex + ox, ey + oy, ez + oz);
          const uint8_t fl = (A.mask_in && A.nflags) ? A.nflags[m] : 0;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double v = ((fl >> a) & 1) ? 0.0 : __ldg(A.u + 3 * m + a);
            acc[a] = fma(row[j], v, acc[a]);
          }
        }
      }
  const uint8_t fo = (A.mask_out && A.nflags) ? A.nflags[n] : 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double v = ((fo >> a) & 1) ? 0.0 : A.scale * acc[a];
    if (A.accumulate) v += A.y[3 * n + a];
    A.y[3 * n + a] = v;
  }
}

cudaError_t launch_geo_matvec(const GeoArgs& A, cudaStream_t s) {
  k_geo_matvec<<<(unsigned)((A.g.nn + 255) / 256), 256, 0, s>>>(A);
  return cudaGetLastError();
}

__global__ void k_lumped_mass(Grid G, double coef, const double* occ, double* mass) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= G.nn) return;
  const int x = (int)(n % G.px), y = (int)((n / G.px) % G.py), z = (int)(n / ((long long)G.px * G.py));
  double s = 0.0;
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy, ez = z + dz;
        if (ex >= 0 && ex < G.nx && ey >= 0 && ey < G.ny && ez >= 0 && ez < G.nz) s += occ[G.elem(ex, ey, ez)];
      }
  const double m = coef * s;
  mass[3 * n] = m;
  mass[3 * n + 1] = m;
  mass[3 * n + 2] = m;
}

cudaError_t launch_lumped_mass(const Grid& G, double coef, const double* occ, double* mass, cudaStream_t s) {
  k_lumped_mass<<<(unsigned)((G.nn + 255) / 256), 256, 0, s>>>(G, coef, occ, mass);
  return cudaGetLastError();
}

// centroid strain from the 8 corner nodes (B_c entries +-1/(4h)), same
// arithmetic as fields.cu centroid_strain
__device__ __forceinline__ void corner_strain(const Grid& G, const double* __restrict__ u, int ex, int ey, int ez,
                                              double inv4h, double (&eps)[6], double (&ubar)[3]) {
  double gx[3] = {0, 0, 0}, gy[3] = {0, 0, 0}, gz[3] = {0, 0, 0}, us[3] = {0, 0, 0};
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const int ox = b & 1, oy = (b >> 1) & 1, oz = b >> 2;
    const long long n = G.node(ex + ox, ey + oy, ez + oz);
    const double sx = ox ? 1.0 : -1.0, sy = oy ? 1.0 : -1.0, sz = oz ? 1.0 : -1.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v = __ldg(u + 3 * n + a);
      gx[a] = fma(sx, v, gx[a]);
      gy[a] = fma(sy, v, gy[a]);
      gz[a] = fma(sz, v, gz[a]);
      us[a] += v;
    }
  }
  eps[0] = gx[0] * inv4h;
  eps[1] = gy[1] * inv4h;
  eps[2] = gz[2] * inv4h;
  eps[3] = (gy[0] + gx[1]) * inv4h;
  eps[4] = (gz[1] + gy[2]) * inv4h;
  eps[5] = (gz[0] + gx[2]) * inv4h;
#pragma unroll
  for (int a = 0; a < 3; ++a) ubar[a] = 0.125 * us[a];
}

__global__ void k_eigen_sens(ElemArgs A, double omega2rho, double* out) {
  const Grid& G = A.g;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= G.ne) return;
  const int ex = (int)(e % G.nx), ey = (int)((e / G.nx) % G.ny), ez = (int)(e / ((long long)G.nx * G.ny));
  double eps[6], ub[3];
  corner_strain(G, A.u, ex, ey, ez, A.inv4h, eps, ub);
  const double occ = A.occ[e];
  const Elastic& D = A.D;
  // sigma = occ D eps, the arithmetic of fields.cu stress_of
  const double tr = eps[0] + eps[1] + eps[2];
  const double s0 = occ * fma(D.d0 - D.d1, eps[0], D.d1 * tr);
  const double s1 = occ * fma(D.d0 - D.d1, eps[1], D.d1 * tr);
  const double s2 = occ * fma(D.d0 - D.d1, eps[2], D.d1 * tr);
  const double s3 = occ * (D.d2 * eps[3]), s4 = occ * (D.d2 * eps[4]), s5 = occ * (D.d2 * eps[5]);
  const double se = s0 * eps[0] + s1 * eps[1] + s2 * eps[2] + s3 * eps[3] + s4 * eps[4] + s5 * eps[5];
  const double ke = ub[0] * ub[0] + ub[1] * ub[1] + ub[2] * ub[2];
  out[e] = se - omega2rho * occ * ke;
}

cudaError_t launch_eigen_sens(const ElemArgs& A, double omega2rho, double* out, cudaStream_t s) {
  k_eigen_sens<<<(unsigned)((A.g.ne + 255) / 256), 256, 0, s>>>(A, omega2rho, out);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_buckling_sens(Grid G, const double* k0, const double* Bk,
                                                       const double* stress, const double* u, const double* occ,
                                                       double lambda, double* out) {
  __shared__ double sk[24 * 24];
  __shared__ double sB[6 * 64];
  for (int i = threadIdx.x; i < 24 * 24; i += blockDim.x) sk[i] = k0[i];
  for (int i = threadIdx.x; i < 6 * 64; i += blockDim.x) sB[i] = Bk[i];
  __syncthreads();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= G.ne) return;
  const int ex = (int)(e % G.nx), ey = (int)((e / G.nx) % G.ny), ez = (int)(e / ((long long)G.nx * G.ny));
  double ue[24];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int ox, oy, oz;
    vtk_offset(i, ox, oy, oz);
    const long long n = G.node(ex + ox, ey + oy, ez + oz);
#pragma unroll
    for (int a = 0; a < 3; ++a) ue[3 * i + a] = __ldg(u + 3 * n + a);
  }
  double e1 = 0.0;
  for (int r = 0; r < 24; ++r) {
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < 24; ++c) t = fma(sk[24 * r + c], ue[c], t);
    e1 = fma(ue[r], t, e1);
  }
  double s[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) s[k] = stress[6 * e + k];
  double e2 = 0.0;
  for (int i = 0; i < 8; ++i) {
    double t[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      double b = 0.0;
#pragma unroll
      for (int k = 0; k < 6; ++k) b = fma(s[k], sB[64 * k + 8 * i + j], b);
#pragma unroll
      for (int a = 0; a < 3; ++a) t[a] = fma(b, ue[3 * j + a], t[a]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) e2 = fma(ue[3 * i + a], t[a], e2);
  }
  out[e] = occ[e] * e1 + lambda * e2;
}

cudaError_t launch_buckling_sens(const Grid& G, const double* k0, const double* Bk, const double* stress,
                                 const double* u, const double* occ, double lambda, double* out, cudaStream_t s) {
  k_buckling_sens<<<(unsigned)((G.ne + 255) / 256), 256, 0, s>>>(G, k0, Bk, stress, u, occ, lambda, out);
  return cudaGetLastError();
}

}  // namespace tvb
