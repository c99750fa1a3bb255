// K10-K14: per-element state, topological sensitivities and level-set
// extraction.
//
//   k_element_state   batch_element_state (topovox/fea.py:302-309) + T_J
//                      + p-norm partial sums
//   k_stress_sens     T_sigma
//   k_adjoint_h/gather  d sigma_PN / du as an atomic-free
//                     node gather
//   k_maxabs/k_combine  normalize_field + combine
//   radix select      extract: order-statistic threshold with
//                     ascending-index tie-break, exact and deterministic
//
// All element maps are HBM-bound streaming kernels: one thread per element,
// the 8 corner nodes gathered from the interleaved node vector (neighbouring
// threads share nodes through L1/L2).
#include <algorithm>
#include <cstdlib>

#include "fields.cuh"
#include "vec.cuh"

namespace tvb {

// Centroid strain (Voigt, engineering shear) from the element's 24 DOFs:
// B_c has entries +-1/(4h) (shape-function gradients at the centroid).
__device__ __forceinline__ void centroid_strain(const Grid& G, const double* __restrict__ u, int ex, int ey, int ez,
                                                double inv4h, double (&eps)[6]) {
  double gx[3] = {0, 0, 0}, gy[3] = {0, 0, 0}, gz[3] = {0, 0, 0};  // d u_a / d x, y, z
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
    }
  }
  eps[0] = gx[0] * inv4h;
  eps[1] = gy[1] * inv4h;
  eps[2] = gz[2] * inv4h;
  eps[3] = (gy[0] + gx[1]) * inv4h;
  eps[4] = (gz[1] + gy[2]) * inv4h;
  eps[5] = (gz[0] + gx[2]) * inv4h;
}

__device__ __forceinline__ void stress_of(const Elastic& D, double occ, const double (&e)[6], double (&s)[6]) {
  const double tr = e[0] + e[1] + e[2];
  s[0] = occ * fma(D.d0 - D.d1, e[0], D.d1 * tr);
  s[1] = occ * fma(D.d0 - D.d1, e[1], D.d1 * tr);
  s[2] = occ * fma(D.d0 - D.d1, e[2], D.d1 * tr);
  s[3] = occ * (D.d2 * e[3]);
  s[4] = occ * (D.d2 * e[4]);
  s[5] = occ * (D.d2 * e[5]);
}

__device__ __forceinline__ double vm_of(const double (&s)[6]) {
  const double q = s[0] * s[0] + s[1] * s[1] + s[2] * s[2] - s[0] * s[1] - s[1] * s[2] - s[0] * s[2] +
                   3.0 * (s[3] * s[3] + s[4] * s[4] + s[5] * s[5]);
  return sqrt(fmax(q, 0.0));
}

// 4/(1+nu) s.e - (1-3nu)/(1-nu^2) tr(s) tr(e)
__device__ __forceinline__ double sens_of(const Elastic& D, const double (&s)[6], const double (&e)[6]) {
  double se = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) se = fma(s[i], e[i], se);
  const double trs = s[0] + s[1] + s[2], tre = e[0] + e[1] + e[2];
  return D.c1 * se - D.c2 * trs * tre;
}

__device__ __forceinline__ void elem_xyz(const Grid& G, long long e, int& ex, int& ey, int& ez) {
  ex = (int)(e % G.nx);
  ey = (int)((e / G.nx) % G.ny);
  ez = (int)(e / ((long long)G.nx * G.ny));
}

// powi for the (even, small) p-norm exponent; exact repeated squaring
__device__ __forceinline__ double powi(double x, int p) {
  double r = 1.0;
  double b = x;
  while (p > 0) {
    if (p & 1) r *= b;
    b *= b;
    p >>= 1;
  }
  return r;
}

// ---- z-marching element maps --------------------------------------------
// Thread = one element column segment (ex, ey, [z0, z1)); consecutive threads
// take consecutive ex. The centroid gradient splits into face sums,
//   d/dx = Sx(bottom) + Sx(top), d/dy = Sy(bottom) + Sy(top), d/dz = S(top) - S(bottom)
// (Sx = sum of +-u over the face's 4 nodes by x side, S = plain sum), so each
// element loads only its top face (4 nodes) and reuses the bottom face of
// the element below: half the gather loads and index math of the one-
// element-per-thread form. Segments are sized to give ~2 waves of threads.
struct FaceSums {
  double sx[3], sy[3], s[3];
};

__device__ __forceinline__ void face_sums(const Grid& G, const double* __restrict__ u, int ex, int ey, int z,
                                          FaceSums& F) {
  const long long n00 = G.node(ex, ey, z), n01 = n00 + G.px;
  double v[4][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    v[0][a] = __ldg(u + 3 * n00 + a);
    v[1][a] = __ldg(u + 3 * n00 + 3 + a);
    v[2][a] = __ldg(u + 3 * n01 + a);
    v[3][a] = __ldg(u + 3 * n01 + 3 + a);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    F.sx[a] = (v[1][a] - v[0][a]) + (v[3][a] - v[2][a]);
    F.sy[a] = (v[2][a] - v[0][a]) + (v[3][a] - v[1][a]);
    F.s[a] = (v[0][a] + v[1][a]) + (v[2][a] + v[3][a]);
  }
}

__device__ __forceinline__ void strain_of_faces(const FaceSums& B, const FaceSums& T, double inv4h,
                                                double (&eps)[6]) {
  const double gx0 = B.sx[0] + T.sx[0], gx1 = B.sx[1] + T.sx[1], gx2 = B.sx[2] + T.sx[2];
  const double gy0 = B.sy[0] + T.sy[0], gy1 = B.sy[1] + T.sy[1], gy2 = B.sy[2] + T.sy[2];
  const double gz0 = T.s[0] - B.s[0], gz1 = T.s[1] - B.s[1], gz2 = T.s[2] - B.s[2];
  eps[0] = gx0 * inv4h;
  eps[1] = gy1 * inv4h;
  eps[2] = gz2 * inv4h;
  eps[3] = (gy0 + gx1) * inv4h;
  eps[4] = (gz1 + gy2) * inv4h;
  eps[5] = (gz0 + gx2) * inv4h;
}

// segment length along z so that nx * ny * ceil(nz / L) threads make ~2 waves
__host__ __device__ inline int march_len(const Grid& G) {
  const long long cols = (long long)G.nx * G.ny;
  const long long want = 148LL * 2048;
  long long seg = (want + cols - 1) / cols;  // segments per column
  if (seg < 1) seg = 1;
  if (seg > G.nz) seg = G.nz;
  return (int)((G.nz + seg - 1) / seg);
}

__host__ __device__ inline long long march_threads(const Grid& G) {
  const int L = march_len(G);
  return (long long)G.nx * G.ny * ((G.nz + L - 1) / L);
}

#define TVB_MARCH_BEGIN(G)                                                        \
  const int L = march_len(G);                                                     \
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;         \
  const long long cols = (long long)(G).nx * (G).ny;                              \
  const bool live = tid < march_threads(G);                                       \
  const int ex = (int)(tid % (G).nx), ey = (int)((tid / (G).nx) % (G).ny);        \
  const int z0 = (int)(tid / cols) * L, z1 = min((G).nz, z0 + L);

__global__ void __launch_bounds__(256) k_element_state_z(ElemArgs A) {
  __shared__ double red[32];
  const Grid& G = A.g;
  TVB_MARCH_BEGIN(G)
  double pn = 0.0, oc = 0.0;
  if (live) {
    FaceSums Fb, Ft;
    face_sums(G, A.u, ex, ey, z0, Fb);
    for (int z = z0; z < z1; ++z) {
      face_sums(G, A.u, ex, ey, z + 1, Ft);
      const long long e = G.elem(ex, ey, z);
      double eps[6], sig[6];
      strain_of_faces(Fb, Ft, A.inv4h, eps);
      const double occ = A.occ[e];
      stress_of(A.D, occ, eps, sig);
      const double vm = vm_of(sig);
      if (A.strains)
        for (int i = 0; i < 6; ++i) A.strains[6 * e + i] = eps[i];
      if (A.stresses)
        for (int i = 0; i < 6; ++i) A.stresses[6 * e + i] = sig[i];
      if (A.vm) A.vm[e] = vm;
      if (A.tj) A.tj[e] = sens_of(A.D, sig, eps);
      if (A.pnorm_partials) {
        pn += occ * powi(vm, A.p);
        oc += occ;
      }
      Fb = Ft;
    }
  }
  if (A.pnorm_partials) {
    pn = block_sum(pn, red);
    oc = block_sum(oc, red);
    if (threadIdx.x == 0) {
      A.pnorm_partials[2 * blockIdx.x] = pn;
      A.pnorm_partials[2 * blockIdx.x + 1] = oc;
    }
  }
}

__global__ void __launch_bounds__(256) k_stress_sens_z(ElemArgs A, const double* lam, double* ts) {
  const Grid& G = A.g;
  TVB_MARCH_BEGIN(G)
  if (!live) return;
  FaceSums Ub, Ut, Lb, Lt;
  face_sums(G, A.u, ex, ey, z0, Ub);
  face_sums(G, lam, ex, ey, z0, Lb);
  for (int z = z0; z < z1; ++z) {
    face_sums(G, A.u, ex, ey, z + 1, Ut);
    face_sums(G, lam, ex, ey, z + 1, Lt);
    const long long e = G.elem(ex, ey, z);
    double eu[6], sig[6], el[6];
    strain_of_faces(Ub, Ut, A.inv4h, eu);
    stress_of(A.D, A.occ[e], eu, sig);
    strain_of_faces(Lb, Lt, A.inv4h, el);
    ts[e] = sens_of(A.D, sig, el);
    Ub = Ut;
    Lb = Lt;
  }
}

// h_e (see k_adjoint_h) on element column segments, face sums reused
__global__ void __launch_bounds__(256) k_adjoint_h_z(ElemArgs A, const double* sums, double* h6) {
  const Grid& G = A.g;
  TVB_MARCH_BEGIN(G)
  if (!live) return;
  const double S = sums[0] / sums[1];
  const double inv_occ_sum = 1.0 / sums[1];
  const double sp = pow(S, 1.0 / A.p - 1.0);
  FaceSums Fb, Ft;
  face_sums(G, A.u, ex, ey, z0, Fb);
  for (int z = z0; z < z1; ++z) {
    face_sums(G, A.u, ex, ey, z + 1, Ft);
    const long long e = G.elem(ex, ey, z);
    double eps[6], sig[6];
    strain_of_faces(Fb, Ft, A.inv4h, eps);
    const double occ = A.occ[e];
    stress_of(A.D, occ, eps, sig);
    const double vm = vm_of(sig);
    const double coef = sp * (occ * inv_occ_sum) * powi(vm, A.p - 2) * occ;
    double qs[6];
    qs[0] = sig[0] - 0.5 * (sig[1] + sig[2]);
    qs[1] = sig[1] - 0.5 * (sig[0] + sig[2]);
    qs[2] = sig[2] - 0.5 * (sig[0] + sig[1]);
    qs[3] = 3.0 * sig[3];
    qs[4] = 3.0 * sig[4];
    qs[5] = 3.0 * sig[5];
    double out[6];
    stress_of(A.D, coef, qs, out);
    double2* h2 = reinterpret_cast<double2*>(h6 + 6 * e);
    h2[0] = make_double2(out[0], out[1]);
    h2[1] = make_double2(out[2], out[3]);
    h2[2] = make_double2(out[4], out[5]);
    Fb = Ft;
  }
}

// rhs on node column segments: the node at (x, y, z) sums the B_c^T h of its
// 8 elements; the 4 elements of layer z-1 were the "upper" layer of the
// previous node, so each step loads one element layer (4 x 6 doubles).
__global__ void __launch_bounds__(256) k_adjoint_gather_z(Grid G, double inv4h, const double* h6,
                                                          const uint8_t* nflags, double* rhs) {
  const long long cols = (long long)G.px * G.py;
  const long long seg = (148LL * 2048 + cols - 1) / cols;
  const int L = (int)((G.pz + min(seg, (long long)G.pz) - 1) / min(seg, (long long)G.pz));
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nseg = (G.pz + L - 1) / L;
  if (tid >= cols * nseg) return;
  const int x = (int)(tid % G.px), y = (int)((tid / G.px) % G.py);
  const int z0 = (int)(tid / cols) * L, z1 = min(G.pz, z0 + L);
  // per element layer: contribution to this node from the 4 elements (dx, dy) in {-1,0}^2 of that layer,
  // split by the node's local z side (oz = 0: the node is on the element's bottom face)
  auto layer = [&](int ez, double (&bot)[3], double (&top)[3]) {
    // bot: node on the bottom face of layer ez (sz = -1); top: node on its top face (sz = +1)
#pragma unroll
    for (int a = 0; a < 3; ++a) bot[a] = top[a] = 0.0;
    if (ez < 0 || ez >= G.nz) return;
#pragma unroll
    for (int dy = -1; dy <= 0; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy;
        if (ex < 0 || ex >= G.nx || ey < 0 || ey >= G.ny) continue;
        const double* h = h6 + 6 * G.elem(ex, ey, ez);
        const double2 h01 = __ldg(reinterpret_cast<const double2*>(h));
        const double2 h23 = __ldg(reinterpret_cast<const double2*>(h) + 1);
        const double2 h45 = __ldg(reinterpret_cast<const double2*>(h) + 2);
        const double sx = dx ? 1.0 : -1.0, sy = dy ? 1.0 : -1.0;
        // terms without sz, and the sz coefficients
        const double r0 = sx * h01.x + sy * h23.y, c0 = h45.y;
        const double r1 = sy * h01.y + sx * h23.y, c1 = h45.x;
        const double r2 = sy * h45.x + sx * h45.y, c2 = h23.x;
        bot[0] += r0 - c0; top[0] += r0 + c0;
        bot[1] += r1 - c1; top[1] += r1 + c1;
        bot[2] += r2 - c2; top[2] += r2 + c2;
      }
  };
  double lowTop[3], lowBot[3], upBot[3], upTop[3];
  layer(z0 - 1, lowBot, lowTop);  // the node is on the TOP face of layer z - 1
  for (int z = z0; z < z1; ++z) {
    layer(z, upBot, upTop);        // ... and on the BOTTOM face of layer z
    const long long n = G.node(x, y, z);
    const uint8_t fl = nflags ? nflags[n] : 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double r = (upBot[a] + lowTop[a]) * inv4h;
      rhs[3 * n + a] = ((fl >> a) & 1) ? 0.0 : r;
      lowTop[a] = upTop[a];
    }
  }
}

__global__ void k_element_state(ElemArgs A) {
  __shared__ double red[32];
  const Grid& G = A.g;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double pn = 0.0, oc = 0.0;
  if (e < G.ne) {
    int ex, ey, ez;
    elem_xyz(G, e, ex, ey, ez);
    double eps[6], sig[6];
    centroid_strain(G, A.u, ex, ey, ez, A.inv4h, eps);
    const double occ = A.occ[e];
    stress_of(A.D, occ, eps, sig);
    const double vm = vm_of(sig);
    if (A.strains)
      for (int i = 0; i < 6; ++i) A.strains[6 * e + i] = eps[i];
    if (A.stresses)
      for (int i = 0; i < 6; ++i) A.stresses[6 * e + i] = sig[i];
    if (A.vm) A.vm[e] = vm;
    if (A.tj) A.tj[e] = sens_of(A.D, sig, eps);
    if (A.pnorm_partials) {
      pn = occ * powi(vm, A.p);
      oc = occ;
    }
  }
  if (A.pnorm_partials) {
    pn = block_sum(pn, red);
    oc = block_sum(oc, red);
    if (threadIdx.x == 0) {
      A.pnorm_partials[2 * blockIdx.x] = pn;
      A.pnorm_partials[2 * blockIdx.x + 1] = oc;
    }
  }
}

__global__ void k_stress_sens(ElemArgs A, const double* lam, double* ts) {
  const Grid& G = A.g;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= G.ne) return;
  int ex, ey, ez;
  elem_xyz(G, e, ex, ey, ez);
  double eu[6], sig[6], el[6];
  centroid_strain(G, A.u, ex, ey, ez, A.inv4h, eu);
  stress_of(A.D, A.occ[e], eu, sig);
  centroid_strain(G, lam, ex, ey, ez, A.inv4h, el);
  ts[e] = sens_of(A.D, sig, el);
}

// h_e = S^(1/p-1) w_e vm^(p-2) occ_e * D Q sigma_e   (w_e = occ_e / sum occ)
__global__ void k_adjoint_h(ElemArgs A, const double* sums, double* h6) {
  const Grid& G = A.g;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= G.ne) return;
  const double S = sums[0] / sums[1];  // sum w vm^p with w = occ / sum(occ)
  const double inv_occ_sum = 1.0 / sums[1];
  int ex, ey, ez;
  elem_xyz(G, e, ex, ey, ez);
  double eps[6], sig[6];
  centroid_strain(G, A.u, ex, ey, ez, A.inv4h, eps);
  const double occ = A.occ[e];
  stress_of(A.D, occ, eps, sig);
  const double vm = vm_of(sig);
  const double coef = pow(S, 1.0 / A.p - 1.0) * (occ * inv_occ_sum) * powi(vm, A.p - 2) * occ;
  // Q sigma
  double qs[6];
  qs[0] = sig[0] - 0.5 * (sig[1] + sig[2]);
  qs[1] = sig[1] - 0.5 * (sig[0] + sig[2]);
  qs[2] = sig[2] - 0.5 * (sig[0] + sig[1]);
  qs[3] = 3.0 * sig[3];
  qs[4] = 3.0 * sig[4];
  qs[5] = 3.0 * sig[5];
  double out[6];
  stress_of(A.D, coef, qs, out);  // D (Q sigma) scaled
  for (int i = 0; i < 6; ++i) h6[6 * e + i] = out[i];
}

// rhs_n = sum_{e ∋ n} B_c[:, dofs(n in e)]^T h_e, fixed DOFs zeroed. Fixed order.
__global__ void k_adjoint_gather(Grid G, double inv4h, const double* h6, const uint8_t* nflags, double* rhs) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= G.nn) return;
  const int x = (int)(n % G.px), y = (int)((n / G.px) % G.py), z = (int)(n / ((long long)G.px * G.py));
  double r[3] = {0, 0, 0};
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy, ez = z + dz;
        if (ex < 0 || ex >= G.nx || ey < 0 || ey >= G.ny || ez < 0 || ez >= G.nz) continue;
        const double* h = h6 + 6 * G.elem(ex, ey, ez);
        // node is local corner (ox,oy,oz) = (-dx,-dy,-dz); corner sign 2*o-1
        const double sx = dx ? 1.0 : -1.0, sy = dy ? 1.0 : -1.0, sz = dz ? 1.0 : -1.0;
        r[0] += (sx * h[0] + sy * h[3] + sz * h[5]) * inv4h;
        r[1] += (sy * h[1] + sx * h[3] + sz * h[4]) * inv4h;
        r[2] += (sz * h[2] + sy * h[4] + sx * h[5]) * inv4h;
      }
  const uint8_t fl = nflags ? nflags[n] : 0;
  for (int a = 0; a < 3; ++a) rhs[3 * n + a] = ((fl >> a) & 1) ? 0.0 : r[a];
}

// ---------------------------------------------------------------------------
// max |t| (deterministic: max is order independent) and combination
// ---------------------------------------------------------------------------
__global__ void k_maxabs(const double* t, long long n, double* partials) {
  __shared__ double red[32];
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(t[i]));
  m = block_max(m, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = m;
}

__global__ void k_maxabs_final(const double* partials, int np, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) m = fmax(m, partials[i]);
  m = block_max(m, red);
  if (threadIdx.x == 0) *out = m;
}

// out = sum_i w_i * t_i / max_i   (fields with weight 0 or max 0 skipped)
__global__ void k_combine(CombineArgs C, long long n, double* out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  double v = 0.0;
  for (int i = 0; i < C.k; ++i) {
    const double m = C.maxabs[i];
    if (C.w[i] == 0.0) continue;
    const double t = (m == 0.0) ? C.f[i][e] : C.f[i][e] / m;
    v = fma(C.w[i], t, v);
  }
  out[e] = v;
}

// ---------------------------------------------------------------------------
// exact order-statistic selection (radix select on order-preserving keys)
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long okey(double v) {
  if (v == 0.0) v = 0.0;  // -0 -> +0
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// state: [0] prefix key bits, [1] prefix mask, [2] k remaining, [3] count greater.
// One launch per 8-bit digit: every CTA adds its histogram of the candidates
// (keys matching the prefix so far); the last CTA to finish (done counter)
// picks the digit holding the k-th largest key, extends the prefix, and
// clears the histogram and the counter for the next digit -- no separate
// single-CTA pick launch (round 1: 8 x 7-16 us of launch-latency-bound picks).
__global__ void __launch_bounds__(256) k_radix_hist(const double* ls, const uint8_t* design, long long n,
                                                    unsigned long long* state, int shift, unsigned int* hist,
                                                    unsigned int* done) {
  __shared__ unsigned int sh[256];
  __shared__ bool last;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const unsigned long long pref = state[0], mask = state[1];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (design && !design[i]) continue;
    const unsigned long long k = okey(ls[i]);
    if ((k & mask) != pref) continue;
    atomicAdd(&sh[(k >> shift) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    sh[i] = atomicAdd(&hist[i], 0u);  // L2-coherent read of the completed histogram
    hist[i] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long kr = state[2], gt = state[3];
    int d = 255;
    for (; d >= 0; --d) {
      const unsigned long long c = sh[d];
      if (c >= kr) break;
      kr -= c;
      gt += c;
    }
    if (d < 0) d = 0;
    state[0] = pref | ((unsigned long long)d) << shift;
    state[1] = mask | 255ull << shift;
    state[2] = kr;
    state[3] = gt;
    *done = 0u;
  }
}

// per-block count of design elements whose key equals the threshold key
__global__ void k_eq_count(const double* ls, const uint8_t* design, long long n, const unsigned long long* state,
                           unsigned int* bcount) {
  __shared__ unsigned int c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && (!design || design[i]) && okey(ls[i]) == state[0]) atomicAdd(&c, 1u);
  __syncthreads();
  if (threadIdx.x == 0) bcount[blockIdx.x] = c;
}

// exclusive scan of the block counts (single CTA, sequential chunks)
__global__ void k_scan_counts(unsigned int* bcount, int nb) {
  __shared__ unsigned int carry;
  __shared__ unsigned int tmp[1024];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += 1024) {
    const int i = base + threadIdx.x;
    const unsigned int v = i < nb ? bcount[i] : 0u;
    tmp[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const unsigned int a = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0u;
      __syncthreads();
      tmp[threadIdx.x] += a;
      __syncthreads();
    }
    if (i < nb) bcount[i] = carry + tmp[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += tmp[1023];
    __syncthreads();
  }
}

// occ = 1 for key > tau, or key == tau among the first (k - #greater) by index
// (all_ties: every key == tau -- casting extraction, "best-feasible")
__global__ void k_apply_threshold(const double* ls, const uint8_t* design, long long n,
                                  const unsigned long long* state, const unsigned int* boff, double ersatz,
                                  double nondesign, double* occ, int all_ties) {
  __shared__ unsigned int flags[1024];
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool in = i < n;
  const bool des = in && (!design || design[i]);
  const unsigned long long k = in ? okey(ls[i]) : 0ull;
  const unsigned long long tau = state[0];
  const bool eq = des && k == tau;
  flags[threadIdx.x] = eq ? 1u : 0u;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const unsigned int a = threadIdx.x >= off ? flags[threadIdx.x - off] : 0u;
    __syncthreads();
    flags[threadIdx.x] += a;
    __syncthreads();
  }
  if (!in) return;
  const unsigned long long need = state[2];  // how many ties to take
  const unsigned long long rank = boff[blockIdx.x] + flags[threadIdx.x] - (eq ? 1u : 0u);
  double v;
  if (!des) v = nondesign;
  else if (k > tau || (eq && (all_ties || rank < need))) v = 1.0;
  else v = ersatz;
  occ[i] = v;
}

// ---------------------------------------------------------------------------
// casting projection (§3.7): along every element column
// parallel to `axis`, replace values by the running minimum moving away from
// the parting plane -- element layers i >= P form the +axis mold half (walked
// upwards), i < P the -axis half (walked downwards). One thread per column;
// consecutive threads take consecutive columns of the fastest non-axis
// dimension, so for axis y / z every step is a coalesced row. In place is
// allowed (each value is read before its own thread writes it).
// ---------------------------------------------------------------------------
__global__ void k_casting_project(Grid G, int axis, int P, const double* in, double* out) {
  const long long ncol = axis == 0 ? (long long)G.ny * G.nz : axis == 1 ? (long long)G.nx * G.nz
                                                                       : (long long)G.nx * G.ny;
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  long long base, stride;
  int na;
  if (axis == 0) {
    base = c * G.nx;  // (y, z) -> row start
    stride = 1;
    na = G.nx;
  } else if (axis == 1) {
    const long long x = c % G.nx, z = c / G.nx;
    base = x + (long long)G.nx * G.ny * z;
    stride = G.nx;
    na = G.ny;
  } else {
    base = c;  // (x, y)
    stride = (long long)G.nx * G.ny;
    na = G.nz;
  }
  double m = 0.0;
  for (int i = P; i < na; ++i) {  // +axis half
    const double v = in[base + stride * i];
    m = (i == P || v < m) ? v : m;
    out[base + stride * i] = m;
  }
  for (int i = P - 1; i >= 0; --i) {  // -axis half
    const double v = in[base + stride * i];
    m = (i == P - 1 || v < m) ? v : m;
    out[base + stride * i] = m;
  }
}

cudaError_t launch_casting_project(const Grid& G, int axis, int P, const double* in, double* out, cudaStream_t s) {
  const long long ncol = axis == 0 ? (long long)G.ny * G.nz : axis == 1 ? (long long)G.nx * G.nz
                                                                       : (long long)G.nx * G.ny;
  k_casting_project<<<(unsigned)((ncol + 127) / 128), 128, 0, s>>>(G, axis, P, in, out);
  return cudaGetLastError();
}

int elem_grid(long long n) { return (int)((n + 255) / 256); }

// CTAs of the element-state launch (= number of p-norm partial pairs)
int elem_state_ctas(const Grid& G) { return (int)((march_threads(G) + 255) / 256); }

cudaError_t launch_element_state(const ElemArgs& A, cudaStream_t s) {
  if (getenv("TVB_ELEM_FLAT")) k_element_state<<<elem_grid(A.g.ne), 256, 0, s>>>(A);  // A/B only
  else k_element_state_z<<<elem_state_ctas(A.g), 256, 0, s>>>(A);
  return cudaGetLastError();
}

// T_sigma gathers two node vectors per element: the one-element-per-thread
// form (more loads in flight) measured faster than the z-marching one at C4
// (ncu 32.9 vs 39.3 us), so it stays the default
cudaError_t launch_stress_sens(const ElemArgs& A, const double* lam, double* ts, cudaStream_t s) {
  if (getenv("TVB_ELEM_MARCH")) k_stress_sens_z<<<elem_state_ctas(A.g), 256, 0, s>>>(A, lam, ts);
  else k_stress_sens<<<elem_grid(A.g.ne), 256, 0, s>>>(A, lam, ts);
  return cudaGetLastError();
}

cudaError_t launch_adjoint(const ElemArgs& A, const double* sums, double* h6, const uint8_t* nflags, double* rhs,
                           cudaStream_t s) {
  if (getenv("TVB_ELEM_FLAT")) {  // A/B only
    k_adjoint_h<<<elem_grid(A.g.ne), 256, 0, s>>>(A, sums, h6);
    k_adjoint_gather<<<(unsigned)((A.g.nn + 255) / 256), 256, 0, s>>>(A.g, A.inv4h, h6, nflags, rhs);
    return cudaGetLastError();
  }
  k_adjoint_h_z<<<elem_state_ctas(A.g), 256, 0, s>>>(A, sums, h6);
  const Grid& G = A.g;
  const long long cols = (long long)G.px * G.py;
  const long long seg = std::min((148LL * 2048 + cols - 1) / cols, (long long)G.pz);
  const long long L = (G.pz + seg - 1) / seg;
  const long long nthr = cols * ((G.pz + L - 1) / L);
  k_adjoint_gather_z<<<(unsigned)((nthr + 255) / 256), 256, 0, s>>>(G, A.inv4h, h6, nflags, rhs);
  return cudaGetLastError();
}

__global__ void k_sum_pairs(const double* partials, int np, double* out) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    a += partials[2 * i];
    b += partials[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

cudaError_t launch_sum_pairs(const double* partials, int np, double* out2, cudaStream_t s) {
  k_sum_pairs<<<1, 256, 0, s>>>(partials, np, out2);
  return cudaGetLastError();
}

cudaError_t launch_maxabs(const double* t, long long n, double* partials, double* out, cudaStream_t s) {
  int nb = (int)((n + 255) / 256);
  if (nb > 1184) nb = 1184;
  if (nb < 1) nb = 1;
  k_maxabs<<<nb, 256, 0, s>>>(t, n, partials);
  k_maxabs_final<<<1, 256, 0, s>>>(partials, nb, out);
  return cudaGetLastError();
}

cudaError_t launch_combine(const CombineArgs& C, long long n, double* out, cudaStream_t s) {
  k_combine<<<elem_grid(n), 256, 0, s>>>(C, n, out);
  return cudaGetLastError();
}

size_t select_ws_bytes(long long n) {
  const long long nb = (n + 1023) / 1024;
  return 64 + 256 * sizeof(unsigned int) + (size_t)nb * sizeof(unsigned int) + 64;
}

cudaError_t launch_select(const double* ls, const uint8_t* design, long long n, long long k, double ersatz,
                          double nondesign, double* occ, void* ws, unsigned long long* state_out, cudaStream_t s,
                          int all_ties) {
  unsigned long long* state = (unsigned long long*)ws;
  unsigned int* hist = (unsigned int*)((char*)ws + 64);
  unsigned int* bcount = hist + 256;
  const unsigned long long init[4] = {0ull, 0ull, (unsigned long long)(k > 0 ? k : 1), 0ull};
  cudaError_t e = cudaMemcpyAsync(state, init, sizeof(init), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  unsigned int* done = (unsigned int*)((char*)ws + 32);
  e = cudaMemsetAsync(done, 0, 32 + 256 * sizeof(unsigned int), s);  // counter and histogram
  if (e != cudaSuccess) return e;
  int nbh = (int)((n + 255) / 256);
  if (nbh > 1184) nbh = 1184;
  if (nbh < 1) nbh = 1;
  for (int shift = 56; shift >= 0; shift -= 8) k_radix_hist<<<nbh, 256, 0, s>>>(ls, design, n, state, shift, hist, done);
  const int nb = (int)((n + 1023) / 1024);
  if (k <= 0) {
    // nothing retained: threshold above every key
    const unsigned long long none[4] = {~0ull, ~0ull, 0ull, 0ull};
    e = cudaMemcpyAsync(state, none, sizeof(none), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
  }
  k_eq_count<<<nb, 1024, 0, s>>>(ls, design, n, state, bcount);
  k_scan_counts<<<1, 1024, 0, s>>>(bcount, nb);
  k_apply_threshold<<<nb, 1024, 0, s>>>(ls, design, n, state, bcount, ersatz, nondesign, occ,
                                        k > 0 ? all_ties : 0);
  if (state_out) {
    e = cudaMemcpyAsync(state_out, state, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace tvb
