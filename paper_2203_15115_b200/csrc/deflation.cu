// Deflation space of the DPCG solve (topovox/fea.py:95-215, "a5"-"a8" of
// SURVEY §8a): per-agglomerate rigid-body modes, their restriction W^T y and
// prolongation W mu, and the Galerkin coarse operator E = W^T A W.
//
// W is never materialised. Per block we keep the structural-node centroid and
// a 6x6 transform S from the raw (masked) rigid modes to an orthonormal basis
// of the same span. Restriction is then a force/torque moment sum over the
// block's closed node box followed by S^T; prolongation evaluates the rigid
// motion t + omega x r of every block containing a node.
#include <algorithm>
#include <cstdlib>

#include "deflation.cuh"
#include "vec.cuh"

namespace tvb {

// ---------------------------------------------------------------------------
// node flags
// ---------------------------------------------------------------------------
__global__ void k_struct_flags(Grid G, const double* occ, uint8_t* nflags) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= G.nn) return;
  const int x = (int)(n % G.px), y = (int)((n / G.px) % G.py), z = (int)(n / ((long long)G.px * G.py));
  bool st = false;
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy, ez = z + dz;
        if (ex >= 0 && ex < G.nx && ey >= 0 && ey < G.ny && ez >= 0 && ez < G.nz)
          st |= (occ[G.elem(ex, ey, ez)] == 1.0);
      }
  nflags[n] = st ? kStructBit : 0;
}

__global__ void k_fixed_flags(const long long* dofs, long long nfixed, long long ndofs, uint8_t* nflags) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nfixed) return;
  const long long d = dofs[i];
  if (d < 0 || d >= ndofs) return;
  const long long n = d / 3;
  const int a = (int)(d % 3);
  unsigned int* word = (unsigned int*)((uintptr_t)(nflags + n) & ~(uintptr_t)3);
  const int shift = 8 * (int)((uintptr_t)(nflags + n) & 3);
  atomicOr(word, (1u << a) << shift);
}

cudaError_t launch_node_flags(const Grid& G, const long long* fixed_dofs, long long nfixed, const double* occ,
                              uint8_t* nflags, cudaStream_t s) {
  k_struct_flags<<<(unsigned)((G.nn + 255) / 256), 256, 0, s>>>(G, occ, nflags);
  if (nfixed > 0)
    k_fixed_flags<<<(unsigned)((nfixed + 255) / 256), 256, 0, s>>>(fixed_dofs, nfixed, 3 * G.nn, nflags);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// per-block basis: centroid + modified Gram-Schmidt (two passes) on the six
// raw masked rigid modes, tracking the transform S. One CTA per block.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void box_of(const Agglo& A, long long B, int& bx, int& by, int& bz, int& nxl, int& nyl,
                                       int& nzl) {
  bx = (int)(B % A.mx);
  by = (int)((B / A.mx) % A.my);
  bz = (int)(B / ((long long)A.mx * A.my));
  // closed node box [b*bx, min(b*bx+b, n)]
  nxl = min(A.b, A.g.nx - A.b * bx) + 1;
  nyl = min(A.b, A.g.ny - A.b * by) + 1;
  nzl = min(A.b, A.g.nz - A.b * bz) + 1;
}

// raw rigid-mode column j at (local node l, axis a) about centroid c (grid units), times h
__device__ __forceinline__ double raw_mode(int j, int a, double rx, double ry, double rz) {
  switch (j) {
    case 0: return a == 0 ? 1.0 : 0.0;
    case 1: return a == 1 ? 1.0 : 0.0;
    case 2: return a == 2 ? 1.0 : 0.0;
    case 3: return a == 1 ? -rz : (a == 2 ? ry : 0.0);  // rotation about x
    case 4: return a == 0 ? rz : (a == 2 ? -rx : 0.0);  // rotation about y
    default: return a == 0 ? -ry : (a == 1 ? rx : 0.0); // rotation about z
  }
}

constexpr int kBasisThreads = 256;

__device__ double cta_sum_bcast(double v, double* red, double* bc) {
  const double s = block_sum(v, red);
  if (threadIdx.x == 0) *bc = s;
  __syncthreads();
  const double r = *bc;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kBasisThreads) k_block_basis(Agglo A, const double* occ, const uint8_t* nflags,
                                                               DeflData D) {
  extern __shared__ double col[];  // [6][L]
  __shared__ double red[32], bc[1], Ssh[36], Rd[6];
  __shared__ int used[6];
  const long long B = blockIdx.x;
  int bx, by, bz, nxl, nyl, nzl;
  box_of(A, B, bx, by, bz, nxl, nyl, nzl);
  const Grid& G = A.g;
  const int nnl = nxl * nyl * nzl;
  const int L = 3 * nnl;
  const int X0 = A.b * bx, Y0 = A.b * by, Z0 = A.b * bz;

  // any solid element inside the block (topovox/fea.py:135)
  const int nex = nxl - 1, ney = nyl - 1, nez = nzl - 1;
  double solid = 0.0;
  for (int i = threadIdx.x; i < nex * ney * nez; i += blockDim.x) {
    const int lx = i % nex, ly = (i / nex) % ney, lz = i / (nex * ney);
    if (occ[G.elem(X0 + lx, Y0 + ly, Z0 + lz)] == 1.0) solid = 1.0;
  }
  const double nsolid = cta_sum_bcast(solid, red, bc);
  // centroid of structural nodes (fixed ones included, topovox/fea.py:138-141)
  double cnt = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
  for (int i = threadIdx.x; i < nnl; i += blockDim.x) {
    const int lx = i % nxl, ly = (i / nxl) % nyl, lz = i / (nxl * nyl);
    if (nflags[G.node(X0 + lx, Y0 + ly, Z0 + lz)] & kStructBit) {
      cnt += 1.0;
      sx += lx;
      sy += ly;
      sz += lz;
    }
  }
  cnt = cta_sum_bcast(cnt, red, bc);
  sx = cta_sum_bcast(sx, red, bc);
  sy = cta_sum_bcast(sy, red, bc);
  sz = cta_sum_bcast(sz, red, bc);
  if (nsolid == 0.0 || cnt == 0.0) {
    if (threadIdx.x < 36) D.S[36 * B + threadIdx.x] = 0.0;
    if (threadIdx.x < 3) D.cen[3 * B + threadIdx.x] = 0.0;
    if (threadIdx.x == 0) D.keep[B] = 0;
    return;
  }
  const double cx = sx / cnt, cy = sy / cnt, cz = sz / cnt;
  // raw masked columns
  for (int i = threadIdx.x; i < nnl; i += blockDim.x) {
    const int lx = i % nxl, ly = (i / nxl) % nyl, lz = i / (nxl * nyl);
    const uint8_t fl = nflags[G.node(X0 + lx, Y0 + ly, Z0 + lz)];
    const double rx = A.h * (lx - cx), ry = A.h * (ly - cy), rz = A.h * (lz - cz);
    for (int a = 0; a < 3; ++a) {
      const bool on = (fl & kStructBit) && !((fl >> a) & 1);
      for (int j = 0; j < 6; ++j) col[j * L + 3 * i + a] = on ? raw_mode(j, a, rx, ry, rz) : 0.0;
    }
  }
  if (threadIdx.x < 36) Ssh[threadIdx.x] = (threadIdx.x % 7 == 0) ? 1.0 : 0.0;  // identity, S[i + 6j]
  __syncthreads();

  for (int j = 0; j < 6; ++j) {
    double* v = col + j * L;
    double nb = 0.0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) nb = fma(v[i], v[i], nb);
    nb = sqrt(cta_sum_bcast(nb, red, bc));
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = 0; i < j; ++i) {
        if (!used[i]) continue;
        const double* qi = col + i * L;
        double d = 0.0;
        for (int k = threadIdx.x; k < L; k += blockDim.x) d = fma(qi[k], v[k], d);
        d = cta_sum_bcast(d, red, bc);
        for (int k = threadIdx.x; k < L; k += blockDim.x) v[k] = fma(-d, qi[k], v[k]);
        if (threadIdx.x < 6) Ssh[threadIdx.x + 6 * j] = fma(-d, Ssh[threadIdx.x + 6 * i], Ssh[threadIdx.x + 6 * j]);
        __syncthreads();
      }
    }
    double rn = 0.0;
    for (int k = threadIdx.x; k < L; k += blockDim.x) rn = fma(v[k], v[k], rn);
    rn = sqrt(cta_sum_bcast(rn, red, bc));
    const bool u = nb > 0.0 && rn > 1e-13 * nb;
    if (threadIdx.x == 0) {
      used[j] = u;
      Rd[j] = rn;
    }
    const double inv = u ? 1.0 / rn : 0.0;
    for (int k = threadIdx.x; k < L; k += blockDim.x) v[k] *= inv;
    if (threadIdx.x < 6) Ssh[threadIdx.x + 6 * j] *= inv;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int j = 0; j < 6; ++j) mx = fmax(mx, Rd[j]);
    int keep = 0;
    for (int j = 0; j < 6; ++j)
      if (used[j] && Rd[j] > 1e-10 * fmax(mx, 1e-300)) keep |= 1 << j;
    D.keep[B] = keep;
    bc[0] = (double)keep;
  }
  __syncthreads();
  const int keep = (int)bc[0];
  if (threadIdx.x < 36) {
    const int j = threadIdx.x / 6;
    D.S[36 * B + threadIdx.x] = ((keep >> j) & 1) ? Ssh[threadIdx.x] : 0.0;
  }
  if (threadIdx.x == 0) {
    D.cen[3 * B + 0] = cx;
    D.cen[3 * B + 1] = cy;
    D.cen[3 * B + 2] = cz;
  }
}

cudaError_t launch_block_basis(const Agglo& A, const double* occ, const uint8_t* nflags, DeflData D, cudaStream_t s) {
  const int nn = (A.b + 1) * (A.b + 1) * (A.b + 1);
  const size_t smem = sizeof(double) * 6 * 3 * (size_t)nn;
  cudaFuncSetAttribute(k_block_basis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_block_basis<<<(unsigned)A.nb, kBasisThreads, smem, s>>>(A, occ, nflags, D);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// restriction: yc_B = S_B^T [sum y~ ; sum r x y~] over structural nodes of the
// closed box, y~ = y with fixed DOFs zeroed. One CTA per block, fixed order.
// ---------------------------------------------------------------------------
constexpr int kRestrictThreads = 128;  // measured best at C4 (256 threads: +5 us per restriction)

// BS > 0: compile-time block size (the closed box has at most (BS+1)^3 nodes;
// positions outside a clipped boundary box are skipped); BS = 0: runtime size.
template <int BS>
__global__ void __launch_bounds__(kRestrictThreads) k_restrict(Agglo A, const uint8_t* __restrict__ nflags, DeflData D,
                                                               const double* __restrict__ y,
                                                               const double* __restrict__ y2, const SolverState* st,
                                                               double* yc, const int* stop) {
  pdl_entry();
  __shared__ double red[6 * (kRestrictThreads / 32)], m[6];
  if (stop != nullptr && *stop) return;
  const double beta = (y2 != nullptr) ? st->beta : 0.0;  // restrict y + beta*y2
  const long long B = blockIdx.x;
  const long long PB = D.perm != nullptr ? (long long)D.perm[B] : B;  // coarse-vector position
  const int keep = D.keep[B];
  if (keep == 0) {
    if (threadIdx.x < 6) yc[6 * PB + threadIdx.x] = 0.0;
    return;
  }
  int bx, by, bz, nxl, nyl, nzl;
  box_of(A, B, bx, by, bz, nxl, nyl, nzl);
  const Grid& G = A.g;
  const int X0 = A.b * bx, Y0 = A.b * by, Z0 = A.b * bz;
  const double cx = D.cen[3 * B], cy = D.cen[3 * B + 1], cz = D.cen[3 * B + 2];
  const int PX = BS > 0 ? BS + 1 : nxl, PY = BS > 0 ? BS + 1 : nyl, PZ = BS > 0 ? BS + 1 : nzl;
  const int npos = PX * PY * PZ;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  // up to kNodes nodes per thread per step, all their loads issued before use
  constexpr int kNodes = 4;
  for (int i0 = threadIdx.x; i0 < npos; i0 += kNodes * blockDim.x) {
    uint8_t fl[kNodes];
    double w[kNodes][3];
    int lxs[kNodes], lys[kNodes], lzs[kNodes];
#pragma unroll
    for (int k = 0; k < kNodes; ++k) {
      const int i = i0 + k * blockDim.x;
      const int lx = i % PX, ly = (i / PX) % PY, lz = i / (PX * PY);
      lxs[k] = lx;
      lys[k] = ly;
      lzs[k] = lz;
      fl[k] = 0;
      w[k][0] = w[k][1] = w[k][2] = 0.0;
      if (i < npos && lx < nxl && ly < nyl && lz < nzl) {
        const long long n = G.node(X0 + lx, Y0 + ly, Z0 + lz);
        fl[k] = __ldg(nflags + n);
        w[k][0] = __ldg(y + 3 * n);
        w[k][1] = __ldg(y + 3 * n + 1);
        w[k][2] = __ldg(y + 3 * n + 2);
        if (y2 != nullptr) {
          w[k][0] = fma(beta, __ldg(y2 + 3 * n), w[k][0]);
          w[k][1] = fma(beta, __ldg(y2 + 3 * n + 1), w[k][1]);
          w[k][2] = fma(beta, __ldg(y2 + 3 * n + 2), w[k][2]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kNodes; ++k) {
      if (!(fl[k] & kStructBit)) continue;  // also covers positions outside the box (fl = 0)
      const double vx = (fl[k] & 1) ? 0.0 : w[k][0];
      const double vy = (fl[k] & 2) ? 0.0 : w[k][1];
      const double vz = (fl[k] & 4) ? 0.0 : w[k][2];
      const double rx = A.h * (lxs[k] - cx), ry = A.h * (lys[k] - cy), rz = A.h * (lzs[k] - cz);
      acc[0] += vx;
      acc[1] += vy;
      acc[2] += vz;
      acc[3] += ry * vz - rz * vy;
      acc[4] += rz * vx - rx * vz;
      acc[5] += rx * vy - ry * vx;
    }
  }
  // the six moment sums reduced together: warp trees, then 6 threads sum the
  // per-warp values in warp order (one barrier)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double s = warp_sum(acc[k]);
    if (lane == 0) red[6 * wid + k] = s;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[6 * w + threadIdx.x];
    m[threadIdx.x] = s;
  }
  __syncwarp();
  if (threadIdx.x < 6) {
    const int j = threadIdx.x;
    const double* S = D.S + 36 * B;
    double v = 0.0;
    for (int i = 0; i < 6; ++i) v = fma(S[i + 6 * j], m[i], v);
    yc[6 * PB + j] = v;
  }
}

// Warp-per-block variant: a 256-thread CTA restricts 8 blocks, one warp each
// (lane-strided over the block's closed node box, 4 nodes' loads in flight per
// lane, warp-shuffle trees, no shared memory or CTA barrier). Small blocks
// (b = 4: 125 nodes) left the one-CTA-per-block kernel launch/latency-bound
// (32768 CTAs of 128 threads at C2(b)).
constexpr int kRestrictWarpThreads = 256;

template <int BS>
__global__ void __launch_bounds__(kRestrictWarpThreads) k_restrict_warp(Agglo A, const uint8_t* __restrict__ nflags,
                                                                        DeflData D, const double* __restrict__ y,
                                                                        const double* __restrict__ y2,
                                                                        const SolverState* st, double* yc,
                                                                        const int* stop) {
  pdl_entry();
  if (stop != nullptr && *stop) return;
  const int lane = threadIdx.x & 31;
  const long long B = (long long)blockIdx.x * (kRestrictWarpThreads / 32) + (threadIdx.x >> 5);
  if (B >= A.nb) return;
  const double beta = (y2 != nullptr) ? st->beta : 0.0;  // restrict y + beta*y2
  const long long PB = D.perm != nullptr ? (long long)D.perm[B] : B;
  const int keep = D.keep[B];
  if (keep == 0) {
    if (lane < 6) yc[6 * PB + lane] = 0.0;
    return;
  }
  int bx, by, bz, nxl, nyl, nzl;
  box_of(A, B, bx, by, bz, nxl, nyl, nzl);
  const Grid& G = A.g;
  const int X0 = A.b * bx, Y0 = A.b * by, Z0 = A.b * bz;
  const double cx = D.cen[3 * B], cy = D.cen[3 * B + 1], cz = D.cen[3 * B + 2];
  const int PX = BS > 0 ? BS + 1 : nxl, PY = BS > 0 ? BS + 1 : nyl, PZ = BS > 0 ? BS + 1 : nzl;
  const int npos = PX * PY * PZ;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  constexpr int kNodes = 4;
  for (int i0 = lane; i0 < npos; i0 += kNodes * 32) {
    uint8_t fl[kNodes];
    double w[kNodes][3];
    int lxs[kNodes], lys[kNodes], lzs[kNodes];
#pragma unroll
    for (int k = 0; k < kNodes; ++k) {
      const int i = i0 + k * 32;
      const int lx = i % PX, ly = (i / PX) % PY, lz = i / (PX * PY);
      lxs[k] = lx;
      lys[k] = ly;
      lzs[k] = lz;
      fl[k] = 0;
      w[k][0] = w[k][1] = w[k][2] = 0.0;
      if (i < npos && lx < nxl && ly < nyl && lz < nzl) {
        const long long n = G.node(X0 + lx, Y0 + ly, Z0 + lz);
        fl[k] = __ldg(nflags + n);
        w[k][0] = __ldg(y + 3 * n);
        w[k][1] = __ldg(y + 3 * n + 1);
        w[k][2] = __ldg(y + 3 * n + 2);
        if (y2 != nullptr) {
          w[k][0] = fma(beta, __ldg(y2 + 3 * n), w[k][0]);
          w[k][1] = fma(beta, __ldg(y2 + 3 * n + 1), w[k][1]);
          w[k][2] = fma(beta, __ldg(y2 + 3 * n + 2), w[k][2]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kNodes; ++k) {
      if (!(fl[k] & kStructBit)) continue;
      const double vx = (fl[k] & 1) ? 0.0 : w[k][0];
      const double vy = (fl[k] & 2) ? 0.0 : w[k][1];
      const double vz = (fl[k] & 4) ? 0.0 : w[k][2];
      const double rx = A.h * (lxs[k] - cx), ry = A.h * (lys[k] - cy), rz = A.h * (lzs[k] - cz);
      acc[0] += vx;
      acc[1] += vy;
      acc[2] += vz;
      acc[3] += ry * vz - rz * vy;
      acc[4] += rz * vx - rx * vz;
      acc[5] += rx * vy - ry * vx;
    }
  }
  double m[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) m[k] = __shfl_sync(0xffffffffu, warp_sum(acc[k]), 0);
  if (lane < 6) {
    const double* S = D.S + 36 * B;
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < 6; ++i) v = fma(S[i + 6 * lane], m[i], v);
    yc[6 * PB + lane] = v;
  }
}

cudaError_t launch_restrict(const Agglo& A, const uint8_t* nflags, DeflData D, const double* y, double* yc,
                            cudaStream_t s, const int* stop, const double* y2, const void* state) {
  const SolverState* st = (const SolverState*)state;
  static int mode = -1;  // TVB_RESTRICT=cta|warp (A/B); default: warp per block below 8^3 blocks when there are > 1000
  if (mode < 0) {
    const char* e = getenv("TVB_RESTRICT");
    mode = e == nullptr ? 0 : (e[0] == 'w' ? 1 : 2);
  }
  // few small blocks (C1: 250): one CTA per block spreads them over the SMs (C1 solve 5.29 -> 5.11 ms);
  // at C3's 2000 blocks the warp-per-block kernel is ahead again (113.4 vs 115.2 us per iteration)
  const bool warp = mode == 1 || (mode == 0 && A.b < 8 && A.nb > 1000);
  if (warp) {
    const unsigned gw = (unsigned)((A.nb + 7) / 8);
    if (A.b == 8) launch_k(k_restrict_warp<8>, gw, kRestrictWarpThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
    else if (A.b == 4) launch_k(k_restrict_warp<4>, gw, kRestrictWarpThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
    else launch_k(k_restrict_warp<0>, gw, kRestrictWarpThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
    return cudaGetLastError();
  }
  const unsigned g = (unsigned)A.nb;
  if (A.b == 8) launch_k(k_restrict<8>, g, kRestrictThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
  else if (A.b == 4) launch_k(k_restrict<4>, g, kRestrictThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
  else launch_k(k_restrict<0>, g, kRestrictThreads, 0, s, A, nflags, D, y, y2, st, yc, stop);
  return cudaGetLastError();
}

// nu_B = S_B mu_B
__global__ void k_block_nu(long long nb, const double* S, const int* perm, const double* mu, double* nu,
                           const int* stop) {
  pdl_entry();
  if (stop != nullptr && *stop) return;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 6 * nb) return;
  const long long B = t / 6;
  const long long PB = perm != nullptr ? (long long)perm[B] : B;
  const int i = (int)(t % 6);
  double v = 0.0;
  for (int j = 0; j < 6; ++j) v = fma(S[36 * B + i + 6 * j], mu[6 * PB + j], v);
  nu[t] = v;
}

cudaError_t launch_block_nu(const Agglo& A, DeflData D, const double* mu, double* nu, cudaStream_t s,
                            const int* stop) {
  launch_k(k_block_nu, (unsigned)((6 * A.nb + 255) / 256), 256, 0, s, A.nb, D.S, D.perm, mu, nu, stop);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// prolongation: (W mu)_n = sum_{B containing n} mask(t_B + omega_B x r_{n,B})
// ---------------------------------------------------------------------------
// One thread per node (1-D grid, 32-bit index math: Nn < 2^31). All loads of
// the node (flags, p, z) are issued before the rigid-motion evaluation.
// BS > 0: compile-time block size (divisions by BS become shifts / mul-hi).
constexpr int kProlongThreads = 128;  // measured best at C4 (256: +2 us)

template <int BS>
__global__ void __launch_bounds__(kProlongThreads) k_prolong(Agglo A, const uint8_t* __restrict__ nflags,
                                                 const double* __restrict__ cen, const double* __restrict__ nu,
                                                 double* __restrict__ out, const double* __restrict__ z,
                                                 double* __restrict__ x, const SolverState* st, int mode) {
  pdl_entry();
  const Grid& G = A.g;
  const unsigned n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= (unsigned)G.nn) return;
  if (st != nullptr && st->done) return;
  const uint8_t fl = nflags[n];
  double o[3] = {0.0, 0.0, 0.0}, zv[3] = {0.0, 0.0, 0.0};
  if (mode != 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) zv[a] = z[3ull * n + a];
  }
  if (mode == 1) {
#pragma unroll
    for (int a = 0; a < 3; ++a) o[a] = out[3ull * n + a];
  }
  double v[3] = {0.0, 0.0, 0.0};
  if (fl & kStructBit) {
    const unsigned px = (unsigned)G.px, py = (unsigned)G.py;
    const unsigned t = n / px;
    const unsigned zu = t / py;
    const int x = (int)(n - t * px), y = (int)(t - zu * py), zz = (int)zu;
    const int b = BS > 0 ? BS : A.b;
    int bxs[2], bys[2], bzs[2], nbx = 0, nby = 0, nbz = 0;
    // blocks whose closed box contains the coordinate, ascending
    if (x % b == 0 && x > 0 && x / b - 1 < A.mx) bxs[nbx++] = x / b - 1;
    if (x / b < A.mx) bxs[nbx++] = x / b;
    if (y % b == 0 && y > 0 && y / b - 1 < A.my) bys[nby++] = y / b - 1;
    if (y / b < A.my) bys[nby++] = y / b;
    if (zz % b == 0 && zz > 0 && zz / b - 1 < A.mz) bzs[nbz++] = zz / b - 1;
    if (zz / b < A.mz) bzs[nbz++] = zz / b;
    for (int k = 0; k < nbz; ++k)
      for (int j = 0; j < nby; ++j)
        for (int i = 0; i < nbx; ++i) {
          // nu_B = S_B mu_B is exactly zero for inactive blocks (S_B == 0): no keep lookup
          const long long B = bxs[i] + (long long)A.mx * (bys[j] + (long long)A.my * bzs[k]);
          const double* w = nu + 6 * B;
          const double rx = A.h * (x - b * bxs[i] - cen[3 * B]);
          const double ry = A.h * (y - b * bys[j] - cen[3 * B + 1]);
          const double rz = A.h * (zz - b * bzs[k] - cen[3 * B + 2]);
          v[0] += w[0] + (w[4] * rz - w[5] * ry);
          v[1] += w[1] + (w[5] * rx - w[3] * rz);
          v[2] += w[2] + (w[3] * ry - w[4] * rx);
        }
    for (int a = 0; a < 3; ++a)
      if ((fl >> a) & 1) v[a] = 0.0;
  }
  const double beta = mode == 1 ? st->beta : 0.0;
  if (mode == 1 && x != nullptr) {  // deferred x += alpha p_old of this iteration (p_old = o)
    const double alpha = st->alpha;
#pragma unroll
    for (int a = 0; a < 3; ++a) x[3ull * n + a] = fma(alpha, o[a], x[3ull * n + a]);
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double r = mode == 0 ? v[a] : (mode == 1 ? fma(beta, o[a], zv[a]) - v[a] : zv[a] - v[a]);
    out[3ull * n + a] = r;
  }
}

cudaError_t launch_prolong(const Agglo& A, const uint8_t* nflags, DeflData D, const double* nu, double* out,
                           const double* z, const void* state, int mode, cudaStream_t s, double* x) {
  const unsigned g = (unsigned)((A.g.nn + kProlongThreads - 1) / kProlongThreads);
  const SolverState* st = (const SolverState*)state;
  if (A.b == 8) launch_k(k_prolong<8>, g, kProlongThreads, 0, s, A, nflags, D.cen, nu, out, z, x, st, mode);
  else if (A.b == 4) launch_k(k_prolong<4>, g, kProlongThreads, 0, s, A, nflags, D.cen, nu, out, z, x, st, mode);
  else launch_k(k_prolong<0>, g, kProlongThreads, 0, s, A, nflags, D.cen, nu, out, z, x, st, mode);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Galerkin coarse operator by probing. Blocks are 3-coloured per axis
// (27 colours); two blocks of one colour are >= 3 apart along some axis, so
// A W_C for one colour never reaches another same-colour block's box
// (block size >= 2). One probe (colour, mode j) yields E[B, C][:, j] for
// every block B and its unique colour-k neighbour C.
// Eb layout: [B][27 neighbour slots d = (dx+1) + 3(dy+1) + 9(dz+1)][6 i][6 j].
// ---------------------------------------------------------------------------
__device__ __forceinline__ int color_of(int bx, int by, int bz) { return bx % 3 + 3 * (by % 3) + 9 * (bz % 3); }

__global__ void k_probe_nu(Agglo A, const double* S, int color, int j, double* nu) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 6 * A.nb) return;
  const long long B = t / 6;
  const int i = (int)(t % 6);
  const int bx = (int)(B % A.mx), by = (int)((B / A.mx) % A.my), bz = (int)(B / ((long long)A.mx * A.my));
  nu[t] = (color_of(bx, by, bz) == color) ? S[36 * B + i + 6 * j] : 0.0;
}

cudaError_t launch_probe_nu(const Agglo& A, DeflData D, int color, int j, double* nu, cudaStream_t s) {
  k_probe_nu<<<(unsigned)((6 * A.nb + 255) / 256), 256, 0, s>>>(A, D.S, color, j, nu);
  return cudaGetLastError();
}

__global__ void k_probe_scatter(Agglo A, int color, int j, const double* yc, double* Eb) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= 6 * A.nb) return;
  const long long B = t / 6;
  const int i = (int)(t % 6);
  const int bx = (int)(B % A.mx), by = (int)((B / A.mx) % A.my), bz = (int)(B / ((long long)A.mx * A.my));
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int cx = bx + dx, cy = by + dy, cz = bz + dz;
        if (cx < 0 || cx >= A.mx || cy < 0 || cy >= A.my || cz < 0 || cz >= A.mz) continue;
        if (color_of(cx, cy, cz) != color) continue;
        const int d = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
        Eb[((B * 27 + d) * 6 + i) * 6 + j] = yc[6 * B + i];
      }
}

cudaError_t launch_probe_scatter(const Agglo& A, int color, int j, const double* yc, double* Eb, cudaStream_t s) {
  k_probe_scatter<<<(unsigned)((6 * A.nb + 255) / 256), 256, 0, s>>>(A, color, j, yc, Eb);
  return cudaGetLastError();
}

// Es = (Eb + Eb^T)/2 (topovox/fea.py:198); dropped / inactive coarse DOFs get
// a unit diagonal so the block-regular coarse system stays SPD.
__global__ void k_coarse_finish(Agglo A, const int* keepv, const double* Eb, double* Es) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= A.nb * 27 * 36) return;
  const long long B = t / (27 * 36);
  const int d = (int)((t / 36) % 27);
  const int i = (int)((t / 6) % 6), j = (int)(t % 6);
  const int bx = (int)(B % A.mx), by = (int)((B / A.mx) % A.my), bz = (int)(B / ((long long)A.mx * A.my));
  const int dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
  const int cx = bx + dx, cy = by + dy, cz = bz + dz;
  double v = 0.0;
  if (cx >= 0 && cx < A.mx && cy >= 0 && cy < A.my && cz >= 0 && cz < A.mz) {
    const long long C = cx + (long long)A.mx * (cy + (long long)A.my * cz);
    const int dt = 26 - d;
    v = 0.5 * (Eb[t] + Eb[((C * 27 + dt) * 6 + j) * 6 + i]);
    if (d == 13 && i == j && !((keepv[B] >> i) & 1)) v = 1.0;
  }
  Es[t] = v;
}

cudaError_t launch_coarse_finish(const Agglo& A, DeflData D, const double* Eb, double* Es, cudaStream_t s) {
  const long long n = A.nb * 27 * 36;
  k_coarse_finish<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A, D.keep, Eb, Es);
  return cudaGetLastError();
}

// dense n_c x n_c copy of the block stencil (small coarse spaces only)
__global__ void k_coarse_dense(Agglo A, const double* Es, double* Ed) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= A.nb * 27 * 36) return;
  const long long B = t / (27 * 36);
  const int d = (int)((t / 36) % 27);
  const int i = (int)((t / 6) % 6), j = (int)(t % 6);
  const int bx = (int)(B % A.mx), by = (int)((B / A.mx) % A.my), bz = (int)(B / ((long long)A.mx * A.my));
  const int cx = bx + d % 3 - 1, cy = by + (d / 3) % 3 - 1, cz = bz + d / 9 - 1;
  if (cx < 0 || cx >= A.mx || cy < 0 || cy >= A.my || cz < 0 || cz >= A.mz) return;
  const long long C = cx + (long long)A.mx * (cy + (long long)A.my * cz);
  const long long nc = 6 * A.nb;
  Ed[(6 * B + i) * nc + 6 * C + j] = Es[t];
}

cudaError_t launch_coarse_dense(const Agglo& A, const double* Es, double* Ed, cudaStream_t s) {
  const long long n = A.nb * 27 * 36;
  k_coarse_dense<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(A, Es, Ed);
  return cudaGetLastError();
}

}  // namespace tvb
