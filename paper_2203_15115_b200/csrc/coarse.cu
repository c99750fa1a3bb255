// a7: per-iteration coarse solve E mu = y with the nested-dissection factor
// built by paper_2203_15115_b200/coarse.py. Replaces the dense
// scipy.linalg.cho_solve of DeflationSpace.coarse_solve (topovox/fea.py:208-211).
// Vectors are in ND order (every separator a contiguous DOF range).
//
// Bottom tree node N (separator S, update set U, front F = S u U):
//   forward  (heights 0..H0-1): f_S = y_S + sum_children c_child|S,
//                               f_U =       sum_children c_child|U,
//                               c_U = f_U - G f_S            (G = F_US F_SS^-1)
//   backward (heights H0-1..0): x_S = [Z | -G^T] [f_S ; x_U]  (Z = F_SS^-1)
// Top set T (heights >= H0): x_T = S_T^-1 (y_T + sum_children c_child|T).
//
// The solve is latency-bound (12k-200k coarse DOFs, a few MB of factor per
// level), so it is built for short dependency chains:
//   * front vectors are GATHERED: each front position lists the update-vector
//     entries of (at most two) children, so assembly has no barriers, atomics
//     or serial child loops (the fixed child order keeps it deterministic);
//   * work items are (node, row chunk) pairs for one 256-thread CTA; long rows
//     are split across WPR = 1/2/4/8 warps (8/WPR rows per CTA), every warp a
//     fixed-order lane-strided dot product + shuffle tree, the WPR parts summed
//     in order through shared memory;
//   * default schedule = ONE persistent dataflow kernel (k_coarse_flow): CTAs
//     pull items in topological order from an atomic counter; each item waits
//     (acquire) on one counter -- its children finished (forward), its parent
//     finished (backward) -- and on completion bumps its node's counter, the
//     last finisher releasing the dependants. No grid-wide barrier and no
//     launch gap between tree levels; an item only ever waits on items with a
//     smaller index, all of which are held by running CTAs, so it cannot
//     deadlock. Counters are epoch-based (never reset).
//   * fallback schedule (items == nullptr): one launch per tree level.
// Bitwise reproducible run to run (the arithmetic of an item does not depend
// on which CTA runs it or when).
#include <algorithm>
#include <cstdio>

#include "coarse.cuh"

namespace tvb {

constexpr int kCoarseThreads = 256;
constexpr int kCoarseWarps = kCoarseThreads / 32;
constexpr int kRedStride = 4 * kCoarseWarps;  // per-column slice of the row-reduction scratch

enum CoarseItem : int { kFwd = 0, kAsm = 1, kRows = 2, kTopGather = 3, kTopRows = 4, kBwd = 5 };

// Multi-RHS: every kernel below is templated on MC, the number of right-hand
// sides solved together (1..kCoarseMaxCols). A factor row is loaded once and
// dotted with all MC columns; the arithmetic of each column is exactly the
// single-column sequence (same accumulators, same order), so a column of a
// batched solve is bitwise equal to the same vector solved alone.
struct ColSet {
  const double* y;   // column c at y + c * ldy (ND order)
  long long ldy;
  double* x;         // column c at x + c * ldx
  long long ldx;
  const int* stop;   // column c stopped <=> stop[c * stop_ld] != 0 (nullptr: never)
  long long stop_ld;
};

template <int MC>
__device__ __forceinline__ bool all_stopped(const ColSet& C) {
  if (C.stop == nullptr) return false;
#pragma unroll
  for (int c = 0; c < MC; ++c)
    if (!C.stop[c * C.stop_ld]) return false;
  return true;
}

// Part `part` of row . vector (lane-strided over WPR warps), row streamed from
// global memory with 8 independent loads in flight per lane; MC vectors at
// stride ldb.
template <int WPR, int MC>
__device__ __forceinline__ void part_dot(const double* __restrict__ a, const double* b, int ldb, int n, int part,
                                         int lane, double (&out)[MC]) {
  constexpr int st = 32 * WPR;
  double s[MC][4];
#pragma unroll
  for (int c = 0; c < MC; ++c) s[c][0] = s[c][1] = s[c][2] = s[c][3] = 0.0;
  int i = part * 32 + lane;
  for (; i + 7 * st < n; i += 8 * st) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(a + i + st * k);
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const double* bc = b + c * ldb;
      s[c][0] = fma(v[0], bc[i], s[c][0]);
      s[c][1] = fma(v[1], bc[i + st], s[c][1]);
      s[c][2] = fma(v[2], bc[i + 2 * st], s[c][2]);
      s[c][3] = fma(v[3], bc[i + 3 * st], s[c][3]);
      s[c][0] = fma(v[4], bc[i + 4 * st], s[c][0]);
      s[c][1] = fma(v[5], bc[i + 5 * st], s[c][1]);
      s[c][2] = fma(v[6], bc[i + 6 * st], s[c][2]);
      s[c][3] = fma(v[7], bc[i + 7 * st], s[c][3]);
    }
  }
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = (i + st * k < n) ? __ldg(a + i + st * k) : 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (i + st * k < n)
#pragma unroll
      for (int c = 0; c < MC; ++c) s[c][0] = fma(v[k], b[c * ldb + i + st * k], s[c][0]);
#pragma unroll
  for (int c = 0; c < MC; ++c) out[c] = warp_sum((s[c][0] + s[c][1]) + (s[c][2] + s[c][3]));
}

// RPW rows at once by one warp (WPR = 1): 8 loads in flight per lane split
// over the rows. out[q][c] = row q . b_c (full warp sum).
template <int RPW, int MC>
__device__ __forceinline__ void multi_dot(const double* __restrict__ a, long long n, const double* b, int ldb,
                                          int lane, double (&out)[RPW][MC]) {
  constexpr int K = 8 / RPW;
  double s[RPW][MC][2];
#pragma unroll
  for (int q = 0; q < RPW; ++q)
#pragma unroll
    for (int c = 0; c < MC; ++c) s[q][c][0] = s[q][c][1] = 0.0;
  int i = lane;
  for (; i + (K - 1) * 32 < n; i += K * 32) {
    double w[RPW][K];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int k = 0; k < K; ++k) w[q][k] = __ldg(a + q * n + i + 32 * k);
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int c = 0; c < MC; ++c) s[q][c][k & 1] = fma(w[q][k], b[c * ldb + i + 32 * k], s[q][c][k & 1]);
  }
  for (; i < n; i += 32)
#pragma unroll
    for (int q = 0; q < RPW; ++q) {
      const double aq = __ldg(a + q * n + i);
#pragma unroll
      for (int c = 0; c < MC; ++c) s[q][c][0] = fma(aq, b[c * ldb + i], s[q][c][0]);
    }
#pragma unroll
  for (int q = 0; q < RPW; ++q)
#pragma unroll
    for (int c = 0; c < MC; ++c) out[q][c] = warp_sum(s[q][c][0] + s[q][c][1]);
}

// Rows r0 .. r0 + 8*RPW/WPR - 1 (< r1) of M (row length n) dotted with the
// MC shared vectors v + c*ldv: WPR warps per row (RPW = 1) or RPW rows per
// warp (WPR = 1). Leaves the full dots in d[] of threads t < 8*RPW/WPR (row
// r0 + t). red: MC * kRedStride doubles.
template <int WPR, int RPW, int MC>
__device__ __forceinline__ void rows_dot(const double* __restrict__ M, long long n, const double* v, int ldv, int r0,
                                         int r1, double* red, double (&d)[MC]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (RPW == 1) {
    const int j = r0 + warp / WPR;
    double p[MC];
    if (j < r1) {
      part_dot<WPR, MC>(M + (long long)j * n, v, ldv, (int)n, warp % WPR, lane, p);
    } else {
#pragma unroll
      for (int c = 0; c < MC; ++c) p[c] = 0.0;
    }
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < MC; ++c) red[c * kRedStride + warp] = p[c];
  } else {
    const int j0 = r0 + warp * RPW;
    double p[RPW][MC];
#pragma unroll
    for (int q = 0; q < RPW; ++q)
#pragma unroll
      for (int c = 0; c < MC; ++c) p[q][c] = 0.0;
    if (j0 < r1) {
      const int jl = min(j0 + RPW, r1) - j0;
      if (jl == RPW) {
        multi_dot<RPW, MC>(M + (long long)j0 * n, n, v, ldv, lane, p);
      } else {
        for (int q = 0; q < jl; ++q) {
          double t1[1][MC];
          multi_dot<1, MC>(M + (long long)(j0 + q) * n, n, v, ldv, lane, t1);
#pragma unroll
          for (int c = 0; c < MC; ++c) p[q][c] = t1[0][c];
        }
      }
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < RPW; ++q)
#pragma unroll
        for (int c = 0; c < MC; ++c) red[c * kRedStride + warp * RPW + q] = p[q][c];
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < MC; ++c) d[c] = 0.0;
  if (threadIdx.x < kCoarseWarps * RPW / WPR) {
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      if (RPW == 1) {
#pragma unroll
        for (int k = 0; k < WPR; ++k) d[c] += red[c * kRedStride + threadIdx.x * WPR + k];
      } else {
        d[c] = red[c * kRedStride + threadIdx.x];
      }
    }
  }
}

// mode = WPR | RPW << 4 (RPW 0 or 1 = one row per warp)
__device__ __forceinline__ int mode_rows(int mode) {
  const int wpr = mode & 15, rpw = max(1, mode >> 4);
  return kCoarseWarps * rpw / wpr;
}

template <int MC>
__device__ __forceinline__ void rows_dot_w(int mode, const double* __restrict__ M, long long n, const double* v,
                                           int ldv, int r0, int r1, double* red, double (&d)[MC]) {
  switch (mode) {
    case 1: rows_dot<1, 1, MC>(M, n, v, ldv, r0, r1, red, d); break;
    case 2: rows_dot<2, 1, MC>(M, n, v, ldv, r0, r1, red, d); break;
    case 4: rows_dot<4, 1, MC>(M, n, v, ldv, r0, r1, red, d); break;
    case 8: rows_dot<8, 1, MC>(M, n, v, ldv, r0, r1, red, d); break;
    case 1 | (2 << 4): rows_dot<1, 2, MC>(M, n, v, ldv, r0, r1, red, d); break;
    default: rows_dot<1, 4, MC>(M, n, v, ldv, r0, r1, red, d); break;
  }
}

// front position p of a node, column c: base + child-0 entry + child-1 entry
// (fixed order). cU is written during the solve: read through L2 (__ldcg).
__device__ __forceinline__ double gather_front(const CoarseNDDev& D, long long gm, int p, double base, int c) {
  const int g0 = __ldg(D.gmap + gm + 2 * p), g1 = __ldg(D.gmap + gm + 2 * p + 1);
  const double* cu = D.cU + c * D.cu_ld;
  if (g0 >= 0) base += __ldcg(cu + g0);
  if (g1 >= 0) base += __ldcg(cu + g1);
  return base;
}

// dst[i] = f(i) for i < n with 8 independent element loads in flight per
// thread (all loads of a batch are issued before any store).
template <typename F, typename S>
__device__ __forceinline__ void batched(int n, F f, S store) {
  for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * blockDim.x;
      v[k] = i < n ? f(i) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * blockDim.x;
      if (i < n) store(i, v[k]);
    }
  }
}

template <typename F>
__device__ __forceinline__ void fill_batched(double* dst, int n, F f) {
  batched(n, f, [&](int i, double v) { dst[i] = v; });
}

// ---- item bodies (all threads of the CTA; contain __syncthreads) ----------

// A bottom node's layout (meta row: s, u, g_off, b_off, sd_off, ud_off, gm_off).
struct NodeInfo {
  int s, u;
  long long g_off, b_off, sd_off, ud_off, gm;
};

__device__ __forceinline__ NodeInfo node_info(const long long* __restrict__ m) {
  NodeInfo n;
  n.s = (int)__ldg(m);
  n.u = (int)__ldg(m + 1);
  n.g_off = __ldg(m + 2);
  n.b_off = __ldg(m + 3);
  n.sd_off = __ldg(m + 4);
  n.ud_off = __ldg(m + 5);
  n.gm = __ldg(m + 6);
  return n;
}

// per-launch item record (level schedule): the node's meta row + rows [r0, r1),
// 10 x int64, read with independent 16-byte loads (one round trip)
__device__ __forceinline__ NodeInfo item_record(const long long* __restrict__ rec, int& r0, int& r1) {
  const longlong2* q = reinterpret_cast<const longlong2*>(rec);
  const longlong2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3), e = __ldg(q + 4);
  NodeInfo n;
  n.s = (int)a.x;
  n.u = (int)a.y;
  n.g_off = b.x;
  n.b_off = b.y;
  n.sd_off = c.x;
  n.ud_off = c.y;
  n.gm = d.x;
  r0 = (int)e.x;
  r1 = (int)e.y;
  return n;
}

// Forward rows: c_U[j] = f_U[j] - G[j,:] f_S. assembled: f_S / f_U were written
// by the node's assembly item; else gathered here (the node's first item
// also stores f_S for the backward pass). fs: MC x s shared doubles.
template <int MC>
__device__ __forceinline__ void item_fwd(const CoarseNDDev& D, bool assembled, int wpr, const NodeInfo& n, int r0,
                                         int r1, const ColSet& C, double* fs, double* red) {
  const int s = n.s;
  const long long g_off = n.g_off, sd_off = n.sd_off, ud_off = n.ud_off, gm = n.gm;
  if (assembled) {
    fill_batched(fs, MC * s, [&](int i) {
      const int c = i / s, k = i - c * s;
      return __ldcg(D.fS + c * D.fs_ld + sd_off + k);
    });
  } else {
    fill_batched(fs, MC * s, [&](int i) {
      const int c = i / s, k = i - c * s;
      return gather_front(D, gm, k, C.y[c * C.ldy + sd_off + k], c);
    });
    if (r0 == 0)
      for (int i = threadIdx.x; i < MC * s; i += blockDim.x) {  // own writes: no barrier
        const int c = i / s, k = i - c * s;
        D.fS[c * D.fs_ld + sd_off + k] = fs[i];
      }
  }
  __syncthreads();
  double d[MC];
  rows_dot_w<MC>(wpr, D.G + g_off, s, fs, s, r0, r1, red, d);
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < mode_rows(wpr) && j < r1) {
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const double fu = assembled ? __ldcg(D.cU + c * D.cu_ld + ud_off + j) : gather_front(D, gm, s + j, 0.0, c);
      D.cU[c * D.cu_ld + ud_off + j] = fu - d[c];
    }
  }
}

// Large fronts, assembly: f_S -> fS, f_U -> cU (whole node, all columns).
template <int MC>
__device__ __forceinline__ void item_asm(const CoarseNDDev& D, const NodeInfo& n, const ColSet& C) {
  const int s = n.s, u = n.u, f = s + u;
  const long long sd_off = n.sd_off, ud_off = n.ud_off, gm = n.gm;
  batched(
      MC * f,
      [&](int i) {
        const int c = i / f, p = i - c * f;
        return gather_front(D, gm, p, p < s ? C.y[c * C.ldy + sd_off + p] : 0.0, c);
      },
      [&](int i, double v) {
        const int c = i / f, p = i - c * f;
        if (p < s) D.fS[c * D.fs_ld + sd_off + p] = v;
        else D.cU[c * D.cu_ld + ud_off + p - s] = v;
      });
}

// Backward rows: x_S[j] = [Z | -G^T][j,:] . [f_S ; x_U]. v: MC x (s+u) shared.
template <int MC>
__device__ __forceinline__ void item_bwd(const CoarseNDDev& D, int wpr, const NodeInfo& n, int r0, int r1,
                                         const ColSet& C, double* v, double* red) {
  const int s = n.s, u = n.u, f = s + u;
  const long long b_off = n.b_off, sd_off = n.sd_off, ud_off = n.ud_off;
  fill_batched(v, MC * f, [&](int i) {
    const int c = i / f, k = i - c * f;
    return k < s ? __ldcg(D.fS + c * D.fs_ld + sd_off + k) : __ldcg(C.x + c * C.ldx + __ldg(D.udof + ud_off + k - s));
  });
  __syncthreads();
  double d[MC];
  rows_dot_w<MC>(wpr, D.B + b_off, f, v, f, r0, r1, red, d);
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < mode_rows(wpr) && j < r1)
#pragma unroll
    for (int c = 0; c < MC; ++c) C.x[c * C.ldx + sd_off + j] = d[c];
}

// Top set, gather: fT[i] = y_T[i] + children's update entries (CSR, fixed order).
template <int MC>
__device__ __forceinline__ void item_top_gather(const CoarseNDDev& D, int i0, int i1, const ColSet& C) {
  const int i = i0 + threadIdx.x;
  if (i >= i1) return;
  const int a = __ldg(D.tptr + i), b = __ldg(D.tptr + i + 1);
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    double v = C.y[c * C.ldy + D.top_off + i];
    for (int k = a; k < b; ++k) v += __ldcg(D.cU + c * D.cu_ld + __ldg(D.tidx + k));
    D.fT[c * D.ft_ld + i] = v;
  }
}

// Top set, rows: x_T = S_T^-1 fT. ft: MC x n_top shared.
// Per-level schedule: the top vector is read straight from global memory
// (L1/L2-resident, written by the previous gather launch; kernel boundaries
// make it coherent) -- staging it per CTA cost a serial fill + barrier in each
// of the ~500 CTAs of this latency-bound launch. The persistent dataflow
// kernel stages it through L2 (__ldcg): fT is written by other CTAs of the
// same launch, so L1 could hold stale lines.
template <int MC>
__device__ __forceinline__ void item_top_rows(const CoarseNDDev& D, int wpr, int r0, int r1, const ColSet& C,
                                              double* ft, double* red, bool stage) {
  const int n = D.n_top;
  double d[MC];
  if (stage) {
    fill_batched(ft, MC * n, [&](int i) {
      const int c = i / n, k = i - c * n;
      return __ldcg(D.fT + c * D.ft_ld + k);
    });
    __syncthreads();
    rows_dot_w<MC>(wpr, D.ZT, n, ft, n, r0, r1, red, d);
  } else {
    rows_dot_w<MC>(wpr, D.ZT, n, D.fT, (int)D.ft_ld, r0, r1, red, d);
  }
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < mode_rows(wpr) && j < r1)
#pragma unroll
    for (int c = 0; c < MC; ++c) C.x[c * C.ldx + D.top_off + j] = d[c];
}

// ---- packed symmetric top: x_T = S_T^-1 f_T from the lower tiles -----------
// Tile (I, J), J <= I, is read once and serves both products it appears in:
// rows  P[I][J] = T_IJ f_J            (64 partials of block row I)
// cols  P[J][I] = T_IJ^T f_I  (J < I) (64 partials of block row J)
// and k_top_reduce sums x_I = sum_J P[I][J] in J order. Half the bytes of the
// dense inverse; fixed summation order (deterministic).
constexpr int kTopTile = 64;

__device__ __forceinline__ void tile_ij(long long t, int& I, int& J) {
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((long long)(i + 1) * (i + 2) / 2 <= t) ++i;
  while ((long long)i * (i + 1) / 2 > t) --i;
  I = i;
  J = (int)(t - (long long)i * (i + 1) / 2);
}

template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_top_tiles(CoarseNDDev D, ColSet C) {
  pdl_entry();
  __shared__ double colp[kCoarseWarps][MC][kTopTile];
  if (all_stopped<MC>(C)) return;
  int I, J;
  tile_ij(blockIdx.x, I, J);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = D.n_top, nt = D.top_tiles;
  const double* T = D.ZT + (long long)blockIdx.x * kTopTile * kTopTile;
  constexpr int RW = kTopTile / kCoarseWarps;  // rows per warp (8)
  // the warp's 8 rows x 64 columns: 16 independent loads per lane
  double a[RW][2];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    a[q][0] = __ldg(T + (warp * RW + q) * kTopTile + lane);
    a[q][1] = __ldg(T + (warp * RW + q) * kTopTile + lane + 32);
  }
  double fj[MC][2], fi[MC][RW];
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const double* f = D.fT + c * D.ft_ld;
    const int j0 = J * kTopTile + lane, j1 = j0 + 32;
    fj[c][0] = j0 < n ? __ldcg(f + j0) : 0.0;
    fj[c][1] = j1 < n ? __ldcg(f + j1) : 0.0;
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      const int i = I * kTopTile + warp * RW + q;
      fi[c][q] = (I != J && i < n) ? __ldcg(f + i) : 0.0;
    }
  }
  double* P = D.tpart;
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    double* Pc = P + c * D.tpart_ld;
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      const double r = warp_sum(fma(a[q][1], fj[c][1], a[q][0] * fj[c][0]));
      if (lane == 0) Pc[((long long)I * nt + J) * kTopTile + warp * RW + q] = r;
    }
    if (I != J) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < RW; ++q) {
        s0 = fma(a[q][0], fi[c][q], s0);
        s1 = fma(a[q][1], fi[c][q], s1);
      }
      colp[warp][c][lane] = s0;
      colp[warp][c][lane + 32] = s1;
    }
  }
  if (I == J) return;
  __syncthreads();
  if (threadIdx.x < kTopTile) {
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < kCoarseWarps; ++w) v += colp[w][c][threadIdx.x];
      P[c * D.tpart_ld + ((long long)J * nt + I) * kTopTile + threadIdx.x] = v;
    }
  }
}

// x_I[r] = sum_J P[I][J][r]: 4 threads per row, each a contiguous J quarter
// (its loads all in flight), combined in a fixed shuffle order.
template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_top_reduce(CoarseNDDev D, ColSet C) {
  pdl_entry();
  if (all_stopped<MC>(C)) return;
  const int nt = D.top_tiles;
  const int I = blockIdx.x;
  const int r = threadIdx.x >> 2, part = threadIdx.x & 3;
  const int per = (nt + 3) / 4, j0 = part * per, j1 = min(nt, j0 + per);
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const double* Pc = D.tpart + c * D.tpart_ld + (long long)I * nt * kTopTile + r;
    double s = 0.0;
    for (int j = j0; j < j1; ++j) s += __ldcg(Pc + (long long)j * kTopTile);
    s += __shfl_down_sync(0xffffffffu, s, 1);
    s += __shfl_down_sync(0xffffffffu, s, 2);
    const int i = I * kTopTile + r;
    if (part == 0 && i < D.n_top) C.x[c * C.ldx + D.top_off + i] = s;
  }
}

// ---- persistent dataflow schedule -------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// item record (12 ints): type, wpr, node, r0, r1, wait_idx, wait_need,
// done_idx, done_need, rel_begin, rel_end, 0
template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_flow(CoarseNDDev D, ColSet C) {
  pdl_entry();
  extern __shared__ double sm[];
  __shared__ double red[MC * kRedStride];
  __shared__ int s_item;
  if (all_stopped<MC>(C)) return;
  const unsigned long long E = __ldcg(D.ctl + 2) + 1;  // this solve's epoch (1-based)
  unsigned long long* cnt = D.cnt;
  while (true) {
    if (threadIdx.x == 0) s_item = (int)atomicAdd(D.ctl, 1ull);
    __syncthreads();
    const int k = s_item;
    if (k >= D.n_items) break;
    const int* it = D.items + 12 * k;
    const int type = it[0], wpr = it[1], node = it[2], r0 = it[3], r1 = it[4];
    if (threadIdx.x == 0) {
      const int wi = it[5];
      if (wi >= 0) {
        const unsigned long long target = E * (unsigned long long)it[6];
        unsigned int spins = 0;
        while (ld_acquire(cnt + wi) < target) {
          __nanosleep(64);
          if (++spins == (1u << 26)) {  // several seconds: a broken schedule must fail, not hang
            printf("k_coarse_flow: item %d stuck on counter %d (%llu < %llu)\n", k, wi, ld_acquire(cnt + wi),
                   target);
            __trap();
          }
        }
      }
    }
    __syncthreads();
    switch (type) {
      case kFwd: item_fwd<MC>(D, false, wpr, node_info(D.meta + 8 * node), r0, r1, C, sm, red); break;
      case kAsm: item_asm<MC>(D, node_info(D.meta + 8 * node), C); break;
      case kRows: item_fwd<MC>(D, true, wpr, node_info(D.meta + 8 * node), r0, r1, C, sm, red); break;
      case kTopGather: item_top_gather<MC>(D, r0, r1, C); break;
      case kTopRows: item_top_rows<MC>(D, wpr, r0, r1, C, sm, red, true); break;
      default: item_bwd<MC>(D, wpr, node_info(D.meta + 8 * node), r0, r1, C, sm, red); break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned long long old = atomicAdd(cnt + it[7], 1ull);
      if (old + 1 == E * (unsigned long long)it[8]) {
        __threadfence();
        for (int j = it[9]; j < it[10]; ++j) atomicAdd(cnt + __ldg(D.rel + j), 1ull);
      }
    }
  }
  // last CTA out rewinds the item counter and advances the epoch
  if (threadIdx.x == 0) {
    const unsigned long long old = atomicAdd(D.ctl + 1, 1ull);
    if (old == gridDim.x - 1) {
      D.ctl[0] = 0ull;
      D.ctl[1] = 0ull;
      D.ctl[2] = E;
      __threadfence();
    }
  }
}

// ---- per-level schedule (fallback) -----------------------------------------
template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_fwd(CoarseNDDev D, int wpr, int assembled,
                                                               const long long* recs, ColSet C) {
  pdl_entry();
  extern __shared__ double sm[];
  __shared__ double red[MC * kRedStride];
  if (all_stopped<MC>(C)) return;
  int r0, r1;
  const NodeInfo n = item_record(recs + 10LL * blockIdx.x, r0, r1);
  item_fwd<MC>(D, assembled != 0, wpr, n, r0, r1, C, sm, red);
}

template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_asm(CoarseNDDev D, const int* nodes, ColSet C) {
  pdl_entry();
  if (all_stopped<MC>(C)) return;
  item_asm<MC>(D, node_info(D.meta + 8 * nodes[blockIdx.x]), C);
}

template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_bwd(CoarseNDDev D, int wpr, const long long* recs,
                                                               ColSet C) {
  pdl_entry();
  extern __shared__ double sm[];
  __shared__ double red[MC * kRedStride];
  if (all_stopped<MC>(C)) return;
  int r0, r1;
  const NodeInfo n = item_record(recs + 10LL * blockIdx.x, r0, r1);
  item_bwd<MC>(D, wpr, n, r0, r1, C, sm, red);
}

template <int MC>
__global__ void k_coarse_top_gather(CoarseNDDev D, ColSet C) {
  pdl_entry();
  if (all_stopped<MC>(C)) return;
  item_top_gather<MC>(D, blockIdx.x * blockDim.x, D.n_top, C);
}

template <int MC>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_top_rows(CoarseNDDev D, ColSet C) {
  pdl_entry();
  extern __shared__ double sm[];
  __shared__ double red[MC * kRedStride];
  if (all_stopped<MC>(C)) return;
  const int rpc = mode_rows(D.top_wpr);
  const int r0 = blockIdx.x * rpc;
  item_top_rows<MC>(D, D.top_wpr, r0, min(D.n_top, r0 + rpc), C, sm, red, D.top_smem != 0);
}

template <typename K>
static void allow_smem(K kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

static int max_optin_smem() {
  static int v = 0;
  if (v == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (v <= 0) v = 227 * 1024;
  }
  return v;
}

// per-column shared footprint of the row items (front / separator / top vectors)
static int col_smem(const CoarseNDDev& D) {
  const int smem_bwd = (int)(sizeof(double) * (size_t)D.max_front);
  const int smem_top = (int)(sizeof(double) * (size_t)(D.n_top + 1));
  return std::max(smem_bwd, smem_top);
}

template <int MC>
static cudaError_t launch_coarse_cols(const CoarseNDDev& D, const ColSet& C, cudaStream_t s) {
  static int attr_max = 0;
  const int smem_fwd = MC * (int)(sizeof(double) * (size_t)D.max_sep);
  const int smem_bwd = MC * (int)(sizeof(double) * (size_t)D.max_front);
  const int smem_top = MC * (int)(sizeof(double) * (size_t)(D.n_top + 1));
  const int smem_max = MC * col_smem(D);
  if (smem_max > attr_max) {
    allow_smem(k_coarse_flow<MC>, smem_max);
    allow_smem(k_coarse_fwd<MC>, smem_max);
    allow_smem(k_coarse_bwd<MC>, smem_max);
    allow_smem(k_coarse_top_rows<MC>, smem_max);
    attr_max = smem_max;
  }
  if (D.items != nullptr && D.n_items > 0) {
    static int cached_smem = -1, cached_ctas = 0;
    if (cached_smem != smem_max) {
      int dev = 0, nsm = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_flow<MC>, kCoarseThreads, smem_max);
      cached_ctas = nsm * std::max(1, per_sm);
      cached_smem = smem_max;
    }
    const int ctas = std::min(cached_ctas, D.n_items);
    launch_k(k_coarse_flow<MC>, (unsigned)ctas, kCoarseThreads, smem_max, s, D, C);
    return cudaGetLastError();
  }
  for (int h = 0; h < D.n_levels; ++h) {
    const long long a = D.fwd_ptr[h], b = D.fwd_ptr[h + 1];
    if (b <= a) continue;
    const int split = D.split[h] != 0;
    if (split) {
      const long long na = D.asm_ptr[h], nb = D.asm_ptr[h + 1];
      launch_k(k_coarse_asm<MC>, (unsigned)(nb - na), kCoarseThreads, 0, s, D, D.asm_nodes + na, C);
    }
    launch_k(k_coarse_fwd<MC>, (unsigned)(b - a), kCoarseThreads, smem_fwd, s, D, D.fwd_wpr[h], split,
                                                                         D.fwd_items + 10 * a, C);
  }
  if (D.n_top > 0 && D.top_tiles > 0) {
    launch_k(k_coarse_top_gather<MC>, (unsigned)((D.n_top + 255) / 256), 256, 0, s, D, C);
    const long long ntiles = (long long)D.top_tiles * (D.top_tiles + 1) / 2;
    launch_k(k_top_tiles<MC>, (unsigned)ntiles, kCoarseThreads, 0, s, D, C);
    launch_k(k_top_reduce<MC>, (unsigned)D.top_tiles, kCoarseThreads, 0, s, D, C);
  } else if (D.n_top > 0) {
    launch_k(k_coarse_top_gather<MC>, (unsigned)((D.n_top + 255) / 256), 256, 0, s, D, C);
    const int rpc = kCoarseWarps * std::max(1, D.top_wpr >> 4) / (D.top_wpr & 15);
    launch_k(k_coarse_top_rows<MC>, (unsigned)((D.n_top + rpc - 1) / rpc), kCoarseThreads, D.top_smem ? smem_top : 0, s,
        D, C);
  }
  for (int h = 0; h < D.n_levels; ++h) {  // bwd groups: top-most bottom level first
    const long long a = D.bwd_ptr[h], b = D.bwd_ptr[h + 1];
    if (b > a)
      launch_k(k_coarse_bwd<MC>, (unsigned)(b - a), kCoarseThreads, smem_bwd, s, D, D.bwd_wpr[h], D.bwd_items + 10 * a, C);
  }
  return cudaGetLastError();
}

int coarse_nd_max_cols(const CoarseNDDev& D) {
  const int per = std::max(col_smem(D), 8);
  return std::max(1, std::min({kCoarseMaxCols, D.max_cols > 0 ? D.max_cols : 1, max_optin_smem() / per}));
}

cudaError_t launch_coarse_nd_multi(const CoarseNDDev& D, int ncols, const double* y, long long ldy, double* x,
                                   long long ldx, const int* stop, long long stop_ld, cudaStream_t s) {
  const int mc = coarse_nd_max_cols(D);
  // column groups of <= mc run one after another in stream order and share
  // the per-column scratch (fS / cU / fT columns 0 .. mc-1)
  for (int c0 = 0; c0 < ncols; c0 += mc) {
    const int k = std::min(mc, ncols - c0);
    ColSet C{y + c0 * ldy, ldy, x + c0 * ldx, ldx, stop ? stop + c0 * stop_ld : nullptr, stop_ld};
    cudaError_t e;
    switch (k) {
      case 1: e = launch_coarse_cols<1>(D, C, s); break;
      case 2: e = launch_coarse_cols<2>(D, C, s); break;
      case 3: e = launch_coarse_cols<3>(D, C, s); break;
      default: e = launch_coarse_cols<4>(D, C, s); break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s) {
  return launch_coarse_nd_multi(D, 1, y, 0, x, 0, stop, 0, s);
}

}  // namespace tvb
