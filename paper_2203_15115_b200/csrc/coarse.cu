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
// level), so the kernels are built for short dependency chains:
//   * front vectors are GATHERED: each front position lists the update-vector
//     entries of (at most two) children, so assembly has no barriers, atomics
//     or serial child loops (the fixed child order keeps it deterministic);
//   * one launch per bottom height and direction (plus a per-node assembly
//     launch for heights with fronts > TVB_ND_SPLIT_FRONT) and two for the top;
//   * work items are (node, row chunk) pairs, one 256-thread CTA each; long
//     rows are split across WPR = 1/2/4/8 warps (8/WPR rows per CTA), every
//     warp a fixed-order lane-strided dot product + shuffle tree, the WPR
//     parts summed in order through shared memory.
// Bitwise reproducible run to run.
#include <algorithm>

#include "coarse.cuh"

namespace tvb {

constexpr int kCoarseThreads = 256;
constexpr int kCoarseWarps = kCoarseThreads / 32;

// Part `part` of row . vector (lane-strided over WPR warps), row streamed from
// global memory with 8 independent loads in flight per lane.
template <int WPR>
__device__ __forceinline__ double part_dot(const double* __restrict__ a, const double* b, int n, int part, int lane) {
  constexpr int st = 32 * WPR;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = part * 32 + lane;
  for (; i + 7 * st < n; i += 8 * st) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(a + i + st * k);
    s0 = fma(v[0], b[i], s0);
    s1 = fma(v[1], b[i + st], s1);
    s2 = fma(v[2], b[i + 2 * st], s2);
    s3 = fma(v[3], b[i + 3 * st], s3);
    s0 = fma(v[4], b[i + 4 * st], s0);
    s1 = fma(v[5], b[i + 5 * st], s1);
    s2 = fma(v[6], b[i + 6 * st], s2);
    s3 = fma(v[7], b[i + 7 * st], s3);
  }
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = (i + st * k < n) ? __ldg(a + i + st * k) : 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (i + st * k < n) s0 = fma(v[k], b[i + st * k], s0);
  return warp_sum((s0 + s1) + (s2 + s3));
}

// Rows r0 .. r0+8/WPR-1 (< r1) of M (row length n) dotted with the shared
// vector v. Returns the full dot to threads t < 8/WPR (row r0 + t).
template <int WPR>
__device__ __forceinline__ double rows_dot(const double* __restrict__ M, long long n, const double* v, int r0, int r1,
                                           double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = r0 + warp / WPR;
  const double p = (j < r1) ? part_dot<WPR>(M + (long long)j * n, v, (int)n, warp % WPR, lane) : 0.0;
  if (lane == 0) red[warp] = p;
  __syncthreads();
  double d = 0.0;
  if (threadIdx.x < kCoarseWarps / WPR) {
#pragma unroll
    for (int k = 0; k < WPR; ++k) d += red[threadIdx.x * WPR + k];
  }
  return d;
}

// front position p of a node: base + child-0 entry + child-1 entry (fixed order)
__device__ __forceinline__ double gather_front(const CoarseNDDev& D, long long gm, int p, double base) {
  const int g0 = __ldg(D.gmap + gm + 2 * p), g1 = __ldg(D.gmap + gm + 2 * p + 1);
  if (g0 >= 0) base += D.cU[g0];
  if (g1 >= 0) base += D.cU[g1];
  return base;
}

// Forward rows: c_U[j] = f_U[j] - G[j,:] f_S. ASSEMBLED: f_S / f_U were
// written by k_coarse_asm (large fronts); else gathered here (and the node's
// first item stores f_S for the backward pass).
template <int WPR, bool ASSEMBLED>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_fwd(CoarseNDDev D, const int* items, const double* y,
                                                               const int* stop) {
  extern __shared__ double fs[];
  __shared__ double red[kCoarseWarps];
  if (stop != nullptr && *stop) return;
  const int* it = items + 3 * blockIdx.x;
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0];
  const long long g_off = m[2], sd_off = m[4], ud_off = m[5], gm = m[6];
  for (int i = threadIdx.x; i < s; i += blockDim.x) {
    if (ASSEMBLED) {
      fs[i] = D.fS[sd_off + i];
    } else {
      const double v = gather_front(D, gm, i, y[sd_off + i]);
      fs[i] = v;
      if (r0 == 0) D.fS[sd_off + i] = v;
    }
  }
  __syncthreads();
  const double d = rows_dot<WPR>(D.G + g_off, s, fs, r0, r1, red);
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < kCoarseWarps / WPR && j < r1) {
    const double fu = ASSEMBLED ? D.cU[ud_off + j] : gather_front(D, gm, s + j, 0.0);
    D.cU[ud_off + j] = fu - d;
  }
}

// Large fronts, assembly pass: f_S -> fS, f_U -> cU (one CTA per node).
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_asm(CoarseNDDev D, const int* nodes, const double* y,
                                                               const int* stop) {
  if (stop != nullptr && *stop) return;
  const int node = nodes[blockIdx.x];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long sd_off = m[4], ud_off = m[5], gm = m[6];
  for (int p = threadIdx.x; p < s + u; p += blockDim.x) {
    if (p < s) D.fS[sd_off + p] = gather_front(D, gm, p, y[sd_off + p]);
    else D.cU[ud_off + p - s] = gather_front(D, gm, p, 0.0);
  }
}

// Backward rows: x_S[j] = [Z | -G^T][j,:] . [f_S ; x_U].
template <int WPR>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_bwd(CoarseNDDev D, const int* items, double* x,
                                                               const int* stop) {
  extern __shared__ double v[];
  __shared__ double red[kCoarseWarps];
  if (stop != nullptr && *stop) return;
  const int* it = items + 3 * blockIdx.x;
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long b_off = m[3], sd_off = m[4], ud_off = m[5];
  for (int i = threadIdx.x; i < s + u; i += blockDim.x)
    v[i] = i < s ? D.fS[sd_off + i] : x[__ldg(D.udof + ud_off + i - s)];
  __syncthreads();
  const double d = rows_dot<WPR>(D.B + b_off, s + u, v, r0, r1, red);
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < kCoarseWarps / WPR && j < r1) x[sd_off + j] = d;
}

// Top set, part 1: fT = y_T + children's update entries (CSR, fixed order).
__global__ void k_coarse_top_gather(CoarseNDDev D, const double* y, const int* stop) {
  if (stop != nullptr && *stop) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n_top) return;
  double v = y[D.top_off + i];
  const int a = __ldg(D.tptr + i), b = __ldg(D.tptr + i + 1);
  for (int k = a; k < b; ++k) v += D.cU[__ldg(D.tidx + k)];
  D.fT[i] = v;
}

// Top set, part 2: x_T = S_T^-1 fT (dense rows).
template <int WPR>
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_top_rows(CoarseNDDev D, double* x, const int* stop) {
  extern __shared__ double ft[];
  __shared__ double red[kCoarseWarps];
  if (stop != nullptr && *stop) return;
  const int n = D.n_top;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ft[i] = D.fT[i];
  __syncthreads();
  const int r0 = blockIdx.x * (kCoarseWarps / WPR);
  const int r1 = min(n, r0 + kCoarseWarps / WPR);
  const double d = rows_dot<WPR>(D.ZT, n, ft, r0, r1, red);
  const int j = r0 + threadIdx.x;
  if (threadIdx.x < kCoarseWarps / WPR && j < r1) x[D.top_off + j] = d;
}

template <typename K>
static void allow_smem(K kernel, int bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int WPR>
static void set_smem_all(int bytes) {
  allow_smem(k_coarse_fwd<WPR, false>, bytes);
  allow_smem(k_coarse_fwd<WPR, true>, bytes);
  allow_smem(k_coarse_bwd<WPR>, bytes);
  allow_smem(k_coarse_top_rows<WPR>, bytes);
}

template <int WPR>
static void launch_fwd(bool assembled, unsigned n, int smem, const CoarseNDDev& D, const int* items, const double* y,
                       const int* stop, cudaStream_t s) {
  if (assembled) k_coarse_fwd<WPR, true><<<n, kCoarseThreads, smem, s>>>(D, items, y, stop);
  else k_coarse_fwd<WPR, false><<<n, kCoarseThreads, smem, s>>>(D, items, y, stop);
}

#define TVB_WPR_DISPATCH(w, CALL) \
  switch (w) {                    \
    case 1: CALL(1); break;       \
    case 2: CALL(2); break;       \
    case 4: CALL(4); break;       \
    default: CALL(8); break;      \
  }

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s) {
  static int attr_max = 0;
  const int smem_bwd = (int)(sizeof(double) * (size_t)D.max_front);
  const int smem_fwd = (int)(sizeof(double) * (size_t)D.max_sep);
  const int smem_top = (int)(sizeof(double) * (size_t)(D.n_top + 1));
  const int smem_max = std::max(smem_bwd, smem_top);
  if (smem_max > attr_max) {
    set_smem_all<1>(smem_max);
    set_smem_all<2>(smem_max);
    set_smem_all<4>(smem_max);
    set_smem_all<8>(smem_max);
    attr_max = smem_max;
  }
  for (int h = 0; h < D.n_levels; ++h) {
    const long long a = D.fwd_ptr[h], b = D.fwd_ptr[h + 1];
    if (b <= a) continue;
    const bool split = D.split[h] != 0;
    if (split) {
      const long long na = D.asm_ptr[h], nb = D.asm_ptr[h + 1];
      k_coarse_asm<<<(unsigned)(nb - na), kCoarseThreads, 0, s>>>(D, D.asm_nodes + na, y, stop);
    }
#define TVB_FWD(W) launch_fwd<W>(split, (unsigned)(b - a), smem_fwd, D, D.fwd_items + 3 * a, y, stop, s)
    TVB_WPR_DISPATCH(D.fwd_wpr[h], TVB_FWD)
#undef TVB_FWD
  }
  if (D.n_top > 0) {
    k_coarse_top_gather<<<(unsigned)((D.n_top + 255) / 256), 256, 0, s>>>(D, y, stop);
#define TVB_TOP(W)                                                                                           \
  k_coarse_top_rows<W><<<(unsigned)((D.n_top + kCoarseWarps / W - 1) / (kCoarseWarps / W)), kCoarseThreads, \
                         smem_top, s>>>(D, x, stop)
    TVB_WPR_DISPATCH(D.top_wpr, TVB_TOP)
#undef TVB_TOP
  }
  for (int h = 0; h < D.n_levels; ++h) {  // bwd groups: top-most bottom level first
    const long long a = D.bwd_ptr[h], b = D.bwd_ptr[h + 1];
    if (b <= a) continue;
#define TVB_BWD(W) \
  k_coarse_bwd<W><<<(unsigned)(b - a), kCoarseThreads, smem_bwd, s>>>(D, D.bwd_items + 3 * a, x, stop)
    TVB_WPR_DISPATCH(D.bwd_wpr[h], TVB_BWD)
#undef TVB_BWD
  }
  return cudaGetLastError();
}

}  // namespace tvb
