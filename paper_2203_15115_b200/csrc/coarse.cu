// a7: per-iteration coarse solve E mu = y with the nested-dissection factor
// built by paper_2203_15115_b200/coarse.py. Replaces the dense
// scipy.linalg.cho_solve of DeflationSpace.coarse_solve (topovox/fea.py:208-211).
// Vectors are in ND order (every separator a contiguous DOF range).
//
// Bottom tree node N (separator S, update set U, front F = S u U):
//   forward  (heights 0..H0-1): f_S = y_S + sum_children c_child|S,
//                               f_U =       sum_children c_child|U,
//                               c_U = f_U - G f_S            (G = F_US F_SS^-1)
//   backward (heights H0-1..0): x_S = Z f_S - G^T x_U         (Z = F_SS^-1)
// Top set T (heights >= H0): x_T = S_T^-1 (y_T + sum_children c_child|T).
// One launch per bottom height and direction (two for forward heights with
// large fronts: a per-node assembly pass, then the rows) and two for the top;
// work items are (node, 8-row chunk) pairs, one CTA each, one warp per matrix
// row with a fixed-order lane-strided dot product + shuffle tree. Children are
// extend-added in a fixed order: the solve is bitwise reproducible.
#include "coarse.cuh"

namespace tvb {

constexpr int kCoarseThreads = 256;

// Row . vector with the row streamed from global memory: 8 independent loads
// in flight per lane. Fixed summation order.
__device__ __forceinline__ double warp_dot(const double* __restrict__ a, const double* b, int n, int lane) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = lane;
  for (; i + 7 * 32 < n; i += 8 * 32) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(a + i + 32 * k);
    s0 = fma(v[0], b[i], s0);
    s1 = fma(v[1], b[i + 32], s1);
    s2 = fma(v[2], b[i + 64], s2);
    s3 = fma(v[3], b[i + 96], s3);
    s0 = fma(v[4], b[i + 128], s0);
    s1 = fma(v[5], b[i + 160], s1);
    s2 = fma(v[6], b[i + 192], s2);
    s3 = fma(v[7], b[i + 224], s3);
  }
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = (i + 32 * k < n) ? __ldg(a + i + 32 * k) : 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (i + 32 * k < n) s0 = fma(v[k], b[i + 32 * k], s0);
  return warp_sum((s0 + s1) + (s2 + s3));
}

// extend-add the children's update vectors into a front vector f (fixed order)
__device__ __forceinline__ void add_children(const CoarseNDDev& D, int cb, int ce, double* f) {
  for (int k = cb; k < ce; ++k) {
    __syncthreads();
    const int cn = (int)D.children[2 * k];
    const long long co = D.children[2 * k + 1];
    const long long* cm = D.meta + 8 * cn;
    const int cu = (int)cm[1];
    const double* cc = D.cU + cm[5];
    for (int t = threadIdx.x; t < cu; t += blockDim.x) f[D.cmap[co + t]] += cc[t];
  }
  __syncthreads();
}

// Fused forward item (small fronts): assemble the front vector in shared
// memory, then c_U = f_U - G f_S for this item's rows.
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_fwd(CoarseNDDev D, const int* items, const double* y,
                                                               const int* stop) {
  extern __shared__ double f[];
  if (stop != nullptr && *stop) return;
  const int* it = items + 3 * blockIdx.x;
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long g_off = m[2], sd_off = m[4], ud_off = m[5];
  for (int i = threadIdx.x; i < s + u; i += blockDim.x) f[i] = i < s ? y[sd_off + i] : 0.0;
  add_children(D, (int)m[6], (int)m[7], f);
  if (r0 == 0)
    for (int i = threadIdx.x; i < s; i += blockDim.x) D.fS[sd_off + i] = f[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = r0 + warp; j < r1; j += nw) {
    const double d = warp_dot(D.G + g_off + (long long)j * s, f, s, lane);
    if (lane == 0) D.cU[ud_off + j] = f[s + j] - d;
  }
}

// Split forward (large fronts), part 1: assemble f_S into fS and f_U into cU,
// once per node.
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_asm(CoarseNDDev D, const int* nodes, const double* y,
                                                               const int* stop) {
  if (stop != nullptr && *stop) return;
  const int node = nodes[blockIdx.x];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long sd_off = m[4], ud_off = m[5];
  double* fS = D.fS + sd_off;
  double* fU = D.cU + ud_off;
  for (int i = threadIdx.x; i < s + u; i += blockDim.x) {
    if (i < s) fS[i] = y[sd_off + i];
    else fU[i - s] = 0.0;
  }
  for (int k = (int)m[6]; k < (int)m[7]; ++k) {
    __syncthreads();
    const int cn = (int)D.children[2 * k];
    const long long co = D.children[2 * k + 1];
    const long long* cm = D.meta + 8 * cn;
    const int cu = (int)cm[1];
    const double* cc = D.cU + cm[5];
    for (int t = threadIdx.x; t < cu; t += blockDim.x) {
      const int pos = D.cmap[co + t];
      if (pos < s) fS[pos] += cc[t];
      else fU[pos - s] += cc[t];
    }
  }
}

// Split forward, part 2: c_U[j] = f_U[j] - G[j,:] f_S in place (one warp per row).
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_rows(CoarseNDDev D, const int* items, const int* stop) {
  extern __shared__ double fs[];
  if (stop != nullptr && *stop) return;
  const int* it = items + 3 * blockIdx.x;
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0];
  const long long g_off = m[2], sd_off = m[4], ud_off = m[5];
  for (int i = threadIdx.x; i < s; i += blockDim.x) fs[i] = D.fS[sd_off + i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = r0 + warp; j < r1; j += nw) {
    const double d = warp_dot(D.G + g_off + (long long)j * s, fs, s, lane);
    if (lane == 0) D.cU[ud_off + j] -= d;
  }
}

// Top set, part 1: fT = y_T + children's update vectors (one CTA, fixed order).
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_top_asm(CoarseNDDev D, const double* y, const int* stop) {
  if (stop != nullptr && *stop) return;
  for (int i = threadIdx.x; i < D.n_top; i += blockDim.x) D.fT[i] = y[D.top_off + i];
  for (int k = 0; k < D.n_tchildren; ++k) {
    __syncthreads();
    const int cn = (int)D.tchildren[2 * k];
    const long long to = D.tchildren[2 * k + 1];
    const long long* cm = D.meta + 8 * cn;
    const int cu = (int)cm[1];
    const double* cc = D.cU + cm[5];
    for (int t = threadIdx.x; t < cu; t += blockDim.x) D.fT[D.tmap[to + t]] += cc[t];
  }
}

// Top set, part 2: x_T = S_T^-1 fT (dense, one warp per row, 8 rows per CTA).
__global__ void __launch_bounds__(kCoarseThreads) k_coarse_top_rows(CoarseNDDev D, double* x, const int* stop) {
  extern __shared__ double ft[];
  if (stop != nullptr && *stop) return;
  const int n = D.n_top;
  for (int i = threadIdx.x; i < n; i += blockDim.x) ft[i] = D.fT[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * (kCoarseThreads / 32) + warp;
  if (j < n) {
    const double d = warp_dot(D.ZT + (long long)j * n, ft, n, lane);
    if (lane == 0) x[D.top_off + j] = d;
  }
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse_bwd(CoarseNDDev D, const int* items, double* x,
                                                               const int* stop) {
  extern __shared__ double sm[];
  if (stop != nullptr && *stop) return;
  const int* it = items + 3 * blockIdx.x;
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long g_off = m[2], z_off = m[3], sd_off = m[4], ud_off = m[5];
  double* fs = sm;
  double* xu = sm + s;
  for (int i = threadIdx.x; i < s; i += blockDim.x) fs[i] = D.fS[sd_off + i];
  for (int k = threadIdx.x; k < u; k += blockDim.x) xu[k] = x[D.udof[ud_off + k]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = r0 + warp; j < r1; j += nw) {
    const double a = warp_dot(D.Z + z_off + (long long)j * s, fs, s, lane);
    const double b = u ? warp_dot(D.Gt + g_off + (long long)j * u, xu, u, lane) : 0.0;
    if (lane == 0) x[sd_off + j] = a - b;
  }
}

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s) {
  static int attr_max = 0;
  const int smem = (int)(sizeof(double) * (size_t)D.max_front);
  const int smem_top = (int)(sizeof(double) * (size_t)(D.n_top + 1));
  const int smem_max = smem > smem_top ? smem : smem_top;
  if (smem_max > attr_max) {
    cudaFuncSetAttribute(k_coarse_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    cudaFuncSetAttribute(k_coarse_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    cudaFuncSetAttribute(k_coarse_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    cudaFuncSetAttribute(k_coarse_top_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
    attr_max = smem_max;
  }
  for (int h = 0; h < D.n_levels; ++h) {
    const long long a = D.fwd_ptr[h], b = D.fwd_ptr[h + 1];
    if (b <= a) continue;
    if (D.split[h]) {
      const long long na = D.asm_ptr[h], nb = D.asm_ptr[h + 1];
      k_coarse_asm<<<(unsigned)(nb - na), kCoarseThreads, 0, s>>>(D, D.asm_nodes + na, y, stop);
      k_coarse_rows<<<(unsigned)(b - a), kCoarseThreads, (int)(sizeof(double) * D.max_sep), s>>>(
          D, D.fwd_items + 3 * a, stop);
    } else {
      k_coarse_fwd<<<(unsigned)(b - a), kCoarseThreads, smem, s>>>(D, D.fwd_items + 3 * a, y, stop);
    }
  }
  if (D.n_top > 0) {
    k_coarse_top_asm<<<1, kCoarseThreads, 0, s>>>(D, y, stop);
    const int rows_per_cta = kCoarseThreads / 32;
    k_coarse_top_rows<<<(unsigned)((D.n_top + rows_per_cta - 1) / rows_per_cta), kCoarseThreads, smem_top, s>>>(
        D, x, stop);
  }
  for (int h = 0; h < D.n_levels; ++h) {  // bwd_ptr groups are ordered top-most bottom level first
    const long long a = D.bwd_ptr[h], b = D.bwd_ptr[h + 1];
    if (b > a) k_coarse_bwd<<<(unsigned)(b - a), kCoarseThreads, smem, s>>>(D, D.bwd_items + 3 * a, x, stop);
  }
  return cudaGetLastError();
}

}  // namespace tvb
