// a7: per-iteration coarse solve E mu = y with the nested-dissection block
// LDL^T factor built by paper_2203_15115_b200/coarse.py. Replaces the dense
// scipy.linalg.cho_solve of DeflationSpace.coarse_solve (topovox/fea.py:208-211).
//
// For every tree node N (separator S, update set U, front F = S u U):
//   forward  (leaves -> root): f_S = y_S + sum_children c_child|S,
//                              f_U =       sum_children c_child|U,
//                              c_U = f_U - G f_S                (G = F_US F_SS^-1)
//   backward (root -> leaves): x_S = Z f_S - G^T x_U            (Z = F_SS^-1)
// One launch per tree height and direction; inside a launch, work items are
// (node, 32-row chunk) pairs, one CTA each, one warp per matrix row with a
// fixed-order lane-strided dot product + shuffle tree (deterministic).
// Children are extend-added in a fixed order, so the solve is bitwise
// reproducible. Row-major G (forward) and G^T / Z (backward) make every
// warp read contiguous rows.
#include "coarse.cuh"

namespace tvb {

constexpr int kCoarseThreads = 256;

// Row . vector with the row streamed from global memory: 8 independent loads
// in flight per lane (the row is not L1-resident; a dependent load chain
// would cost a full memory latency per 32 elements). Fixed summation order.
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

// Four rows . one vector per warp: 4 x 4 independent loads in flight per lane.
__device__ __forceinline__ void warp_dot4(const double* __restrict__ a0, long long stride, const double* b, int n,
                                          int lane, int nrows, double (&out)[4]) {
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  const double* a[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) a[r] = a0 + (r < nrows ? r : 0) * stride;
  int i = lane;
  for (; i + 3 * 32 < n; i += 4 * 32) {
    double v[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 4; ++k) v[r][k] = __ldg(a[r] + i + 32 * k);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double bk = b[i + 32 * k];
#pragma unroll
      for (int r = 0; r < 4; ++r) s[r] = fma(v[r][k], bk, s[r]);
    }
  }
  for (; i < n; i += 32) {
    const double bk = b[i];
#pragma unroll
    for (int r = 0; r < 4; ++r) s[r] = fma(__ldg(a[r] + i), bk, s[r]);
  }
  // warp_sum leaves the total in lane 0; broadcast so lane r can store row r
#pragma unroll
  for (int r = 0; r < 4; ++r) out[r] = __shfl_sync(0xffffffffu, warp_sum(s[r]), 0);
}

__device__ __forceinline__ void fwd_item(const CoarseNDDev& D, const int* it, const double* y, double* f) {
  const int node = it[0], r0 = it[1], r1 = it[2];
  const long long* m = D.meta + 8 * node;
  const int s = (int)m[0], u = (int)m[1];
  const long long g_off = m[2], sd_off = m[4], ud_off = m[5];
  const int cb = (int)m[6], ce = (int)m[7];
  for (int i = threadIdx.x; i < s + u; i += blockDim.x) f[i] = i < s ? y[D.sdof[sd_off + i]] : 0.0;
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
  if (r0 == 0)
    for (int i = threadIdx.x; i < s; i += blockDim.x) D.fS[sd_off + i] = f[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = r0 + 4 * warp; j < r1; j += 4 * nw) {
    const int nr = min(4, r1 - j);
    double d[4];
    warp_dot4(D.G + g_off + (long long)j * s, s, f, s, lane, nr, d);
    if (lane < nr) {
      const double dv = lane == 0 ? d[0] : lane == 1 ? d[1] : lane == 2 ? d[2] : d[3];
      D.cU[ud_off + j + lane] = f[s + j + lane] - dv;
    }
  }
}

__device__ __forceinline__ void bwd_item(const CoarseNDDev& D, const int* it, double* x, double* sm) {
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
  for (int j = r0 + 4 * warp; j < r1; j += 4 * nw) {
    const int nr = min(4, r1 - j);
    double a[4], b[4] = {0.0, 0.0, 0.0, 0.0};
    warp_dot4(D.Z + z_off + (long long)j * s, s, fs, s, lane, nr, a);
    if (u) warp_dot4(D.Gt + g_off + (long long)j * u, u, xu, u, lane, nr, b);
    if (lane < nr) {
      const double av = lane == 0 ? a[0] : lane == 1 ? a[1] : lane == 2 ? a[2] : a[3];
      const double bv = lane == 0 ? b[0] : lane == 1 ? b[1] : lane == 2 ? b[2] : b[3];
      x[D.sdof[sd_off + j + lane]] = av - bv;
    }
  }
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse_fwd(CoarseNDDev D, const int* items, const double* y,
                                                               const int* stop) {
  extern __shared__ double sm[];
  if (stop != nullptr && *stop) return;
  fwd_item(D, items + 3 * blockIdx.x, y, sm);
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse_bwd(CoarseNDDev D, const int* items, double* x,
                                                               const int* stop) {
  extern __shared__ double sm[];
  if (stop != nullptr && *stop) return;
  bwd_item(D, items + 3 * blockIdx.x, x, sm);
}

// Persistent variant: one cooperative launch runs every phase (forward
// heights 0..H, then backward heights H..0). Item i of the concatenated list
// is processed by CTA i % gridDim.x, in list order; before an item of phase
// p > 0 the CTA waits until all items of phase p-1 are complete (phase
// counters in global memory, release/acquire). All CTAs are co-resident
// (cooperative launch), so the waits cannot deadlock. The last CTA of the
// last phase resets the counters for the next solve.
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kCoarseThreads) k_coarse_persistent(CoarseNDDev D, CoarsePhases Ph, const double* y,
                                                                      double* x, const int* stop) {
  extern __shared__ double sm[];
  if (stop != nullptr && *stop) return;
  const int nph = Ph.n_phases;
  const unsigned G = gridDim.x;
  for (int phase = 0; phase < nph; ++phase) {
    if (phase > 0) {  // grid barrier: every CTA has finished phase-1
      if (threadIdx.x == 0)
        while (ld_acquire(Ph.done + phase - 1) < G) __nanosleep(32);
      __syncthreads();
    }
    const long long a = Ph.start[phase], b = Ph.start[phase + 1];
    // items of this phase: CTA-strided, starting at a rotated offset so that
    // consecutive phases land on different CTAs
    for (long long i = a + ((blockIdx.x + (unsigned)(a % G)) % G); i < b; i += G) {
      if (phase <= Ph.last_fwd) fwd_item(D, D.fwd_items + 3 * (i - Ph.start[0]), y, sm);
      else bwd_item(D, D.bwd_items + 3 * (i - Ph.start[Ph.last_fwd + 1]), x, sm);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(Ph.done + phase, 1u);
      if (phase == nph - 1 && prev + 1 == G) {
        for (int p = 0; p < nph; ++p) Ph.done[p] = 0u;  // every CTA passed every phase: reset for the next solve
        __threadfence();
      }
    }
  }
}

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s) {
  static int attr_max = 0;
  const int smem = (int)(sizeof(double) * (size_t)D.max_front);
  if (smem > attr_max) {
    cudaFuncSetAttribute(k_coarse_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_coarse_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_coarse_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_max = smem;
  }
  if (D.phases.done != nullptr) {
    // persistent cooperative launch (all CTAs resident)
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coarse_persistent, kCoarseThreads, smem);
    if (per_sm > 4) per_sm = 4;
    if (per_sm >= 1) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(nsm * per_sm));
      cfg.blockDim = dim3(kCoarseThreads);
      cfg.dynamicSmemBytes = (size_t)smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeCooperative;
      attr[0].val.cooperative = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, k_coarse_persistent, D, D.phases, y, x, stop);
    }
  }
  for (int h = 0; h <= D.height; ++h) {
    const long long a = D.fwd_ptr[h], b = D.fwd_ptr[h + 1];
    if (b > a) k_coarse_fwd<<<(unsigned)(b - a), kCoarseThreads, smem, s>>>(D, D.fwd_items + 3 * a, y, stop);
  }
  for (int h = 0; h <= D.height; ++h) {  // bwd_ptr is ordered root level first
    const long long a = D.bwd_ptr[h], b = D.bwd_ptr[h + 1];
    if (b > a) k_coarse_bwd<<<(unsigned)(b - a), kCoarseThreads, smem, s>>>(D, D.bwd_items + 3 * a, x, stop);
  }
  return cudaGetLastError();
}

}  // namespace tvb
