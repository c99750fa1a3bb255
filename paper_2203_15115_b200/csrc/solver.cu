// a8: (deflated) Jacobi-preconditioned CG driver, replacing solve_static
// (topovox/fea.py:218-299). The host loop only launches CUDA graphs that each
// contain `check_every` complete iterations and reads back two ints per
// launch; all scalars (alpha, beta, residual, stop flag) live on the device.
//
// Algorithm (the reference's, step for step; projection = 0):
//   x0 = W E^-1 W^T f ; r = f - A x0 ; r[fixed] = 0 ; stop if |r|/|f_free| <= tol
//   z = D^-1 r ; p = z - W E^-1 (AW)^T z ; rz = r.z
//   loop: q = A p ; alpha = rz/(p.q) ; x += alpha p ; r -= alpha q
//         stop if |r|/|f_free| <= tol ; z = D^-1 r ; beta = r.z_new / rz
//         p = z + beta p - W E^-1 (AW)^T z
// with (AW)^T z evaluated as W^T (A z) (A symmetric, W zero on fixed DOFs).
//
// Stabilised projection (projection = 1, the Python default): the loop projects z + beta p instead of z,
//     p = z + beta p - W E^-1 W^T (A z + beta q),   q = A p_old,
// which equals the reference update in exact arithmetic (W^T A p_old = 0) but
// re-imposes W^T A p = 0 every iteration. The reference recurrence lets that
// component drift: on a Bernoulli(0.9) cantilever the reference itself
// converges with scipy's cho_solve and diverges when only the rounding of the
// coarse solve changes (explicit inverse), see DESIGN.md §4 / tests.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "deflation.cuh"
#include "matvec.cuh"
#include "solver.cuh"
#include "vec.cuh"

namespace tvb {

// mu = Einv * yc with a dense symmetric inverse; one warp per row, fixed order.
// MC right-hand sides share each row load; per column the arithmetic is the
// single-column sequence (bitwise equal results).
template <int MC>
__global__ void k_dense_gemv(long long nc, const double* Einv, const double* yc, long long ldy, double* mu,
                            long long ldm, const int* stop, long long stop_ld) {
  pdl_entry();
  if (stop != nullptr) {
    bool all = true;
#pragma unroll
    for (int c = 0; c < MC; ++c) all = all && stop[c * stop_ld] != 0;
    if (all) return;
  }
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nc) return;
  const double* a = Einv + row * nc;
  double s[MC];
#pragma unroll
  for (int c = 0; c < MC; ++c) s[c] = 0.0;
  for (long long j = lane; j < nc; j += 32) {
    const double aj = a[j];
#pragma unroll
    for (int c = 0; c < MC; ++c) s[c] = fma(aj, yc[c * ldy + j], s[c]);
  }
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const double v = warp_sum(s[c]);
    if (lane == 0) mu[c * ldm + row] = v;
  }
}

cudaError_t launch_dense_gemv_multi(long long nc, const double* Einv, int ncols, const double* yc, long long ldy,
                                    double* mu, long long ldm, const int* stop, long long stop_ld, cudaStream_t s) {
  const long long threads = nc * 32;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  for (int c0 = 0; c0 < ncols; c0 += 4) {
    const int k = ncols - c0 < 4 ? ncols - c0 : 4;
    const double* y = yc + c0 * ldy;
    double* m = mu + c0 * ldm;
    const int* st = stop ? stop + c0 * stop_ld : nullptr;
    switch (k) {
      case 1: launch_k(k_dense_gemv<1>, grid, 256, 0, s, nc, Einv, y, ldy, m, ldm, st, stop_ld); break;
      case 2: launch_k(k_dense_gemv<2>, grid, 256, 0, s, nc, Einv, y, ldy, m, ldm, st, stop_ld); break;
      case 3: launch_k(k_dense_gemv<3>, grid, 256, 0, s, nc, Einv, y, ldy, m, ldm, st, stop_ld); break;
      default: launch_k(k_dense_gemv<4>, grid, 256, 0, s, nc, Einv, y, ldy, m, ldm, st, stop_ld); break;
    }
  }
  return cudaGetLastError();
}

// Dense coarse solve and nu_B = S_B mu_B in one launch (the iteration's dense
// path). One CTA per agglomerate, kNuWpr warps per coarse row: with one warp
// per row a C1-sized system (1500 rows) puts only ~10 warps on an SM and the
// 18 MB inverse streams at L2 latency (ncu 10.7 us); four warps per row, each
// summing a contiguous quarter of the row lane-strided with four loads in
// flight, then combined in segment order, keep ~40 warps per SM busy. The six
// mu values go through shared memory and threads 0..5 (per column) apply S_B
// in k_block_nu's order. Deterministic (fixed orders); per column the
// arithmetic does not depend on MC, so batched and single solves stay bitwise
// equal.
constexpr int kNuWpr = 4;

template <int MC>
__global__ void __launch_bounds__(6 * kNuWpr * 32) k_dense_gemv_nu(long long nb, const double* __restrict__ Einv,
                                                                   const double* __restrict__ S,
                                                                   const double* __restrict__ yc, long long ldy,
                                                                   double* mu, long long ldm, double* nu,
                                                                   long long ldn, const int* stop,
                                                                   long long stop_ld) {
  pdl_entry();
  __shared__ double part[MC][6][kNuWpr];
  __shared__ double mu_s[MC][6];
  if (stop != nullptr) {
    bool all = true;
#pragma unroll
    for (int c = 0; c < MC; ++c) all = all && stop[c * stop_ld] != 0;
    if (all) return;
  }
  const long long B = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = warp / kNuWpr, q = warp % kNuWpr;  // row of the block, segment of the row
  const long long nc = 6 * nb, row = 6 * B + r;
  const long long seg = ((nc + kNuWpr - 1) / kNuWpr + 31) & ~31LL;  // segment length, a multiple of 32
  const long long j0 = q * seg, j1 = min(nc, j0 + seg);
  const double* a = Einv + row * nc;
  double acc[MC];
#pragma unroll
  for (int c = 0; c < MC; ++c) acc[c] = 0.0;
  long long j = j0 + lane;
  for (; j + 96 < j1; j += 128) {  // four independent row loads in flight, accumulated in index order
    const double a0 = a[j], a1 = a[j + 32], a2 = a[j + 64], a3 = a[j + 96];
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      const double* y = yc + c * ldy + j;
      acc[c] = fma(a0, y[0], acc[c]);
      acc[c] = fma(a1, y[32], acc[c]);
      acc[c] = fma(a2, y[64], acc[c]);
      acc[c] = fma(a3, y[96], acc[c]);
    }
  }
  for (; j < j1; j += 32) {
    const double aj = a[j];
#pragma unroll
    for (int c = 0; c < MC; ++c) acc[c] = fma(aj, yc[c * ldy + j], acc[c]);
  }
#pragma unroll
  for (int c = 0; c < MC; ++c) {
    const double v = warp_sum(acc[c]);
    if (lane == 0) part[c][r][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6 * MC) {
    const int c = threadIdx.x / 6, i = threadIdx.x % 6;
    double v = part[c][i][0];
#pragma unroll
    for (int k = 1; k < kNuWpr; ++k) v += part[c][i][k];
    mu[c * ldm + 6 * B + i] = v;
    mu_s[c][i] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6 * MC) {
    const int c = threadIdx.x / 6, i = threadIdx.x % 6;
    double v = 0.0;
    for (int k = 0; k < 6; ++k) v = fma(S[36 * B + i + 6 * k], mu_s[c][k], v);
    nu[c * ldn + 6 * B + i] = v;
  }
}

cudaError_t launch_dense_gemv_nu_multi(long long nb, const double* Einv, const double* S, int ncols, const double* yc,
                                       long long ldy, double* mu, long long ldm, double* nu, long long ldn,
                                       const int* stop, long long stop_ld, cudaStream_t s) {
  for (int c0 = 0; c0 < ncols; c0 += 4) {
    const int k = ncols - c0 < 4 ? ncols - c0 : 4;
    const double* y = yc + c0 * ldy;
    double* m = mu + c0 * ldm;
    double* n = nu + c0 * ldn;
    const int* st = stop ? stop + c0 * stop_ld : nullptr;
    const unsigned grid = (unsigned)nb;
    switch (k) {
      case 1: launch_k(k_dense_gemv_nu<1>, grid, 6 * kNuWpr * 32, 0, s, nb, Einv, S, y, ldy, m, ldm, n, ldn, st, stop_ld); break;
      case 2: launch_k(k_dense_gemv_nu<2>, grid, 6 * kNuWpr * 32, 0, s, nb, Einv, S, y, ldy, m, ldm, n, ldn, st, stop_ld); break;
      case 3: launch_k(k_dense_gemv_nu<3>, grid, 6 * kNuWpr * 32, 0, s, nb, Einv, S, y, ldy, m, ldm, n, ldn, st, stop_ld); break;
      default: launch_k(k_dense_gemv_nu<4>, grid, 6 * kNuWpr * 32, 0, s, nb, Einv, S, y, ldy, m, ldm, n, ldn, st, stop_ld); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_dense_gemv(long long nc, const double* Einv, const double* yc, double* mu, const int* stop,
                              cudaStream_t s) {
  return launch_dense_gemv_multi(nc, Einv, 1, yc, 0, mu, 0, stop, 0, s);
}

// Device-side loop condition of the whole-solve graph: keep iterating while
// any right-hand side of the group is still running (done flags of RHS
// c_lo .. c_lo + n - 1 at stride ld ints).
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* done, long long ld, int n) {
  unsigned go = 0u;
  for (int c = 0; c < n; ++c) go |= (done[c * ld] == 0) ? 1u : 0u;
  cudaGraphSetConditional(h, go);
}

// count the nodes with an operator-fixed axis that the deflation space's flags do not fix
__global__ void k_flags_uncovered(long long nn, const uint8_t* nflags, const uint8_t* dflags, int* count) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n < nn && ((nflags[n] & 7) & ~(dflags[n] & 7))) atomicAdd(count, 1);
}

// ---------------------------------------------------------------------------
struct PcgWork {
  double *r, *z, *p, *q, *t, *inv_d;
  double *yc, *mu, *nu;
  double* partials;
  SolverState* st;
  int* zero_free;
};

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

size_t pcg_ws_bytes(const Grid& g, int block) {
  const size_t nd = 3 * (size_t)g.nn;
  size_t nb = 0;
  if (block > 0) nb = (size_t)make_agglo(g, block, 1.0).nb;
  size_t b = 0;
  b += 6 * align_up(nd * sizeof(double));
  b += 3 * align_up(6 * nb * sizeof(double) + 8);
  b += align_up((size_t)(2 * kMaxReduceCtas + 65536) * sizeof(double));
  b += align_up(sizeof(SolverState));
  b += align_up(sizeof(int));
  return b;
}

static PcgWork carve(void* ws, const Grid& g, int block) {
  const size_t nd = 3 * (size_t)g.nn;
  size_t nb = 0;
  if (block > 0) nb = (size_t)make_agglo(g, block, 1.0).nb;
  char* p = (char*)ws;
  PcgWork w;
  auto take = [&](size_t bytes) {
    char* q = p;
    p += align_up(bytes);
    return (void*)q;
  };
  w.r = (double*)take(nd * sizeof(double));
  w.z = (double*)take(nd * sizeof(double));
  w.p = (double*)take(nd * sizeof(double));
  w.q = (double*)take(nd * sizeof(double));
  w.t = (double*)take(nd * sizeof(double));
  w.inv_d = (double*)take(nd * sizeof(double));
  w.yc = (double*)take(6 * nb * sizeof(double) + 8);
  w.mu = (double*)take(6 * nb * sizeof(double) + 8);
  w.nu = (double*)take(6 * nb * sizeof(double) + 8);
  w.partials = (double*)take((size_t)(2 * kMaxReduceCtas + 65536) * sizeof(double));
  w.st = (SolverState*)take(sizeof(SolverState));
  w.zero_free = (int*)take(sizeof(int));
  return w;
}

#define TVB_CK(expr)                                 \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) {                         \
      set_last_error(cudaGetErrorString(_e));        \
      return kStatusCuda;                            \
    }                                                \
  } while (0)

// m = P.nrhs independent right-hand sides against one operator / coarse
// factor (multi-RHS batching). Each RHS owns a complete
// single-solve workspace (RHS c at ws + c * per, so its coarse vectors sit at a
// fixed stride from RHS 0's and one coarse-solve launch serves all of them);
// every RHS runs the single-RHS kernels on its own vectors and state and stops
// on its own criterion, so its iterates, iteration count and result are
// bitwise those of solving it alone. Shared per iteration: the coarse solve
// (one pass over the factor for all RHS) and the graph launch / host check.
int pcg_solve_multi(const PcgProblem& P, PcgResult* R, int* rstat, cudaStream_t user_stream) {
  const Grid& G = P.g;
  const long long nd = 3 * G.nn;
  const int m = P.nrhs;
  if (m < 1 || m > kPcgMaxRhs) {
    set_last_error("number of right-hand sides out of range");
    return kStatusBadArg;
  }
  const bool defl = P.block > 0 && (P.coarse_kind == 1 || P.coarse != nullptr);
  Agglo A{};
  if (defl) A = make_agglo(G, P.block, P.h);
  const size_t per = pcg_ws_bytes(G, defl ? P.block : 0);
  if (P.ws_bytes < per * (size_t)m) {
    set_last_error("pcg workspace too small");
    return kStatusWorkspace;
  }
  PcgWork W[kPcgMaxRhs];
  for (int c = 0; c < m; ++c) W[c] = carve((char*)P.ws + per * c, G, defl ? P.block : 0);
  const long long ldc = (long long)(per / sizeof(double));  // coarse-vector stride between RHS
  const long long ld_done = (long long)(per / sizeof(int));  // SolverState::done stride between RHS
  DeflData D{const_cast<double*>(P.cen), const_cast<double*>(P.S), const_cast<int*>(P.keep)};
  if (P.coarse_kind == 1) D.perm = P.nd.perm;  // coarse vectors in the factor's ND order
  for (int c = 0; c < m; ++c) {
    R[c] = PcgResult{};
    rstat[c] = kStatusOk;
  }

  int dev = 0;
  TVB_CK(cudaGetDevice(&dev));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const MatvecPlan plan = plan_matvec(G, nsm);
  if (plan.nblocks() > 65536) {
    set_last_error("matvec grid too large for the partials buffer");
    return kStatusBadDims;
  }

  // own non-blocking stream (graph capture is illegal on the legacy stream)
  TVB_CK(cudaStreamSynchronize(user_stream));
  cudaStream_t s;
  TVB_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } guard{s};

  auto matvec = [&](int c, const double* u, double* y, bool with_dot, const int* stop) {
    MatvecParams mp{};
    mp.g = G;
    mp.u = u;
    mp.y = y;
    mp.occ = P.occ;
    mp.fixed = P.nflags;
    mp.mask_in = 0;  // solver vectors are already zero on fixed DOFs
    mp.mask_out = 1;
    mp.accumulate = 0;
    mp.dot_partial = with_dot ? W[c].partials + 2 * kMaxReduceCtas : nullptr;
    mp.stop = stop;
    return launch_matvec(plan, mp, P.modal, s);
  };
  // mu = E^-1 yc for RHS [c0, c0 + k) (one pass over the coarse factor)
  auto coarse_solve = [&](int c0, int k, const int* stop) -> cudaError_t {
    const int* st = stop ? &W[c0].st->done : nullptr;
    if (P.coarse_kind == 1) return launch_coarse_nd_multi(P.nd, k, W[c0].yc, ldc, W[c0].mu, ldc, st, ld_done, s);
    return launch_dense_gemv_multi(6 * A.nb, P.coarse, k, W[c0].yc, ldc, W[c0].mu, ldc, st, ld_done, s);
  };
  auto coarse_project = [&](int c, const double* v) -> cudaError_t {
    // nu = S E^-1 W^T v  (prologue: v = f or A z)
    cudaError_t e = launch_restrict(A, P.dflags, D, v, W[c].yc, s, nullptr, nullptr, W[c].st);
    if (e != cudaSuccess) return e;
    if ((e = coarse_solve(c, 1, nullptr)) != cudaSuccess) return e;
    return launch_block_nu(A, D, W[c].mu, W[c].nu, s, nullptr);
  };

  // Optional (TVB_L2_PERSIST=1): keep the nested-dissection coarse factor
  // resident in L2 with an access-policy window (captured into the graph's
  // kernel nodes). Measured slower at C3/C4 (the carve-out costs the
  // streaming matvecs more than the coarse solve gains), so off by default.
  if (P.coarse_kind == 1 && P.nd_factor != nullptr && P.nd_factor_bytes > 0 && getenv("TVB_L2_PERSIST")) {
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist > 0 && max_window > 0) {
      const size_t bytes = std::min(P.nd_factor_bytes, (size_t)max_window);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(bytes, (size_t)max_persist));
      cudaStreamAttrValue av = {};
      av.accessPolicyWindow.base_ptr = (void*)P.nd_factor;
      av.accessPolicyWindow.num_bytes = bytes;
      av.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)max_persist / (double)bytes);
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &av);
    }
    cudaGetLastError();  // the window is an optimisation only
  }

  // --- prologue (per RHS) ----------------------------------------------------
  // The Jacobi diagonal depends on the operator only: built once (RHS 0's
  // workspace) and read by every RHS.
  const double* inv_d = W[0].inv_d;
  TVB_CK(cudaMemsetAsync(W[0].zero_free, 0, sizeof(int), s));
  TVB_CK(launch_inv_diag(G, P.occ, P.nflags, P.kdiag, W[0].inv_d, nullptr, W[0].zero_free, s));
  int zero_free = 0;
  TVB_CK(cudaMemcpyAsync(&zero_free, W[0].zero_free, sizeof(int), cudaMemcpyDeviceToHost, s));
  // The iteration's matvecs skip the output mask (q and A z then hold
  // arbitrary values on fixed DOFs): the update kernel keeps r = z = 0 there
  // (inv_d == 0), p is 0 there so p.q is unaffected, and the restriction masks
  // the fixed DOFs of ITS flags -- valid when those cover the operator's
  // (always, unless the deflation space was built for another Dirichlet set:
  // then the masks stay on). TVB_SOLVE_MASKOUT=1 keeps them (A/B; bitwise
  // identical results either way).
  bool iter_mask_out = getenv("TVB_SOLVE_MASKOUT") && atoi(getenv("TVB_SOLVE_MASKOUT")) != 0;
  if (!iter_mask_out && defl && P.dflags != P.nflags) {
    int* d_unc = W[0].zero_free;  // reused after its read-back below
    TVB_CK(cudaStreamSynchronize(s));
    TVB_CK(cudaMemsetAsync(d_unc, 0, sizeof(int), s));
    k_flags_uncovered<<<(unsigned)((G.nn + 255) / 256), 256, 0, s>>>(G.nn, P.nflags, P.dflags, d_unc);
    int unc = 0;
    TVB_CK(cudaMemcpyAsync(&unc, d_unc, sizeof(int), cudaMemcpyDeviceToHost, s));
    TVB_CK(cudaStreamSynchronize(s));
    iter_mask_out = unc != 0;
  }
  bool active[kPcgMaxRhs];
  int n_active = 0;
  const int one = 1;
  for (int c = 0; c < m; ++c) {
    active[c] = false;
    SolverState st0{};
    st0.tol = P.tol;
    st0.max_iters = P.max_iters;
    TVB_CK(cudaMemcpyAsync(W[c].st, &st0, sizeof(st0), cudaMemcpyHostToDevice, s));
    TVB_CK(launch_free_norm(nd, P.fs[c], P.nflags, W[c].partials, W[c].st, s));
    SolverState hst{};
    TVB_CK(cudaMemcpyAsync(&hst, W[c].st, sizeof(hst), cudaMemcpyDeviceToHost, s));
    TVB_CK(cudaStreamSynchronize(s));
    R[c].fnorm = hst.fnorm;
    if (hst.fnorm == 0.0) {  // zero load: zero solution in 0 iterations (fea.py:243-245)
      TVB_CK(cudaMemsetAsync(P.xs[c], 0, nd * sizeof(double), s));
      TVB_CK(cudaMemcpyAsync(&W[c].st->done, &one, sizeof(int), cudaMemcpyHostToDevice, s));
      TVB_CK(cudaStreamSynchronize(s));
      continue;
    }
    if (zero_free > 0) {
      set_last_error("zero stiffness diagonal on a loaded free DOF");
      rstat[c] = kStatusSingular;
      TVB_CK(cudaMemcpyAsync(&W[c].st->done, &one, sizeof(int), cudaMemcpyHostToDevice, s));
      TVB_CK(cudaStreamSynchronize(s));
      continue;
    }
    double* x = P.xs[c];
    // x0
    if (defl) {
      TVB_CK(coarse_project(c, P.fs[c]));
      TVB_CK(launch_prolong(A, P.dflags, D, W[c].nu, x, nullptr, nullptr, 0, s));
    } else {
      TVB_CK(cudaMemsetAsync(x, 0, nd * sizeof(double), s));
    }
    // r = f - A x0 ; z = D^-1 r ; rz ; res
    TVB_CK(matvec(c, x, W[c].r, false, nullptr));
    TVB_CK(launch_pcg_init(nd, P.fs[c], W[c].r, W[c].z, inv_d, P.nflags, 1, W[c].partials, W[c].st, s));
    TVB_CK(cudaMemcpyAsync(&hst, W[c].st, sizeof(hst), cudaMemcpyDeviceToHost, s));
    TVB_CK(cudaStreamSynchronize(s));
    if (hst.done) {
      TVB_CK(launch_zero_fixed(G.nn, x, P.nflags, s));
      TVB_CK(cudaStreamSynchronize(s));
      R[c].residual = hst.res;
      continue;
    }
    // p = z - W E^-1 W^T A z  (or p = z)
    if (defl) {
      TVB_CK(matvec(c, W[c].z, W[c].q, false, nullptr));
      TVB_CK(coarse_project(c, W[c].q));
      TVB_CK(launch_prolong(A, P.dflags, D, W[c].nu, W[c].p, W[c].z, W[c].st, 2, s));
    } else {
      TVB_CK(cudaMemcpyAsync(W[c].p, W[c].z, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    active[c] = true;
    ++n_active;
  }
  if (n_active == 0) {
    for (int c = 0; c < m; ++c)
      if (rstat[c] != kStatusOk) return rstat[c];
    return kStatusOk;
  }
  // RHS that stopped in the prologue are inert in the graph (done flag set);
  // the coarse solve runs over the contiguous range of RHS that can be active
  int c_lo = 0, c_hi = m;
  while (!active[c_lo]) ++c_lo;
  while (!active[c_hi - 1]) --c_hi;

  // --- iteration graph -----------------------------------------------------
  // TVB_SOLVE_SKIP (timing experiments only -- the iterates are then wrong):
  // bitmask of iteration stages left out of the graph, 1 A p, 2 update, 4 A z,
  // 8 restriction, 16 coarse solve, 32 nu + prolongation; the in-graph cost of
  // a stage is the per-iteration time difference.
  const int skip = getenv("TVB_SOLVE_SKIP") ? atoi(getenv("TVB_SOLVE_SKIP")) : 0;
  // Several RHS: each RHS's chain runs on its own capture stream (graph
  // branch), so one RHS's small kernels overlap another's; the branches meet
  // only at the shared coarse solve. TVB_BATCH_FORK=0 serialises them.
  const bool fork = (c_hi - c_lo) > 1 && !(getenv("TVB_BATCH_FORK") && atoi(getenv("TVB_BATCH_FORK")) == 0);
  cudaStream_t bs[kPcgMaxRhs];
  cudaEvent_t ev_fork = nullptr, ev_branch[kPcgMaxRhs] = {};
  int n_streams = 0;
  struct ForkGuard {
    cudaStream_t* s;
    int* n;
    cudaEvent_t* ev0;
    cudaEvent_t* ev;
    ~ForkGuard() {
      for (int i = 0; i < *n; ++i) {
        cudaStreamDestroy(s[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
      }
      if (*ev0) cudaEventDestroy(*ev0);
    }
  } fguard{bs, &n_streams, &ev_fork, ev_branch};
  if (fork) {
    TVB_CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    for (int c = c_lo; c < c_hi; ++c) {
      TVB_CK(cudaStreamCreateWithFlags(&bs[n_streams], cudaStreamNonBlocking));
      TVB_CK(cudaEventCreateWithFlags(&ev_branch[n_streams], cudaEventDisableTiming));
      ++n_streams;
    }
  }
  auto sc = [&](int c) { return fork ? bs[c - c_lo] : s; };
  // s -> every branch (fork) / every branch -> s (join)
  auto fork_from_s = [&]() -> cudaError_t {
    if (!fork) return cudaSuccess;
    cudaError_t e = cudaEventRecord(ev_fork, s);
    for (int c = c_lo; c < c_hi && e == cudaSuccess; ++c) e = cudaStreamWaitEvent(sc(c), ev_fork, 0);
    return e;
  };
  auto join_to_s = [&]() -> cudaError_t {
    if (!fork) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    for (int c = c_lo; c < c_hi && e == cudaSuccess; ++c) {
      e = cudaEventRecord(ev_branch[c - c_lo], sc(c));
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_branch[c - c_lo], 0);
    }
    return e;
  };
  auto one_iteration = [&]() -> cudaError_t {
    cudaError_t e = cudaSuccess;
    for (int c = c_lo; c < c_hi; ++c) {
      const int* stop = &W[c].st->done;
      cudaStream_t cs = sc(c);
      MatvecParams mp{};
      if (!(skip & 1)) {
        mp.g = G;
        mp.u = W[c].p;
        mp.y = W[c].q;
        mp.occ = P.occ;
        mp.fixed = P.nflags;
        mp.mask_out = iter_mask_out ? 1 : 0;
        mp.dot_partial = W[c].partials + 2 * kMaxReduceCtas;
        mp.stop = stop;
        if ((e = launch_matvec(plan, mp, P.modal, cs)) != cudaSuccess) return e;
      }
      if (!(skip & 2) &&
          (e = launch_pcg_update(nd, defl ? nullptr : P.xs[c], W[c].r, W[c].z, W[c].p, W[c].q, inv_d, W[c].st,
                                 W[c].partials, W[c].partials + 2 * kMaxReduceCtas, plan.nblocks(), cs)) !=
              cudaSuccess)
        return e;
      if (!defl) {
        if ((e = launch_pcg_pupdate(nd, W[c].p, W[c].z, W[c].st, cs)) != cudaSuccess) return e;
        continue;
      }
      if (!(skip & 4)) {
        mp = MatvecParams{};
        mp.g = G;
        mp.u = W[c].z;
        mp.y = W[c].t;
        mp.occ = P.occ;
        mp.fixed = P.nflags;
        mp.mask_out = iter_mask_out ? 1 : 0;
        mp.stop = stop;
        if ((e = launch_matvec(plan, mp, P.modal, cs)) != cudaSuccess) return e;
      }
      if (!(skip & 8) &&
          (e = launch_restrict(A, P.dflags, D, W[c].t, W[c].yc, cs, stop, P.stabilized ? W[c].q : nullptr,
                               W[c].st)) != cudaSuccess)
        return e;
    }
    if (!defl) return cudaSuccess;
    if ((e = join_to_s()) != cudaSuccess) return e;
    // dense coarse inverse: mu and nu = S mu in one launch (k_dense_gemv_nu); TVB_DENSE_NU_FUSED=0: two launches
    static const bool fuse_nu_env = !(getenv("TVB_DENSE_NU_FUSED") && atoi(getenv("TVB_DENSE_NU_FUSED")) == 0);
    const bool fused_nu = fuse_nu_env && P.coarse_kind != 1 && !(skip & 48);
    if (fused_nu) {
      if ((e = launch_dense_gemv_nu_multi(A.nb, P.coarse, P.S, c_hi - c_lo, W[c_lo].yc, ldc, W[c_lo].mu, ldc,
                                          W[c_lo].nu, ldc, &W[c_lo].st->done, ld_done, s)) != cudaSuccess)
        return e;
    } else if (!(skip & 16) && (e = coarse_solve(c_lo, c_hi - c_lo, &W[c_lo].st->done)) != cudaSuccess) {
      return e;
    }
    if ((e = fork_from_s()) != cudaSuccess) return e;
    if (skip & 32) return cudaSuccess;
    for (int c = c_lo; c < c_hi; ++c) {
      const int* stop = &W[c].st->done;
      if (!fused_nu && (e = launch_block_nu(A, D, W[c].mu, W[c].nu, sc(c), stop)) != cudaSuccess) return e;
      // p = z + beta p - W nu, and the deferred x += alpha p_old of this iteration
      if ((e = launch_prolong(A, P.dflags, D, W[c].nu, W[c].p, W[c].z, W[c].st, 1, sc(c), P.xs[c])) != cudaSuccess)
        return e;
    }
    return cudaSuccess;
  };
  // TVB_SOLVE_PROFILE=1 (single RHS): run a few iterations eagerly with CUDA
  // events around every stage and print the per-stage device time (tuning only).
  if (getenv("TVB_SOLVE_PROFILE") && m == 1) {
    const char* names[6] = {"matvec_Ap+pq", "pcg_update", "matvec_Az", "restrict", "coarse_solve", "nu+prolong"};
    double acc[6] = {0, 0, 0, 0, 0, 0};
    cudaEvent_t ev[7];
    for (auto& e : ev) cudaEventCreate(&e);
    const int* stop = &W[0].st->done;
    int nit = 0;
    for (; nit < 20; ++nit) {
      cudaEventRecord(ev[0], s);
      matvec(0, W[0].p, W[0].q, true, stop);
      cudaEventRecord(ev[1], s);
      launch_pcg_update(nd, defl ? nullptr : P.xs[0], W[0].r, W[0].z, W[0].p, W[0].q, inv_d, W[0].st,
                        W[0].partials, W[0].partials + 2 * kMaxReduceCtas, plan.nblocks(), s);
      cudaEventRecord(ev[2], s);
      if (defl) {
        matvec(0, W[0].z, W[0].t, false, stop);
        cudaEventRecord(ev[3], s);
        launch_restrict(A, P.dflags, D, W[0].t, W[0].yc, s, stop, P.stabilized ? W[0].q : nullptr, W[0].st);
        cudaEventRecord(ev[4], s);
        coarse_solve(0, 1, stop);
        cudaEventRecord(ev[5], s);
        launch_block_nu(A, D, W[0].mu, W[0].nu, s, stop);
        launch_prolong(A, P.dflags, D, W[0].nu, W[0].p, W[0].z, W[0].st, 1, s, P.xs[0]);
      } else {
        launch_pcg_pupdate(nd, W[0].p, W[0].z, W[0].st, s);
        for (int k = 3; k < 6; ++k) cudaEventRecord(ev[k], s);
      }
      cudaEventRecord(ev[6], s);
      cudaStreamSynchronize(s);
      for (int k = 0; k < 6; ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
        acc[k] += ms;
      }
    }
    fprintf(stderr, "[tvb solve profile] per-iteration us:");
    for (int k = 0; k < 6; ++k) fprintf(stderr, " %s=%.1f", names[k], 1e3 * acc[k] / nit);
    fprintf(stderr, "\n");
    for (auto& e : ev) cudaEventDestroy(e);
  }
  int batch = P.check_every > 0 ? P.check_every : 8;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // Whole-solve graph (TVB_GRAPH_WHILE=1): a conditional WHILE node whose body holds
  // `check_every` iterations (TVB_WHILE_BODY overrides) and a one-thread
  // kernel that re-arms the condition while any RHS is running, so the
  // iteration loop never returns to the host (no per-batch launch + state
  // read-back + synchronise). Measured within noise of the host loop at C1-C4
  // (the per-batch round trips were already hidden), 1 % faster for the 2-RHS
  // C4 batch; bodies of 4-8 iterations beat 1-2 (C1 5.64 vs 6.04 ms per solve).
  // Not the default: kernels inside conditional bodies are invisible to the
  // ncu launch lists (profiles/) and per-kernel tracing, for no measured gain.
  // Default: graphs of `check_every` iterations launched from a host loop.
  static const int while_env = getenv("TVB_GRAPH_WHILE") ? atoi(getenv("TVB_GRAPH_WHILE")) : 0;
  const bool use_while = while_env != 0;
  if (use_while) {
    static const int body_env = getenv("TVB_WHILE_BODY") ? atoi(getenv("TVB_WHILE_BODY")) : 0;
    const int wbatch = body_env > 0 ? body_env : (P.check_every > 0 ? P.check_every : 8);
    TVB_CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    TVB_CK(cudaGraphConditionalHandleCreate(&cond, graph, 1u, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t cnode;
    TVB_CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    TVB_CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    cudaError_t cap = fork_from_s();
    for (int i = 0; i < wbatch && cap == cudaSuccess; ++i) cap = one_iteration();
    if (cap == cudaSuccess) cap = join_to_s();
    if (cap == cudaSuccess) {
      k_loop_cond<<<1, 1, 0, s>>>(cond, &W[c_lo].st->done, ld_done, c_hi - c_lo);
      cap = cudaGetLastError();
    }
    cudaGraph_t body_out = body;
    cudaError_t endcap = cudaStreamEndCapture(s, &body_out);
    if (cap != cudaSuccess || endcap != cudaSuccess) cudaGraphDestroy(graph);
    TVB_CK(cap);
    TVB_CK(endcap);
    cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    if (ie != cudaSuccess) cudaGraphDestroy(graph);
    TVB_CK(ie);
    batch = P.max_iters + wbatch;  // one launch runs the whole solve
  } else {
    TVB_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaError_t cap = fork_from_s();
    for (int i = 0; i < batch && cap == cudaSuccess; ++i) cap = one_iteration();
    if (cap == cudaSuccess) cap = join_to_s();
    cudaError_t endcap = cudaStreamEndCapture(s, &graph);
    TVB_CK(cap);
    TVB_CK(endcap);
    TVB_CK(cudaGraphInstantiate(&exec, graph, 0));
  }
  struct GraphGuard {
    cudaGraph_t g;
    cudaGraphExec_t e;
    ~GraphGuard() {
      if (e) cudaGraphExecDestroy(e);
      if (g) cudaGraphDestroy(g);
    }
  } gguard{graph, exec};

  SolverState hst[kPcgMaxRhs];
  int iters_launched = 0;
  while (true) {
    TVB_CK(cudaGraphLaunch(exec, s));
    iters_launched += batch;
    for (int c = c_lo; c < c_hi; ++c)
      if (active[c]) TVB_CK(cudaMemcpyAsync(&hst[c], W[c].st, sizeof(SolverState), cudaMemcpyDeviceToHost, s));
    TVB_CK(cudaStreamSynchronize(s));
    bool all_done = true;
    for (int c = c_lo; c < c_hi; ++c) all_done = all_done && (!active[c] || hst[c].done);
    if (all_done) break;
    if (use_while || iters_launched > P.max_iters + batch) {  // the device loop exits only when all are done
      set_last_error("solver state did not terminate");
      return kStatusCuda;
    }
  }
  int status = kStatusOk;
  for (int c = 0; c < m; ++c) {
    if (!active[c]) {
      if (rstat[c] != kStatusOk && status == kStatusOk) status = rstat[c];
      continue;
    }
    // the stopping iteration's x += alpha p rode on its (skipped) prolongation
    if (defl && hst[c].iter > 0) TVB_CK(launch_x_finish(nd, P.xs[c], W[c].p, W[c].st, s));
    R[c].iterations = hst[c].iter;
    R[c].residual = hst[c].res;
    if (hst[c].done == 2) {
      char buf[160];
      snprintf(buf, sizeof(buf), "CG did not reach %g in %d iterations (residual %.3e)", P.tol, P.max_iters,
               hst[c].res);
      set_last_error(buf);
      rstat[c] = kStatusNoConvergence;
      if (status == kStatusOk) status = kStatusNoConvergence;
      continue;
    }
    TVB_CK(launch_zero_fixed(G.nn, P.xs[c], P.nflags, s));
  }
  TVB_CK(cudaStreamSynchronize(s));
  return status;
}

int pcg_solve(const PcgProblem& P, PcgResult& R, cudaStream_t user_stream) {
  PcgProblem Q = P;
  Q.nrhs = 1;
  Q.fs[0] = P.f;
  Q.xs[0] = P.x;
  int st1 = 0;
  const int st = pcg_solve_multi(Q, &R, &st1, user_stream);
  return st;
}

}  // namespace tvb
