// a8: (deflated) Jacobi-preconditioned CG driver, replacing solve_static
// (topovox/fea.py:218-299). The host loop only launches CUDA graphs that each
// contain `check_every` complete iterations and reads back two ints per
// launch; all scalars (alpha, beta, residual, stop flag) live on the device.
//
// Algorithm (identical to the reference, step for step):
//   x0 = W E^-1 W^T f ; r = f - A x0 ; r[fixed] = 0 ; stop if |r|/|f_free| <= tol
//   z = D^-1 r ; p = z - W E^-1 (AW)^T z ; rz = r.z
//   loop: q = A p ; alpha = rz/(p.q) ; x += alpha p ; r -= alpha q
//         stop if |r|/|f_free| <= tol ; z = D^-1 r ; beta = r.z_new / rz
//         p = z + beta p - W E^-1 (AW)^T z
// with (AW)^T z evaluated as W^T (A z) (A symmetric, W zero on fixed DOFs).
//
// Stabilised projection: the loop projects z + beta p instead of z,
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
__global__ void k_dense_gemv(long long nc, const double* Einv, const double* yc, double* mu, const int* stop) {
  if (stop != nullptr && *stop) return;
  const long long row = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nc) return;
  const double* a = Einv + row * nc;
  double s = 0.0;
  for (long long j = lane; j < nc; j += 32) s = fma(a[j], yc[j], s);
  s = warp_sum(s);
  if (lane == 0) mu[row] = s;
}

cudaError_t launch_dense_gemv(long long nc, const double* Einv, const double* yc, double* mu, const int* stop,
                              cudaStream_t s) {
  const long long threads = nc * 32;
  k_dense_gemv<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(nc, Einv, yc, mu, stop);
  return cudaGetLastError();
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

int pcg_solve(const PcgProblem& P, PcgResult& R, cudaStream_t user_stream) {
  const Grid& G = P.g;
  const long long nd = 3 * G.nn;
  const bool defl = P.block > 0 && (P.coarse_kind == 1 || P.coarse != nullptr);
  Agglo A{};
  if (defl) A = make_agglo(G, P.block, P.h);
  if (P.ws_bytes < pcg_ws_bytes(G, defl ? P.block : 0)) {
    set_last_error("pcg workspace too small");
    return kStatusWorkspace;
  }
  PcgWork W = carve(P.ws, G, defl ? P.block : 0);
  DeflData D{const_cast<double*>(P.cen), const_cast<double*>(P.S), const_cast<int*>(P.keep)};
  if (P.coarse_kind == 1) D.perm = P.nd.perm;  // coarse vectors in the factor's ND order

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

  auto matvec = [&](const double* u, double* y, bool with_dot, const int* stop) {
    MatvecParams mp{};
    mp.g = G;
    mp.u = u;
    mp.y = y;
    mp.occ = P.occ;
    mp.fixed = P.nflags;
    mp.mask_in = 0;  // solver vectors are already zero on fixed DOFs
    mp.mask_out = 1;
    mp.accumulate = 0;
    mp.dot_partial = with_dot ? W.partials + 2 * kMaxReduceCtas : nullptr;
    mp.stop = stop;
    return launch_matvec(plan, mp, P.modal, s);
  };
  auto coarse_project = [&](const double* v, const int* stop, const double* v2 = nullptr) -> cudaError_t {
    // nu = S E^-1 W^T (v + beta v2)  (v = f, A z ; v2 = q)
    cudaError_t e = launch_restrict(A, P.nflags, D, v, W.yc, s, stop, v2, W.st);
    if (e != cudaSuccess) return e;
    if (P.coarse_kind == 1) e = launch_coarse_nd(P.nd, W.yc, W.mu, stop, s);
    else e = launch_dense_gemv(6 * A.nb, P.coarse, W.yc, W.mu, stop, s);
    if (e != cudaSuccess) return e;
    return launch_block_nu(A, D, W.mu, W.nu, s, stop);
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

  // --- prologue ------------------------------------------------------------
  SolverState st0{};
  st0.tol = P.tol;
  st0.max_iters = P.max_iters;
  TVB_CK(cudaMemcpyAsync(W.st, &st0, sizeof(st0), cudaMemcpyHostToDevice, s));
  TVB_CK(cudaMemsetAsync(W.zero_free, 0, sizeof(int), s));
  TVB_CK(launch_free_norm(nd, P.f, P.nflags, W.partials, W.st, s));
  TVB_CK(launch_inv_diag(G, P.occ, P.nflags, P.kdiag, W.inv_d, nullptr, W.zero_free, s));
  SolverState hst{};
  int zero_free = 0;
  TVB_CK(cudaMemcpyAsync(&hst, W.st, sizeof(hst), cudaMemcpyDeviceToHost, s));
  TVB_CK(cudaMemcpyAsync(&zero_free, W.zero_free, sizeof(int), cudaMemcpyDeviceToHost, s));
  TVB_CK(cudaStreamSynchronize(s));
  R.fnorm = hst.fnorm;
  if (hst.fnorm == 0.0) {
    TVB_CK(cudaMemsetAsync(P.x, 0, nd * sizeof(double), s));
    TVB_CK(cudaStreamSynchronize(s));
    R.iterations = 0;
    R.residual = 0.0;
    return kStatusOk;
  }
  if (zero_free > 0) {
    set_last_error("zero stiffness diagonal on a loaded free DOF");
    return kStatusSingular;
  }
  // x0
  if (defl) {
    TVB_CK(coarse_project(P.f, nullptr));
    TVB_CK(launch_prolong(A, P.nflags, D, W.nu, P.x, nullptr, nullptr, 0, s));
  } else {
    TVB_CK(cudaMemsetAsync(P.x, 0, nd * sizeof(double), s));
  }
  // r = f - A x0 ; z = D^-1 r ; rz ; res
  TVB_CK(matvec(P.x, W.r, false, nullptr));
  TVB_CK(launch_pcg_init(nd, P.f, W.r, W.z, W.inv_d, P.nflags, 1, W.partials, W.st, s));
  TVB_CK(cudaMemcpyAsync(&hst, W.st, sizeof(hst), cudaMemcpyDeviceToHost, s));
  TVB_CK(cudaStreamSynchronize(s));
  if (hst.done) {
    TVB_CK(launch_zero_fixed(G.nn, P.x, P.nflags, s));
    TVB_CK(cudaStreamSynchronize(s));
    R.iterations = 0;
    R.residual = hst.res;
    return kStatusOk;
  }
  // p = z - W E^-1 W^T A z  (or p = z)
  if (defl) {
    TVB_CK(matvec(W.z, W.q, false, nullptr));
    TVB_CK(coarse_project(W.q, nullptr));
    TVB_CK(launch_prolong(A, P.nflags, D, W.nu, W.p, W.z, W.st, 2, s));
  } else {
    TVB_CK(cudaMemcpyAsync(W.p, W.z, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }

  // --- iteration graph -----------------------------------------------------
  const int* stop = &W.st->done;
  // TVB_SOLVE_SKIP (timing experiments only -- the iterates are then wrong):
  // bitmask of iteration stages left out of the graph, 1 A p, 2 update, 4 A z,
  // 8 restriction, 16 coarse solve, 32 nu + prolongation; the in-graph cost of
  // a stage is the per-iteration time difference.
  const int skip = getenv("TVB_SOLVE_SKIP") ? atoi(getenv("TVB_SOLVE_SKIP")) : 0;
  auto one_iteration = [&]() -> cudaError_t {
    cudaError_t e = cudaSuccess;
    if (!(skip & 1) && (e = matvec(W.p, W.q, true, stop)) != cudaSuccess) return e;
    if (!(skip & 2) &&
        (e = launch_pcg_update(nd, defl ? nullptr : P.x, W.r, W.z, W.p, W.q, W.inv_d, W.st, W.partials,
                               W.partials + 2 * kMaxReduceCtas, plan.nblocks(), s)) != cudaSuccess)
      return e;
    if (defl) {
      if (!(skip & 4) && (e = matvec(W.z, W.t, false, stop)) != cudaSuccess) return e;
      if (!(skip & 8) && (e = launch_restrict(A, P.nflags, D, W.t, W.yc, s, stop, W.q, W.st)) != cudaSuccess)
        return e;
      if (!(skip & 16)) {
        e = P.coarse_kind == 1 ? launch_coarse_nd(P.nd, W.yc, W.mu, stop, s)
                               : launch_dense_gemv(6 * A.nb, P.coarse, W.yc, W.mu, stop, s);
        if (e != cudaSuccess) return e;
      }
      if (skip & 32) return cudaSuccess;
      if ((e = launch_block_nu(A, D, W.mu, W.nu, s, stop)) != cudaSuccess) return e;
      // p = z + beta p - W nu, and the deferred x += alpha p_old of this iteration
      return launch_prolong(A, P.nflags, D, W.nu, W.p, W.z, W.st, 1, s, P.x);
    }
    return launch_pcg_pupdate(nd, W.p, W.z, W.st, s);
  };
  // TVB_SOLVE_PROFILE=1: run a few iterations eagerly with CUDA events around
  // every stage and print the per-stage device time (tuning only).
  if (getenv("TVB_SOLVE_PROFILE")) {
    const char* names[6] = {"matvec_Ap+pq", "pcg_update", "matvec_Az", "restrict", "coarse_solve", "nu+prolong"};
    double acc[6] = {0, 0, 0, 0, 0, 0};
    cudaEvent_t ev[7];
    for (auto& e : ev) cudaEventCreate(&e);
    int nit = 0;
    for (; nit < 20; ++nit) {
      cudaEventRecord(ev[0], s);
      matvec(W.p, W.q, true, stop);
      cudaEventRecord(ev[1], s);
      launch_pcg_update(nd, defl ? nullptr : P.x, W.r, W.z, W.p, W.q, W.inv_d, W.st, W.partials,
                        W.partials + 2 * kMaxReduceCtas, plan.nblocks(), s);
      cudaEventRecord(ev[2], s);
      if (defl) {
        matvec(W.z, W.t, false, stop);
        cudaEventRecord(ev[3], s);
        launch_restrict(A, P.nflags, D, W.t, W.yc, s, stop, W.q, W.st);
        cudaEventRecord(ev[4], s);
        if (P.coarse_kind == 1) launch_coarse_nd(P.nd, W.yc, W.mu, stop, s);
        else launch_dense_gemv(6 * A.nb, P.coarse, W.yc, W.mu, stop, s);
        cudaEventRecord(ev[5], s);
        launch_block_nu(A, D, W.mu, W.nu, s, stop);
        launch_prolong(A, P.nflags, D, W.nu, W.p, W.z, W.st, 1, s, P.x);
      } else {
        launch_pcg_pupdate(nd, W.p, W.z, W.st, s);
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
  TVB_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  cudaError_t cap = cudaSuccess;
  for (int i = 0; i < batch && cap == cudaSuccess; ++i) cap = one_iteration();
  cudaError_t endcap = cudaStreamEndCapture(s, &graph);
  TVB_CK(cap);
  TVB_CK(endcap);
  TVB_CK(cudaGraphInstantiate(&exec, graph, 0));
  struct GraphGuard {
    cudaGraph_t g;
    cudaGraphExec_t e;
    ~GraphGuard() {
      if (e) cudaGraphExecDestroy(e);
      if (g) cudaGraphDestroy(g);
    }
  } gguard{graph, exec};

  int iters_launched = 0;
  while (true) {
    TVB_CK(cudaGraphLaunch(exec, s));
    iters_launched += batch;
    TVB_CK(cudaMemcpyAsync(&hst, W.st, sizeof(hst), cudaMemcpyDeviceToHost, s));
    TVB_CK(cudaStreamSynchronize(s));
    if (hst.done) break;
    if (iters_launched > P.max_iters + batch) {
      set_last_error("solver state did not terminate");
      return kStatusCuda;
    }
  }
  // the stopping iteration's x += alpha p rode on its (skipped) prolongation
  if (defl && hst.iter > 0) TVB_CK(launch_x_finish(nd, P.x, W.p, W.st, s));
  R.iterations = hst.iter;
  R.residual = hst.res;
  if (hst.done == 2) {
    char buf[160];
    snprintf(buf, sizeof(buf), "CG did not reach %g in %d iterations (residual %.3e)", P.tol, P.max_iters, hst.res);
    set_last_error(buf);
    return kStatusNoConvergence;
  }
  TVB_CK(launch_zero_fixed(G.nn, P.x, P.nflags, s));
  TVB_CK(cudaStreamSynchronize(s));
  return kStatusOk;
}

}  // namespace tvb
