/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY. Never linked into the product path.
 *
 * Plain-C restatement of the reference's CPU kernels
 * (/root/reference/pkg/src/topovox/backends/numba_kernels.py):
 *   oracle_apply_block24        <- apply_block24        (numba_kernels.py:12-28)
 *   oracle_apply_block24_subset <- apply_block24_subset (numba_kernels.py:31-46)
 *   oracle_diag_block24         <- diag_block24         (numba_kernels.py:49-58)
 * Same arguments, same accumulate-into-`out` contract, same 8-colour
 * phase order (element_coloring, backends/__init__.py:59-66): colours run in
 * sequence, elements of one colour in parallel (pthreads, a barrier between
 * colours), so the result is bitwise independent of the thread count, as in
 * the reference.
 */
#define _POSIX_C_SOURCE 200809L
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <unistd.h>

static int g_threads = 0;

static inline void element_apply(const double* u, double* out, const int32_t* dofs, double s, const double* k0) {
  double ue[24];
  for (int a = 0; a < 24; ++a) ue[a] = u[dofs[a]];
  for (int a = 0; a < 24; ++a) {
    double acc = 0.0;
    const double* row = k0 + 24 * a;
    for (int b = 0; b < 24; ++b) acc += row[b] * ue[b];
    out[dofs[a]] += s * acc;
  }
}

typedef struct {
  const double* u;
  double* out;
  const int32_t* elem_dofs;
  const double* scale;
  const double* k0;
  const int64_t* perm;
  const int64_t* ptr;
  int ncolors, tid, nthreads;
  pthread_barrier_t* bar;
} job_t;

static void* worker(void* arg) {
  job_t* j = (job_t*)arg;
  for (int c = 0; c < j->ncolors; ++c) {
    const int64_t lo = j->ptr[c], hi = j->ptr[c + 1], n = hi - lo;
    const int64_t a = lo + n * j->tid / j->nthreads, b = lo + n * (j->tid + 1) / j->nthreads;
    for (int64_t idx = a; idx < b; ++idx) {
      const int64_t e = j->perm[idx];
      const double s = j->scale[e];
      if (s == 0.0) continue;
      element_apply(j->u, j->out, j->elem_dofs + 24 * e, s, j->k0);
    }
    pthread_barrier_wait(j->bar);
  }
  return NULL;
}

int oracle_max_threads(void) {
  if (g_threads > 0) return g_threads;
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

void oracle_set_threads(int n) { g_threads = n > 0 ? n : 0; }

void oracle_apply_block24(const double* u, double* out, const int32_t* elem_dofs, const double* scale,
                          const double* k0, const int64_t* color_perm, const int64_t* color_ptr, int ncolors) {
  int T = oracle_max_threads();
  if (T > 256) T = 256;
  pthread_t th[256];
  job_t jobs[256];
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)T);
  for (int t = 0; t < T; ++t) {
    jobs[t] = (job_t){u, out, elem_dofs, scale, k0, color_perm, color_ptr, ncolors, t, T, &bar};
    if (t > 0) pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  worker(&jobs[0]);
  for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&bar);
}

void oracle_apply_block24_subset(const double* u, double* out, const int64_t* elem_ids, int64_t m,
                                 const int32_t* elem_dofs, const double* scale, const double* k0) {
  for (int64_t t = 0; t < m; ++t) {
    const int64_t e = elem_ids[t];
    const double s = scale[e];
    if (s == 0.0) continue;
    element_apply(u, out, elem_dofs + 24 * e, s, k0);
  }
}

void oracle_diag_block24(double* out, const int32_t* elem_dofs, const double* scale, int64_t n_elems,
                         const double* k0_diag) {
  for (int64_t e = 0; e < n_elems; ++e) {
    const double s = scale[e];
    if (s == 0.0) continue;
    for (int a = 0; a < 24; ++a) out[elem_dofs[24 * e + a]] += s * k0_diag[a];
  }
}

