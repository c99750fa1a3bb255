#pragma once
#include "common.cuh"

namespace tvb {

constexpr int kMaxReduceCtas = 1184;  // 8 x 148 SMs

// Device-resident scalar state of one (deflated) PCG solve. Kernels read the
// scalars they need from here, so a whole iteration can be replayed from a
// CUDA graph without host round trips; `done` makes every kernel a no-op once
// the solve has stopped.
struct SolverState {
  double rz;      // r . z of the current iterate
  double pq;      // p . A p
  double rr;      // ||r||^2
  double alpha, beta;
  double fnorm;   // ||f_free||
  double tol;
  double res;     // last relative (recursive) residual
  int iter;       // completed iterations
  int max_iters;
  int done;       // 0 running, 1 converged, 2 iteration cap
  unsigned int counter;  // last-CTA counter of the fused reductions
};

int reduce_grid(long long n);

cudaError_t launch_inv_diag(const Grid& G, const double* occ, const uint8_t* nflags, const double kd[3],
                            double* inv_d, double* diag_out, int* zero_free, cudaStream_t s, int accumulate = 0);
cudaError_t launch_dot(const double* a, const double* b, const double* w, long long n, double* ws,
                       unsigned int* counter, double* out, cudaStream_t s);
// pq_parts (optional): the matvec's per-CTA p.q partials (n_parts), summed in
// the update kernel itself; nullptr = st->pq already final
cudaError_t launch_pcg_update(long long n, double* x, double* r, double* z, const double* p, const double* q,
                              const double* inv_d, SolverState* st, double* partials, const double* pq_parts,
                              int n_parts, cudaStream_t s);
// x += alpha p with alpha from the solver state: the last iteration's deferred
// x update (its prolongation, which carries it, is skipped once done is set)
cudaError_t launch_x_finish(long long n, double* x, const double* p, const SolverState* st, cudaStream_t s);
cudaError_t launch_pcg_pupdate(long long n, double* p, const double* z, const SolverState* st, cudaStream_t s);
cudaError_t launch_finalize_pq(const double* partials, int nparts, SolverState* st, cudaStream_t s);
cudaError_t launch_pcg_init(long long n, const double* f, double* r, double* z, const double* inv_d,
                            const uint8_t* nflags, int have_ax, double* partials, SolverState* st, cudaStream_t s);
cudaError_t launch_free_norm(long long n, const double* f, const uint8_t* nflags, double* partials, SolverState* st,
                             cudaStream_t s);
cudaError_t launch_zero_fixed(long long nn, double* x, const uint8_t* nflags, cudaStream_t s);

}  // namespace tvb
