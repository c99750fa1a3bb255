#pragma once
#include "coarse.cuh"
#include "common.cuh"

namespace tvb {

void set_last_error(const char* msg);

constexpr int kPcgMaxRhs = 8;  // right-hand sides per batched solve

struct PcgProblem {
  Grid g;
  double h;
  Modal modal;
  double kdiag[3];
  const double* occ;
  const uint8_t* nflags;
  const double* f;
  double* x;
  void* ws;
  size_t ws_bytes;
  double tol;
  int max_iters;
  int check_every;
  int block;  // <= 0: no deflation
  const double* cen;
  const double* S;
  const int* keep;
  const double* coarse;  // dense inverse (coarse_kind 0)
  int coarse_kind;       // 0 dense inverse, 1 nested dissection
  bool stabilized = false;
  const uint8_t* dflags = nullptr;  // deflation space's node flags (restriction / prolongation)  // projection of z + beta p (solver.cu header) instead of z
  CoarseNDDev nd;
  const double* nd_factor = nullptr;  // L2-persisting window (the ND factor)
  size_t nd_factor_bytes = 0;
  // multi-RHS (pcg_solve_multi): nrhs right-hand sides / solutions
  int nrhs = 1;
  const double* fs[kPcgMaxRhs] = {};
  double* xs[kPcgMaxRhs] = {};
};

struct PcgResult {
  int iterations = 0;
  double residual = 0.0;
  double fnorm = 0.0;
};

size_t pcg_ws_bytes(const Grid& g, int block);
int pcg_solve(const PcgProblem& P, PcgResult& R, cudaStream_t user_stream);
// P.nrhs solves sharing the operator and coarse factor; workspace
// P.nrhs * pcg_ws_bytes(); R / rstat: per-RHS results and statuses. Returns
// the first failing status (kStatusNoConvergence if only convergence failed).
int pcg_solve_multi(const PcgProblem& P, PcgResult* R, int* rstat, cudaStream_t user_stream);
cudaError_t launch_dense_gemv_multi(long long nc, const double* Einv, int ncols, const double* yc, long long ldy,
                                    double* mu, long long ldm, const int* stop, long long stop_ld, cudaStream_t s);
cudaError_t launch_dense_gemv(long long nc, const double* Einv, const double* yc, double* mu, const int* stop,
                              cudaStream_t s);

}  // namespace tvb
