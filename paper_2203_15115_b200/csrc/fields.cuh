#pragma once
#include "common.cuh"

namespace tvb {

// isotropic elasticity in the reference's Voigt form (topovox/elements.py:72-79)
// plus the Eq 3.2 constants: d0 = c(1-nu), d1 = c nu, d2 = c(1-2nu)/2,
// c = E/((1+nu)(1-2nu)); c1 = 4/(1+nu), c2 = (1-3nu)/(1-nu^2).
struct Elastic {
  double d0, d1, d2, c1, c2;
};

struct ElemArgs {
  Grid g;
  Elastic D;
  double inv4h;            // 1/(4h): centroid shape-gradient magnitude
  const double* u;
  const double* occ;
  double* strains;         // [Ne][6] or null
  double* stresses;        // [Ne][6] or null
  double* vm;              // [Ne] or null
  double* tj;              // [Ne] compliance sensitivity or null
  double* pnorm_partials;  // [nblocks][2] = (sum occ vm^p, sum occ) or null
  int p;
};

constexpr int kMaxFields = 8;
struct CombineArgs {
  int k;
  const double* f[kMaxFields];
  double w[kMaxFields];
  const double* maxabs;  // device [k]
};

int elem_grid(long long n);
int elem_state_ctas(const Grid& G);
cudaError_t launch_element_state(const ElemArgs& A, cudaStream_t s);
cudaError_t launch_stress_sens(const ElemArgs& A, const double* lam, double* ts, cudaStream_t s);
// sums: device [2] = (sum occ vm^p, sum occ)
cudaError_t launch_adjoint(const ElemArgs& A, const double* sums, double* h6, const uint8_t* nflags, double* rhs,
                           cudaStream_t s);
cudaError_t launch_sum_pairs(const double* partials, int np, double* out2, cudaStream_t s);
cudaError_t launch_maxabs(const double* t, long long n, double* partials, double* out, cudaStream_t s);
cudaError_t launch_combine(const CombineArgs& C, long long n, double* out, cudaStream_t s);
size_t select_ws_bytes(long long n);
cudaError_t launch_select(const double* ls, const uint8_t* design, long long n, long long k, double ersatz,
                          double nondesign, double* occ, void* ws, unsigned long long* state_out, cudaStream_t s,
                          int all_ties = 0);
// casting projection along axis (0/1/2); element layers >= P form the +axis half
cudaError_t launch_casting_project(const Grid& G, int axis, int P, const double* in, double* out, cudaStream_t s);

}  // namespace tvb
