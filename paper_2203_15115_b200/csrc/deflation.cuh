#pragma once
#include "common.cuh"

namespace tvb {

// node flag byte: bits 0..2 = DOF fixed on axis a, bit 3 = structural node
// (touches an element with occupancy exactly 1.0, topovox/fea.py:119-123).
constexpr uint8_t kStructBit = 8;

// Agglomerate (deflation block) geometry. Block id = bx + mx*(by + my*bz)
// exactly like topovox/fea.py:125-126; a block owns the CLOSED node box
// [b*bx, b*bx + b] x ... clipped to the grid (topovox/fea.py:137).
struct Agglo {
  Grid g;
  int b;
  int mx, my, mz;
  long long nb;
  double h;
};

inline Agglo make_agglo(const Grid& g, int b, double h) {
  Agglo a;
  a.g = g;
  a.b = b;
  a.mx = (g.nx - 1) / b + 1;
  a.my = (g.ny - 1) / b + 1;
  a.mz = (g.nz - 1) / b + 1;
  a.nb = (long long)a.mx * a.my * a.mz;
  a.h = h;
  return a;
}

// Per-block deflation data (W is never stored):
//   cen[3B..3B+2]  centroid of the block's structural nodes, in grid units
//                  relative to the block's low corner
//   S[36B + i + 6j] column j of the basis = sum_i rawcol_i * S[i, j]
//                  (raw columns = masked rigid modes about the centroid,
//                   topovox/fea.py:141-155; S orthonormalises them like the
//                   per-block QR of topovox/fea.py:156-160, zero for dropped)
//   keep[B]        bit j set <=> column j kept (|R_jj| > 1e-10 max |R_ii|)
//   perm[B]        coarse-vector block position of block B (the ND order of
//                  the sparse coarse factor); nullptr = natural order
struct DeflData {
  double* cen;
  double* S;
  int* keep;
  const int* perm = nullptr;
};

cudaError_t launch_node_flags(const Grid& G, const long long* fixed_dofs, long long nfixed, const double* occ,
                              uint8_t* nflags, cudaStream_t s);
cudaError_t launch_block_basis(const Agglo& A, const double* occ, const uint8_t* nflags, DeflData D, cudaStream_t s);
// yc[6B + j] = (W^T y)_Bj, or (W^T (y + beta*y2))_Bj with beta from the solver state
cudaError_t launch_restrict(const Agglo& A, const uint8_t* nflags, DeflData D, const double* y, double* yc,
                            cudaStream_t s, const int* stop = nullptr, const double* y2 = nullptr,
                            const void* state = nullptr);
// nu[6B..] = S_B * mu_B  (rigid motion (t, omega) of each block)
cudaError_t launch_block_nu(const Agglo& A, DeflData D, const double* mu, double* nu, cudaStream_t s,
                            const int* stop = nullptr);
// mode 0: out = W nu ; mode 1: out(=p) = z + beta*p - W nu (beta/done from solver state) ; mode 2: out = z - W nu
// x (mode 1, optional): also x += alpha p_old (the solver's deferred x update;
// alpha from the solver state)
cudaError_t launch_prolong(const Agglo& A, const uint8_t* nflags, DeflData D, const double* nu, double* out,
                           const double* z, const void* state, int mode, cudaStream_t s, double* x = nullptr);
// coarse operator probing helpers
cudaError_t launch_probe_nu(const Agglo& A, DeflData D, int color, int j, double* nu, cudaStream_t s);
cudaError_t launch_probe_scatter(const Agglo& A, int color, int j, const double* yc, double* Eb, cudaStream_t s);
cudaError_t launch_coarse_finish(const Agglo& A, DeflData D, const double* Eb, double* Es, cudaStream_t s);
cudaError_t launch_coarse_dense(const Agglo& A, const double* Es, double* Ed, cudaStream_t s);

}  // namespace tvb
