#pragma once
#include "common.cuh"

namespace tvb {

struct MatvecParams {
  Grid g;
  const double* u;        // input node vector (3*Nn)
  double* y;              // output node vector (3*Nn)
  const double* occ;      // element scale (Ne)
  const uint8_t* fixed;   // node fixed-axis bits, or nullptr
  int mask_in;            // zero fixed DOFs of u on load
  int mask_out;           // zero fixed DOFs of y on store
  int accumulate;         // y += A u instead of y = A u
  int wx, wy;             // element columns per tile (incl. 1 halo column/row)
  int ntx;                // tiles along x
  int ntiles;             // ntx * nty
  int debug;              // tuning experiments only (TVB_MV_DEBUG)
  double* dot_partial;    // per-CTA partial of sum(u_owned * y_owned), or nullptr
  const int* stop;        // if non-null and *stop != 0 the launch is a no-op (solver done)
  int zlo = 0, zhi = -1;  // output node planes [zlo, zhi) (zhi < 0: all); reads input planes [zlo-1, zhi]
  int piece_cost = 0;     // per-piece overhead in plane-steps (halo layer + pipeline fill) charged by the work split
};

// nt threads per CTA, wx x wy element-column tiles (ntx x nty of them),
// nctas persistent CTAs each taking an equal share of the tile x plane work.
struct MatvecPlan {
  int nt, wx, wy, ntx, nty, nctas;
  size_t smem;
  int nblocks() const { return nctas; }
};

MatvecPlan plan_matvec(const Grid& g, int num_sms);
cudaError_t launch_matvec(const MatvecPlan& pl, MatvecParams P, const Modal& M, cudaStream_t s);

}  // namespace tvb
