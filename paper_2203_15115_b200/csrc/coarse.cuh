#pragma once
#include "common.cuh"

namespace tvb {

// Device view of the nested-dissection coarse factor (built by coarse.py; see
// tvb_coarse_nd in include/topovox_b200.h). Coarse vectors are in ND order.
struct CoarseNDDev {
  int n_levels;               // bottom tree heights 0..n_levels-1 (node-wise LDL^T)
  int max_front, max_sep;
  const long long* meta;      // [bottom node][8]: s, u, g_off, b_off, sd_off (ND dof), ud_off, gm_off, 0
  const int* gmap;            // per node [(s+u)][2]: children's cU index per front position (-1 = none)
  const double* G;            // per node u x s, row-major (G = F_US F_SS^-1)
  const double* B;            // per node s x (s+u), row-major: [F_SS^-1 | -G^T]
  const int* udof;            // per node: update-set coarse DOFs (ND numbering)
  double* fS;                 // ND-dof indexed scratch: assembled separator rhs
  double* cU;                 // per node scratch: update vector passed to the parent
  const long long* fwd_items; // [n][10] node meta row (7) + 0 + row0, row1; grouped by height (leaves first)
  const long long* bwd_items; // [n][10], grouped by height (top bottom level first)
  const long long* fwd_ptr;   // host: n_levels+1 group offsets
  const long long* bwd_ptr;   // host
  const int* fwd_wpr;         // host, per group: warps per matrix row (1, 2, 4, 8)
  const int* bwd_wpr;         // host
  const int* split;           // host, per height: 1 = separate assembly pass (large fronts)
  const int* asm_nodes;       // device: nodes grouped by height (assembly pass)
  const long long* asm_ptr;   // host
  // dense top (heights >= n_levels): x_T = S_T^-1 (y_T + children)
  int n_top;
  long long top_off;          // ND dof offset of the top set
  int top_wpr;
  const double* ZT;           // n_top x n_top
  double* fT;                 // scratch n_top
  const int* tptr;            // CSR over top positions: children's cU entries
  const int* tidx;
  const int* perm;            // natural block -> ND block (restriction / prolongation)
  // persistent dataflow schedule (k_coarse_flow); items == nullptr -> per-level launches
  const int* items;           // [n_items][12] type, wpr, node, r0, r1, wait_idx, wait_need, done_idx, done_need,
                              //               rel_begin, rel_end, 0   (topological order)
  int n_items;
  const int* rel;             // counters released by a node's last finishing item
  unsigned long long* cnt;    // dependency counters (epoch-scaled, never reset)
  unsigned long long* ctl;    // [3]: next item, CTAs exited, epoch
  // multi-RHS scratch: column c of fS / cU / fT at + c * fs_ld / cu_ld / ft_ld
  long long fs_ld, cu_ld, ft_ld;
  int max_cols;               // scratch columns allocated (>= 1)
  int top_smem;               // 1: stage the top vector in shared memory per CTA (TVB_TOP_SMEM=1, A/B only)
  // packed symmetric top (per-level schedule): ZT holds the lower 64x64 tiles
  // (I >= J, tile I*(I+1)/2 + J, row-major, zero-padded) instead of the dense
  // n_top^2 inverse; tpart: per-column [nt][nt][64] tile partial products
  int top_tiles;              // nt = ceil(n_top / 64); 0 = dense rows
  double* tpart;
  long long tpart_ld;
};

constexpr int kCoarseMaxCols = 4;  // right-hand sides per coarse-solve launch

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s);
// ncols right-hand sides (column c of y / x at + c * ldy / ldx); column c is
// skipped work-wise only when every column of its launch group is stopped
// (stop[c * stop_ld] != 0). Per-column results are bitwise those of
// launch_coarse_nd on that column alone.
cudaError_t launch_coarse_nd_multi(const CoarseNDDev& D, int ncols, const double* y, long long ldy, double* x,
                                   long long ldx, const int* stop, long long stop_ld, cudaStream_t s);
int coarse_nd_max_cols(const CoarseNDDev& D);

}  // namespace tvb
