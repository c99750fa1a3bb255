#pragma once
#include "common.cuh"

namespace tvb {

// Device view of the nested-dissection coarse factor (see coarse.py /
// tvb_coarse_nd in include/topovox_b200.h).
struct CoarseNDDev {
  int n_nodes, height, max_front;
  const long long* meta;      // [n_nodes][8]: s, u, g_off, z_off, sdof_off, udof_off, child_begin, child_end
  const long long* children;  // [n_child][2]: child node, cmap offset
  const int* cmap;            // child U position -> parent front position
  const double* G;            // per node u x s, row-major (G = F_US F_SS^-1)
  const double* Gt;           // per node s x u, row-major (G^T)
  const double* Z;            // per node s x s, row-major (F_SS^-1)
  const int* sdof;            // per node: separator coarse DOFs
  const int* udof;            // per node: update-set coarse DOFs
  double* fS;                 // per node scratch: assembled separator rhs
  double* cU;                 // per node scratch: update vector passed to the parent
  const int* fwd_items;       // [n][3] (node, row0, row1), grouped by height (leaves first)
  const int* bwd_items;       // [n][3], grouped by height (root first)
  const long long* fwd_ptr;   // host: height+2 group offsets
  const long long* bwd_ptr;   // host
  const int* split;           // host, per height: 1 = separate assembly pass (large fronts)
  const int* asm_nodes;       // device: nodes grouped by height (assembly pass)
  const long long* asm_ptr;   // host: height+2 offsets into asm_nodes
  int max_sep;                // largest separator (smem of the row pass)
};

cudaError_t launch_coarse_nd(const CoarseNDDev& D, const double* y, double* x, const int* stop, cudaStream_t s);

}  // namespace tvb
