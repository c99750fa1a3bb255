// K6: numeric factorisation of the nested-dissection coarse fronts
// (replaces scipy.linalg.cho_factor of E = W^T K W, topovox/fea.py:197-205).
#pragma once
#include "common.cuh"

namespace tvb {

constexpr int kFT = 64;  // tile order of the front factorisation

// One front (device record, int64 fields). The front matrix is row-major
// nf x nf at pool + a_off with the separator in [0, s_pad) and the update set
// in [s_pad, s_pad + u); padding rows / columns carry 1 on the separator
// diagonal and 0 elsewhere. Only tiles (I, J) with I >= J are maintained
// (diagonal tiles in full).
struct FrontRec {
  long long a_off;     // doubles
  long long nf;        // padded order (multiple of kFT)
  long long s, s_pad;  // separator DOFs / padded
  long long u;         // update DOFs
  long long blk_off;   // front blocks (natural ids, separator then update) at blocks + blk_off
  long long nchild, child_off;  // children records at children + 2 * child_off: (front index, gmap offset)
  long long scr_off;   // doubles: P tile, then CT[ntf], R[ntf] tiles
  long long ntf;       // nf / kFT
  long long pad_[2];
};

struct FrontLevel {
  int n_fronts;
  const int* fronts;        // front indices of the level
  int n_tiles;              // lower tiles (front, I, J) of the level's fronts
  const int* tiles;         // int32 triples
  int n_cols;               // (front, K) pairs for the panel kernel
  const int* cols;
  int max_steps;            // max s_pad / kFT over the level
};

struct FrontFactor {
  const FrontRec* fronts;   // device
  double* pool;             // device front storage
  double* scratch;          // device
  const int* blocks;        // device, natural block ids
  const long long* children;  // device (front, gmap offset) pairs
  const int* gmap;          // device: parent front position -> child update index or -1
  const double* Es;         // block stencil f64[nb][27][6][6]
  int mx, my, mz;           // block grid
  int* d_err;               // device int: nonzero = a pivot was not positive
};

cudaError_t launch_front_level(const FrontFactor& F, const FrontLevel& L, cudaStream_t s);

// pack a bottom front into the solver's layout: G (u x s) and B = [Z | -G^T] (s x (s + u))
cudaError_t launch_front_pack(const FrontFactor& F, int front, double* G, double* B, long long s_, long long u_,
                              cudaStream_t s);
// Z = -A of a top / dense front (order n): packed lower 64x64 tiles (tiles > 0) or dense rows
cudaError_t launch_front_pack_top(const FrontFactor& F, int front, long long n, int tiles, double* out,
                                  cudaStream_t s);

}  // namespace tvb
