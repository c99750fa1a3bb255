// extern "C" boundary of libtopovox_b200.so (declarations: include/topovox_b200.h).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>

#include "../../include/topovox_b200.h"
#include "coarse.cuh"
#include "dense.cuh"
#include "deflation.cuh"
#include "eigen.cuh"
#include "fields.cuh"
#include "matvec.cuh"
#include "solver.cuh"
#include "vec.cuh"

namespace tvb {

static thread_local std::string g_last_error;
void set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

#include "modal_entries.inc"

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

static int check(cudaError_t e) {
  if (e != cudaSuccess) {
    set_last_error(cudaGetErrorString(e));
    return kStatusCuda;
  }
  return kStatusOk;
}

static bool bad_dims(int nx, int ny, int nz) { return nx < 1 || ny < 1 || nz < 1; }

// Reduce the 45 mode-space entries (kModalEntries order) to the 8 structural
// constants of modal_apply8; false if the entries do not have the cube
// structure (then the caller's k0 was not an isotropic cube stiffness).
static bool modal_reduce(const double* mh, Modal& m) {
  // representative entries: (3,3) (3,7) (4,4) (9,9) (9,20) (11,11) (11,16) (21,21)
  static const int rep[8] = {0, 1, 3, 14, 15, 18, 19, 42};
  static const int cls[45] = {0, 1, 1, 2, 2, 2, 2, 2, 2, 1, 0, 1, 2, 2, 3, 4, 3, 4, 5, 6, 6, 2, 2,
                              2, 2, 1, 1, 0, 3, 4, 6, 5, 6, 4, 3, 6, 6, 5, 4, 3, 4, 3, 7, 7, 7};
  double v[8], mx = 0.0;
  for (int i = 0; i < 8; ++i) v[i] = mh[rep[i]];
  for (int t = 0; t < 45; ++t) mx = fmax(mx, fabs(mh[t]));
  for (int t = 0; t < 45; ++t)
    if (fabs(mh[t] - v[cls[t]]) > 1e-12 * mx) return false;
  m.k[0] = v[0] - v[1];
  m.k[1] = v[1];
  m.k[2] = v[2];
  m.k[3] = v[3];
  m.k[4] = v[4];
  m.k[5] = v[5] - v[6];
  m.k[6] = v[6];
  m.k[7] = v[7];
  return true;
}



// fp64 pipe probe: 8 independent DFMA chains per thread, 8 CTAs of 256 per SM
__global__ void k_fp64_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_sum_partials(const double* partials, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_subset_scale(const long long* elems, long long m, long long ne, int* counts) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const long long e = elems[i];
  if (e >= 0 && e < ne) atomicAdd(counts + e, 1);
}

__global__ void k_subset_occ(long long ne, const int* counts, const double* occ, double* out) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  out[e] = counts[e] ? (double)counts[e] * occ[e] : 0.0;
}

static CoarseNDDev coarse_nd_dev(const tvb_coarse_nd* d) {
  CoarseNDDev D;
  D.n_levels = d->n_levels;
  D.max_front = d->max_front;
  D.max_sep = d->max_sep;
  D.meta = d->d_meta;
  D.gmap = d->d_gmap;
  D.G = d->d_G;
  D.B = d->d_B;
  D.udof = d->d_udof;
  D.fS = d->d_fS;
  D.cU = d->d_cU;
  D.fwd_items = d->d_fwd_items;
  D.bwd_items = d->d_bwd_items;
  D.fwd_ptr = d->h_fwd_ptr;
  D.bwd_ptr = d->h_bwd_ptr;
  D.fwd_wpr = d->h_fwd_wpr;
  D.bwd_wpr = d->h_bwd_wpr;
  D.split = d->h_split;
  D.asm_nodes = d->d_asm_nodes;
  D.asm_ptr = d->h_asm_ptr;
  D.n_top = d->n_top;
  D.top_off = d->top_off;
  D.top_wpr = d->top_wpr;
  D.ZT = d->d_ZT;
  D.fT = d->d_fT;
  D.tptr = d->d_tptr;
  D.tidx = d->d_tidx;
  D.perm = d->d_perm;
  D.items = d->d_items;
  D.n_items = d->n_items;
  D.rel = d->d_rel;
  D.cnt = d->d_cnt;
  D.ctl = d->d_ctl;
  D.fs_ld = d->fs_ld;
  D.cu_ld = d->cu_ld;
  D.ft_ld = d->ft_ld;
  D.max_cols = d->max_cols > 0 ? d->max_cols : 1;
  D.top_smem = getenv("TVB_TOP_SMEM") ? atoi(getenv("TVB_TOP_SMEM")) : 0;
  D.top_tiles = (d->d_items == nullptr || d->n_items <= 0) ? d->top_tiles : 0;
  D.tpart = d->d_tpart;
  D.tpart_ld = d->tpart_ld;
  return D;
}

}  // namespace tvb

using namespace tvb;

extern "C" {

int tvb_version(void) { return 1; }

const char* tvb_last_error(void) { return g_last_error.c_str(); }

int tvb_modal_from_k0(const double* k0, double* mh45) {
  // VTK local node -> binary index (ox + 2 oy + 4 oz)
  static const int vtk_bin[8] = {0, 1, 3, 2, 4, 5, 7, 6};
  double kb[24][24];
  for (int n = 0; n < 8; ++n)
    for (int a = 0; a < 3; ++a)
      for (int m = 0; m < 8; ++m)
        for (int c = 0; c < 3; ++c) kb[3 * vtk_bin[n] + a][3 * vtk_bin[m] + c] = k0[(3 * n + a) * 24 + 3 * m + c];
  double H[8][8];
  for (int b = 0; b < 8; ++b)
    for (int m = 0; m < 8; ++m) {
      double v = 1.0;
      for (int ax = 0; ax < 3; ++ax)
        if ((m >> ax) & 1) v *= ((b >> ax) & 1) ? 1.0 : -1.0;
      H[b][m] = v;
    }
  // Mh = H3^T kb H3 / 64
  double T[24][24], M[24][24];
  for (int i = 0; i < 24; ++i)
    for (int mj = 0; mj < 24; ++mj) {
      double s = 0.0;
      const int m = mj / 3, c = mj % 3;
      for (int b = 0; b < 8; ++b) s += kb[i][3 * b + c] * H[b][m];
      T[i][mj] = s;
    }
  double mx = 0.0;
  for (int mi = 0; mi < 24; ++mi)
    for (int mj = 0; mj < 24; ++mj) {
      double s = 0.0;
      const int m = mi / 3, a = mi % 3;
      for (int b = 0; b < 8; ++b) s += H[b][m] * T[3 * b + a][mj];
      M[mi][mj] = s / 64.0;
      mx = fmax(mx, fabs(M[mi][mj]));
    }
  bool on[24][24] = {};
  for (int t = 0; t < 45; ++t) {
    on[kModalEntries[t][0]][kModalEntries[t][1]] = true;
    mh45[t] = M[kModalEntries[t][0]][kModalEntries[t][1]];
  }
  for (int i = 0; i < 24; ++i)
    for (int j = 0; j < 24; ++j)
      if (!on[i][j] && fabs(M[i][j]) > 1e-13 * fmax(mx, 1e-300)) {
        set_last_error("k0 is not the stiffness of an isotropic cube (mode pattern violated)");
        return kStatusBadArg;
      }
  Modal probe;
  if (!modal_reduce(mh45, probe)) {
    set_last_error("k0 is not the stiffness of an isotropic cube (mode values violate the cube symmetry)");
    return kStatusBadArg;
  }
  return kStatusOk;
}

// workspace: per-CTA dot partials (65536 max) + a masked copy of u (MASK_IN)
static size_t matvec_partials_bytes() { return sizeof(double) * 65536; }

size_t tvb_matvec_ws_bytes(int nx, int ny, int nz) {
  if (bad_dims(nx, ny, nz)) return 0;
  return matvec_partials_bytes() + sizeof(double) * 3 * (size_t)make_grid(nx, ny, nz).nn;
}

int tvb_matvec(int nx, int ny, int nz, const double* h_mh45, const double* d_u, double* d_out, const double* d_occ,
               const uint8_t* d_nflags, int flags, double* d_dot, void* d_ws, size_t ws_bytes, void* stream) {
  if (bad_dims(nx, ny, nz) || !h_mh45 || !d_u || !d_out || !d_occ) return kStatusBadArg;
  if ((flags & (TVB_MASK_IN | TVB_MASK_OUT)) && !d_nflags) return kStatusBadArg;
  const Grid g = make_grid(nx, ny, nz);
  const MatvecPlan pl = plan_matvec(g, num_sms());
  const bool mask_in = (flags & TVB_MASK_IN) != 0;
  if (d_dot && (!d_ws || ws_bytes < tvb_matvec_ws_bytes(nx, ny, nz) || pl.nblocks() > 65536)) {
    set_last_error("matvec workspace too small");
    return kStatusWorkspace;
  }
  Modal M;
  if (!modal_reduce(h_mh45, M)) return kStatusBadArg;
  cudaStream_t s = (cudaStream_t)stream;
  MatvecParams P{};
  P.g = g;
  P.u = d_u;
  P.y = d_out;
  P.occ = d_occ;
  P.fixed = d_nflags;
  P.mask_in = mask_in ? 1 : 0;  // fused into the staging (matvec.cu MASKIN)
  P.mask_out = (flags & TVB_MASK_OUT) ? 1 : 0;
  P.accumulate = (flags & TVB_ACCUMULATE) ? 1 : 0;
  P.dot_partial = d_dot ? (double*)d_ws : nullptr;
  P.stop = nullptr;
  int st = check(launch_matvec(pl, P, M, s));
  if (st || !d_dot) return st;
  k_sum_partials<<<1, 256, 0, s>>>((const double*)d_ws, pl.nblocks(), d_dot);
  return check(cudaGetLastError());
}

size_t tvb_matvec_host_ws_bytes(int nx, int ny, int nz) {
  if (bad_dims(nx, ny, nz)) return 0;
  return 2 * sizeof(double) * 3 * (size_t)make_grid(nx, ny, nz).nn + 256;
}

// Host-buffer K.u, pipelined over z-slabs of node planes: slab k's input
// planes go host->device on one copy stream while slab k-1 is multiplied and
// slab k-2's output planes go device->host on a second copy stream (the two
// copy engines run concurrently), so a step costs about max(H2D, D2H) instead
// of H2D + K.u + D2H. Node planes are contiguous in the reference numbering
// (z slowest), so every slab copy is one contiguous range. Synchronous.
int tvb_matvec_host(int nx, int ny, int nz, const double* h_mh45, const double* h_u, double* h_out,
                    const double* d_occ, const uint8_t* d_nflags, int flags, int slabs, void* d_ws, size_t ws_bytes,
                    void* stream) {
  if (bad_dims(nx, ny, nz) || !h_mh45 || !h_u || !h_out || !d_occ || !d_ws) return kStatusBadArg;
  if ((flags & (TVB_MASK_IN | TVB_MASK_OUT)) && !d_nflags) return kStatusBadArg;
  if (flags & TVB_ACCUMULATE) {
    set_last_error("tvb_matvec_host: ACCUMULATE is not supported for host buffers");
    return kStatusBadArg;
  }
  if (ws_bytes < tvb_matvec_host_ws_bytes(nx, ny, nz)) {
    set_last_error("matvec workspace too small");
    return kStatusWorkspace;
  }
  Modal M;
  if (!modal_reduce(h_mh45, M)) return kStatusBadArg;
  const Grid g = make_grid(nx, ny, nz);
  const MatvecPlan pl = plan_matvec(g, num_sms());
  const size_t pdoubles = 3 * (size_t)g.px * g.py;  // doubles per node plane
  double* du = (double*)(((uintptr_t)d_ws + 255) & ~(uintptr_t)255);
  double* dy = du + 3 * (size_t)g.nn;
  cudaStream_t s = (cudaStream_t)stream;
  // default 6 slabs: measured best at 128^3 (4-8 within noise; 1 slab = no overlap, 1.31x slower)
  const int K = std::max(1, std::min(slabs > 0 ? slabs : 6, g.pz / 2));

  struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;
    cudaEvent_t start = nullptr, in[64], done[64], end = nullptr;
  };
  static thread_local Pipe P;
  if (P.h2d == nullptr) {
    cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&P.end, cudaEventDisableTiming);
    for (int k = 0; k < 64; ++k) {
      cudaEventCreateWithFlags(&P.in[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.done[k], cudaEventDisableTiming);
    }
  }
  const int KK = std::min(K, 64);
  // the copy streams start after the work already queued on the caller's stream
  cudaEventRecord(P.start, s);
  cudaStreamWaitEvent(P.h2d, P.start, 0);
  cudaStreamWaitEvent(P.d2h, P.start, 0);
  cudaStreamWaitEvent(P.comp, P.start, 0);
  int loaded = 0;  // input planes [0, loaded) issued
  for (int k = 0; k < KK; ++k) {
    const int z0 = (int)((long long)g.pz * k / KK), z1 = (int)((long long)g.pz * (k + 1) / KK);
    const int need = std::min(g.pz, z1 + 1);  // output planes [z0, z1) read input planes up to z1
    if (need > loaded) {
      cudaMemcpyAsync(du + pdoubles * loaded, h_u + pdoubles * loaded, sizeof(double) * pdoubles * (need - loaded),
                      cudaMemcpyHostToDevice, P.h2d);
      loaded = need;
    }
    cudaEventRecord(P.in[k], P.h2d);
    cudaStreamWaitEvent(P.comp, P.in[k], 0);
    MatvecParams mp{};
    mp.g = g;
    mp.u = du;
    mp.y = dy;
    mp.occ = d_occ;
    mp.fixed = d_nflags;
    mp.mask_in = (flags & TVB_MASK_IN) ? 1 : 0;
    mp.mask_out = (flags & TVB_MASK_OUT) ? 1 : 0;
    mp.zlo = z0;
    mp.zhi = z1;
    const int st = check(launch_matvec(pl, mp, M, P.comp));
    if (st) return st;
    cudaEventRecord(P.done[k], P.comp);
    cudaStreamWaitEvent(P.d2h, P.done[k], 0);
    cudaMemcpyAsync(h_out + pdoubles * z0, dy + pdoubles * z0, sizeof(double) * pdoubles * (z1 - z0),
                    cudaMemcpyDeviceToHost, P.d2h);
  }
  cudaEventRecord(P.end, P.d2h);
  cudaStreamWaitEvent(s, P.end, 0);
  return check(cudaStreamSynchronize(s));
}

size_t tvb_matvec_host_batch_ws_bytes(int nx, int ny, int nz) {
  if (bad_dims(nx, ny, nz)) return 0;
  return 4 * sizeof(double) * 3 * (size_t)make_grid(nx, ny, nz).nn + 256;
}

// Host-buffer K.u for a stream of nvec vectors (e.g. every load vector of a
// topology): the single-vector z-slab pipeline of tvb_matvec_host, with two
// device input and two device output buffers used alternately so that vector
// v's host->device copies overlap vector v-1's device->host copies (the two
// copy engines) -- a steady state of max(H2D, D2H) per vector instead of
// H2D + D2H of one synchronous call. Cross-vector dependencies: the copies
// into input buffer v%2 wait for the multiply of vector v-2 to finish
// reading it; the multiply of vector v waits for the read-back of vector v-2
// out of output buffer v%2. Synchronous; results bitwise those of
// tvb_matvec_host / tvb_matvec.
int tvb_matvec_host_batch(int nx, int ny, int nz, const double* h_mh45, int nvec, const double* const* h_u,
                          double* const* h_out, const double* d_occ, const uint8_t* d_nflags, int flags, int slabs,
                          void* d_ws, size_t ws_bytes, void* stream) {
  if (bad_dims(nx, ny, nz) || !h_mh45 || nvec < 0 || (nvec > 0 && (!h_u || !h_out)) || !d_occ || !d_ws)
    return kStatusBadArg;
  if ((flags & (TVB_MASK_IN | TVB_MASK_OUT)) && !d_nflags) return kStatusBadArg;
  if (flags & TVB_ACCUMULATE) {
    set_last_error("tvb_matvec_host_batch: ACCUMULATE is not supported for host buffers");
    return kStatusBadArg;
  }
  if (ws_bytes < tvb_matvec_host_batch_ws_bytes(nx, ny, nz)) {
    set_last_error("matvec workspace too small");
    return kStatusWorkspace;
  }
  for (int v = 0; v < nvec; ++v)
    if (!h_u[v] || !h_out[v]) return kStatusBadArg;
  if (nvec == 0) return kStatusOk;
  Modal M;
  if (!modal_reduce(h_mh45, M)) return kStatusBadArg;
  const Grid g = make_grid(nx, ny, nz);
  const MatvecPlan pl = plan_matvec(g, num_sms());
  const size_t pdoubles = 3 * (size_t)g.px * g.py;
  const size_t nd = 3 * (size_t)g.nn;
  double* base = (double*)(((uintptr_t)d_ws + 255) & ~(uintptr_t)255);
  double* du[2] = {base, base + nd};
  double* dy[2] = {base + 2 * nd, base + 3 * nd};
  cudaStream_t s = (cudaStream_t)stream;
  // default: whole vectors once the stream has >= 3 of them (the overlap is
  // then across vectors; measured at 128^3: 1 slab 1.10 ms/vector = the raw
  // concurrent H2D + D2H copy rate, 6 slabs 1.32 ms), else the 6-slab split
  const int K = std::max(1, std::min(std::min(slabs > 0 ? slabs : (nvec >= 3 ? 1 : 6), g.pz / 2), 64));

  struct Pipe {
    cudaStream_t h2d = nullptr, d2h = nullptr, comp = nullptr;
    cudaEvent_t start = nullptr, end = nullptr, in[64], done[64], comp_done[2], d2h_done[2];
  };
  static thread_local Pipe P;
  if (P.h2d == nullptr) {
    cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&P.comp, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&P.end, cudaEventDisableTiming);
    for (int k = 0; k < 64; ++k) {
      cudaEventCreateWithFlags(&P.in[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.done[k], cudaEventDisableTiming);
    }
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&P.comp_done[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&P.d2h_done[b], cudaEventDisableTiming);
    }
  }
  cudaEventRecord(P.start, s);
  cudaStreamWaitEvent(P.h2d, P.start, 0);
  cudaStreamWaitEvent(P.d2h, P.start, 0);
  cudaStreamWaitEvent(P.comp, P.start, 0);
  for (int v = 0; v < nvec; ++v) {
    const int b = v & 1;
    if (v >= 2) {
      cudaStreamWaitEvent(P.h2d, P.comp_done[b], 0);  // vector v-2 no longer reads du[b]
      cudaStreamWaitEvent(P.comp, P.d2h_done[b], 0);  // vector v-2 read back out of dy[b]
    }
    int loaded = 0;
    for (int k = 0; k < K; ++k) {
      const int z0 = (int)((long long)g.pz * k / K), z1 = (int)((long long)g.pz * (k + 1) / K);
      const int need = std::min(g.pz, z1 + 1);
      if (need > loaded) {
        cudaMemcpyAsync(du[b] + pdoubles * loaded, h_u[v] + pdoubles * loaded,
                        sizeof(double) * pdoubles * (need - loaded), cudaMemcpyHostToDevice, P.h2d);
        loaded = need;
      }
      cudaEventRecord(P.in[k], P.h2d);
      cudaStreamWaitEvent(P.comp, P.in[k], 0);
      MatvecParams mp{};
      mp.g = g;
      mp.u = du[b];
      mp.y = dy[b];
      mp.occ = d_occ;
      mp.fixed = d_nflags;
      mp.mask_in = (flags & TVB_MASK_IN) ? 1 : 0;
      mp.mask_out = (flags & TVB_MASK_OUT) ? 1 : 0;
      mp.zlo = z0;
      mp.zhi = z1;
      const int st = check(launch_matvec(pl, mp, M, P.comp));
      if (st) return st;
      cudaEventRecord(P.done[k], P.comp);
      cudaStreamWaitEvent(P.d2h, P.done[k], 0);
      cudaMemcpyAsync(h_out[v] + pdoubles * z0, dy[b] + pdoubles * z0, sizeof(double) * pdoubles * (z1 - z0),
                      cudaMemcpyDeviceToHost, P.d2h);
    }
    cudaEventRecord(P.comp_done[b], P.comp);
    cudaEventRecord(P.d2h_done[b], P.d2h);
  }
  cudaEventRecord(P.end, P.d2h);
  cudaStreamWaitEvent(s, P.end, 0);
  return check(cudaStreamSynchronize(s));
}

double tvb_fp64_peak_tflops(void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return 0.0;
  const dim3 grid(num_sms() * 8), block(256);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64_probe<<<grid, block, 0, s>>>(sink, 64, 1.0000001, 1e-9);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s);
    k_fp64_probe<<<grid, block, 0, s>>>(sink, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 0.f && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const double fmas = (double)grid.x * block.x * iters * 8.0;
  return 2.0 * fmas / (best * 1e-3) / 1e12;
}

int tvb_matvec_plan(int nx, int ny, int nz, int* out7) {
  if (bad_dims(nx, ny, nz) || !out7) return kStatusBadArg;
  const MatvecPlan pl = plan_matvec(make_grid(nx, ny, nz), num_sms());
  const int v[7] = {pl.nt, pl.wx, pl.wy, pl.ntx, pl.nty, pl.nctas, 0};
  for (int i = 0; i < 7; ++i) out7[i] = v[i];
  return kStatusOk;
}

int tvb_matvec_subset(int nx, int ny, int nz, const double* h_mh45, const double* d_u, double* d_out,
                      const long long* d_elems, long long n_listed, const double* d_occ, void* d_ws, size_t ws_bytes,
                      void* stream) {
  if (bad_dims(nx, ny, nz) || !h_mh45 || !d_u || !d_out || !d_occ || !d_ws) return kStatusBadArg;
  const Grid g = make_grid(nx, ny, nz);
  const size_t need = (size_t)g.ne * (sizeof(double) + sizeof(int));
  if (ws_bytes < need) {
    set_last_error("subset workspace too small");
    return kStatusWorkspace;
  }
  cudaStream_t s = (cudaStream_t)stream;
  double* occ_sub = (double*)d_ws;
  int* counts = (int*)(occ_sub + g.ne);
  if (int st = check(cudaMemsetAsync(counts, 0, g.ne * sizeof(int), s))) return st;
  if (n_listed > 0)
    k_subset_scale<<<(unsigned)((n_listed + 255) / 256), 256, 0, s>>>(d_elems, n_listed, g.ne, counts);
  k_subset_occ<<<(unsigned)((g.ne + 255) / 256), 256, 0, s>>>(g.ne, counts, d_occ, occ_sub);
  if (int st = check(cudaGetLastError())) return st;
  return tvb_matvec(nx, ny, nz, h_mh45, d_u, d_out, occ_sub, nullptr, TVB_ACCUMULATE, nullptr, nullptr, 0, stream);
}

int tvb_diag(int nx, int ny, int nz, const double* d_occ, const uint8_t* d_nflags, const double* h_kdiag3,
             double* d_diag, int accumulate, double* d_inv, int* d_zero_free, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_occ || !h_kdiag3) return kStatusBadArg;
  const Grid g = make_grid(nx, ny, nz);
  return check(launch_inv_diag(g, d_occ, d_nflags, h_kdiag3, d_inv, d_diag, d_zero_free, (cudaStream_t)stream,
                               accumulate));
}

int tvb_node_flags(int nx, int ny, int nz, const long long* d_fixed_dofs, long long n_fixed, const double* d_occ,
                   uint8_t* d_nflags, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_occ || !d_nflags || (n_fixed > 0 && !d_fixed_dofs)) return kStatusBadArg;
  return check(launch_node_flags(make_grid(nx, ny, nz), d_fixed_dofs, n_fixed, d_occ, d_nflags, (cudaStream_t)stream));
}

size_t tvb_reduce_ws_bytes(long long n) { return sizeof(double) * (size_t)(reduce_grid(n) + 8); }

int tvb_dot(const double* d_a, const double* d_b, const double* d_w, long long n, double* d_out, void* d_ws,
            size_t ws_bytes, void* stream) {
  if (!d_a || !d_b || !d_out || !d_ws || n < 0) return kStatusBadArg;
  if (ws_bytes < tvb_reduce_ws_bytes(n)) return kStatusWorkspace;
  double* partials = (double*)d_ws;
  unsigned int* counter = (unsigned int*)(partials + reduce_grid(n) + 4);
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check(cudaMemsetAsync(counter, 0, sizeof(unsigned int), s))) return st;
  return check(launch_dot(d_a, d_b, d_w, n, partials, counter, d_out, s));
}

int tvb_defl_build(int nx, int ny, int nz, int block, double h, const double* d_occ, const uint8_t* d_nflags,
                   double* d_cen, double* d_S, int* d_keep, void* stream) {
  if (bad_dims(nx, ny, nz) || block < 2 || !(h > 0.0)) return kStatusBadArg;
  const Agglo A = make_agglo(make_grid(nx, ny, nz), block, h);
  return check(launch_block_basis(A, d_occ, d_nflags, DeflData{d_cen, d_S, d_keep}, (cudaStream_t)stream));
}

int tvb_restrict(int nx, int ny, int nz, int block, double h, const uint8_t* d_nflags, const double* d_cen,
                 const double* d_S, const int* d_keep, const double* d_y, double* d_yc, void* stream) {
  if (bad_dims(nx, ny, nz) || block < 2) return kStatusBadArg;
  const Agglo A = make_agglo(make_grid(nx, ny, nz), block, h);
  DeflData D{const_cast<double*>(d_cen), const_cast<double*>(d_S), const_cast<int*>(d_keep)};
  return check(launch_restrict(A, d_nflags, D, d_y, d_yc, (cudaStream_t)stream));
}

int tvb_prolong(int nx, int ny, int nz, int block, double h, const uint8_t* d_nflags, const double* d_cen,
                const double* d_S, const int* d_keep, const double* d_mu, double* d_out, double* d_nu_ws,
                void* stream) {
  if (bad_dims(nx, ny, nz) || block < 2 || !d_nu_ws) return kStatusBadArg;
  const Agglo A = make_agglo(make_grid(nx, ny, nz), block, h);
  DeflData D{const_cast<double*>(d_cen), const_cast<double*>(d_S), const_cast<int*>(d_keep)};
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check(launch_block_nu(A, D, d_mu, d_nu_ws, s))) return st;
  return check(launch_prolong(A, d_nflags, D, d_nu_ws, d_out, nullptr, nullptr, 0, s));
}

size_t tvb_coarse_assemble_ws_bytes(int nx, int ny, int nz, int block) {
  if (bad_dims(nx, ny, nz) || block < 2) return 0;
  const Grid g = make_grid(nx, ny, nz);
  const Agglo A = make_agglo(g, block, 1.0);
  return sizeof(double) * (2 * 3 * (size_t)g.nn + 2 * 6 * (size_t)A.nb + (size_t)A.nb * 27 * 36) + 1024;
}

int tvb_coarse_assemble(int nx, int ny, int nz, int block, double h, const double* h_mh45, const double* d_occ,
                        const uint8_t* d_nflags, const double* d_cen, const double* d_S, const int* d_keep,
                        double* d_Es, void* d_ws, size_t ws_bytes, void* stream) {
  if (bad_dims(nx, ny, nz) || block < 2 || !h_mh45) return kStatusBadArg;
  if (ws_bytes < tvb_coarse_assemble_ws_bytes(nx, ny, nz, block)) return kStatusWorkspace;
  const Grid g = make_grid(nx, ny, nz);
  const Agglo A = make_agglo(g, block, h);
  DeflData D{const_cast<double*>(d_cen), const_cast<double*>(d_S), const_cast<int*>(d_keep)};
  cudaStream_t s = (cudaStream_t)stream;
  double* v = (double*)d_ws;
  double* t = v + 3 * g.nn;
  double* nu = t + 3 * g.nn;
  double* yc = nu + 6 * A.nb;
  double* Eb = yc + 6 * A.nb;
  const MatvecPlan pl = plan_matvec(g, num_sms());
  Modal M;
  if (!modal_reduce(h_mh45, M)) return kStatusBadArg;
  if (int st = check(cudaMemsetAsync(Eb, 0, sizeof(double) * A.nb * 27 * 36, s))) return st;
  for (int color = 0; color < 27; ++color) {
    for (int j = 0; j < 6; ++j) {
      if (int st = check(launch_probe_nu(A, D, color, j, nu, s))) return st;
      if (int st = check(launch_prolong(A, d_nflags, D, nu, v, nullptr, nullptr, 0, s))) return st;
      MatvecParams P{};
      P.g = g;
      P.u = v;
      P.y = t;
      P.occ = d_occ;
      P.fixed = d_nflags;
      if (int st = check(launch_matvec(pl, P, M, s))) return st;
      if (int st = check(launch_restrict(A, d_nflags, D, t, yc, s))) return st;
      if (int st = check(launch_probe_scatter(A, color, j, yc, Eb, s))) return st;
    }
  }
  return check(launch_coarse_finish(A, D, Eb, d_Es, s));
}

int tvb_coarse_dense(int nx, int ny, int nz, int block, const double* d_Es, double* d_E, void* stream) {
  if (bad_dims(nx, ny, nz) || block < 2) return kStatusBadArg;
  const Agglo A = make_agglo(make_grid(nx, ny, nz), block, 1.0);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t nc = 6 * (size_t)A.nb;
  if (int st = check(cudaMemsetAsync(d_E, 0, sizeof(double) * nc * nc, s))) return st;
  return check(launch_coarse_dense(A, d_Es, d_E, s));
}

size_t tvb_pcg_ws_bytes(int nx, int ny, int nz, int block) {
  if (bad_dims(nx, ny, nz)) return 0;
  return pcg_ws_bytes(make_grid(nx, ny, nz), block);
}

static int pcg_problem(const tvb_pcg_desc* d, PcgProblem& P) {
  if (!d || bad_dims(d->nx, d->ny, d->nz) || !d->h_mh45 || !d->h_kdiag3 || !d->d_occ || !d->d_nflags || !d->d_ws)
    return kStatusBadArg;
  if (!(d->tol > 0.0) || d->max_iters < 1) return kStatusBadArg;
  P.g = make_grid(d->nx, d->ny, d->nz);
  P.h = d->h;
  if (!modal_reduce(d->h_mh45, P.modal)) return kStatusBadArg;
  for (int a = 0; a < 3; ++a) P.kdiag[a] = d->h_kdiag3[a];
  P.occ = d->d_occ;
  P.nflags = d->d_nflags;
  P.f = d->d_f;
  P.x = d->d_x;
  P.ws = d->d_ws;
  P.ws_bytes = d->ws_bytes;
  P.tol = d->tol;
  P.max_iters = d->max_iters;
  P.check_every = d->check_every;
  P.block = (d->d_coarse != nullptr || d->coarse_nd != nullptr) ? d->block : 0;
  P.cen = d->d_cen;
  P.S = d->d_S;
  P.keep = d->d_keep;
  P.coarse = d->d_coarse;
  P.coarse_kind = d->coarse_kind;
  if (d->projection != 0 && d->projection != 1) return kStatusBadArg;
  P.stabilized = d->projection == 1;
  P.dflags = d->d_defl_nflags ? d->d_defl_nflags : d->d_nflags;
  if (P.coarse_kind == 1) {
    if (!d->coarse_nd) return kStatusBadArg;
    P.nd = coarse_nd_dev(d->coarse_nd);
    P.nd_factor = d->coarse_nd->d_factor;
    P.nd_factor_bytes = d->coarse_nd->factor_bytes;
  }
  if (P.block > 0 && (!P.cen || !P.S || !P.keep)) return kStatusBadArg;
  return kStatusOk;
}

int tvb_pcg_solve(tvb_pcg_desc* d, void* stream) {
  PcgProblem P{};
  if (!d || !d->d_f || !d->d_x) return kStatusBadArg;
  if (int st = pcg_problem(d, P)) return st;
  PcgResult R;
  const int st = pcg_solve(P, R, (cudaStream_t)stream);
  d->iterations = R.iterations;
  d->residual = R.residual;
  d->fnorm = R.fnorm;
  return st;
}

size_t tvb_pcg_batch_ws_bytes(int nx, int ny, int nz, int block, int nrhs) {
  if (bad_dims(nx, ny, nz) || nrhs < 1 || nrhs > kPcgMaxRhs) return 0;
  return (size_t)nrhs * pcg_ws_bytes(make_grid(nx, ny, nz), block);
}

int tvb_pcg_solve_batch(tvb_pcg_desc* d, int nrhs, const double* const* h_d_f, double* const* h_d_x,
                        int* h_iterations, double* h_residuals, int* h_status, void* stream) {
  if (nrhs < 1 || nrhs > kPcgMaxRhs) return kStatusBadArg;
  // every return path reports a per-RHS status: a failure of the whole call
  // (arguments, problem, workspace, CUDA / graph) is never left as "ok"
  auto fail_all = [&](int st) {
    for (int c = 0; c < nrhs; ++c) {
      if (h_iterations) h_iterations[c] = 0;
      if (h_residuals) h_residuals[c] = 0.0;
      if (h_status) h_status[c] = st;
    }
    return st;
  };
  if (!h_d_f || !h_d_x) return fail_all(kStatusBadArg);
  PcgProblem P{};
  if (int st = pcg_problem(d, P)) return fail_all(st);
  P.nrhs = nrhs;
  for (int c = 0; c < nrhs; ++c) {
    if (!h_d_f[c] || !h_d_x[c]) return fail_all(kStatusBadArg);
    P.fs[c] = h_d_f[c];
    P.xs[c] = h_d_x[c];
  }
  PcgResult R[kPcgMaxRhs] = {};
  int rs[kPcgMaxRhs];
  for (int c = 0; c < nrhs; ++c) rs[c] = -1;  // not reached by the solver
  const int st = pcg_solve_multi(P, R, rs, (cudaStream_t)stream);
  const bool call_failed = st != kStatusOk && st != kStatusNoConvergence;
  for (int c = 0; c < nrhs; ++c) {
    int sc = rs[c];
    if (sc == -1 || (call_failed && sc == kStatusOk)) sc = call_failed ? st : kStatusCuda;
    if (h_iterations) h_iterations[c] = R[c].iterations;
    if (h_residuals) h_residuals[c] = R[c].residual;
    if (h_status) h_status[c] = sc;
  }
  return st;
}

static_assert(sizeof(FrontRec) == 12 * sizeof(long long), "front record layout");

static bool front_set(const tvb_front_set* fs, FrontFactor& F) {
  if (!fs || !fs->d_fronts || !fs->d_pool || !fs->d_blocks || !fs->d_Es || !fs->d_err || fs->mx < 1 || fs->my < 1 ||
      fs->mz < 1)
    return false;
  F.fronts = (const FrontRec*)fs->d_fronts;
  F.pool = fs->d_pool;
  F.scratch = fs->d_scratch;
  F.blocks = fs->d_blocks;
  F.children = fs->d_children;
  F.gmap = fs->d_gmap;
  F.Es = fs->d_Es;
  F.mx = fs->mx;
  F.my = fs->my;
  F.mz = fs->mz;
  F.d_err = fs->d_err;
  return true;
}

int tvb_front_level(const tvb_front_set* fs, int n_fronts, const int* d_level_fronts, int n_tiles,
                    const int* d_tiles, int n_cols, const int* d_cols, int max_steps, void* stream) {
  FrontFactor F;
  if (!front_set(fs, F) || n_fronts < 1 || !d_level_fronts || n_tiles < 1 || !d_tiles || n_cols < 1 || !d_cols ||
      max_steps < 0 || !fs->d_scratch)
    return kStatusBadArg;
  FrontLevel L{n_fronts, d_level_fronts, n_tiles, d_tiles, n_cols, d_cols, max_steps};
  return check(launch_front_level(F, L, (cudaStream_t)stream));
}

int tvb_front_pack(const tvb_front_set* fs, int front, double* d_G, double* d_B, long long s, long long u,
                   void* stream) {
  FrontFactor F;
  if (!front_set(fs, F) || front < 0 || !d_B || (u > 0 && !d_G) || s < 1 || u < 0) return kStatusBadArg;
  return check(launch_front_pack(F, front, d_G, d_B, s, u, (cudaStream_t)stream));
}

int tvb_front_pack_top(const tvb_front_set* fs, int front, long long n, int tiles, double* d_out, void* stream) {
  FrontFactor F;
  if (!front_set(fs, F) || front < 0 || n < 1 || tiles < 0 || !d_out) return kStatusBadArg;
  return check(launch_front_pack_top(F, front, n, tiles, d_out, (cudaStream_t)stream));
}

int tvb_coarse_nd_solve(const tvb_coarse_nd* nd, const double* d_y, double* d_x, void* stream) {
  if (!nd || !d_y || !d_x) return kStatusBadArg;
  return check(launch_coarse_nd(coarse_nd_dev(nd), d_y, d_x, nullptr, (cudaStream_t)stream));
}

static Elastic elastic(double E, double nu) {
  const double c = E / ((1.0 + nu) * (1.0 - 2.0 * nu));
  Elastic D;
  D.d0 = c * (1.0 - nu);
  D.d1 = c * nu;
  D.d2 = c * (1.0 - 2.0 * nu) / 2.0;
  D.c1 = 4.0 / (1.0 + nu);
  D.c2 = (1.0 - 3.0 * nu) / (1.0 - nu * nu);
  return D;
}

static ElemArgs elem_args(int nx, int ny, int nz, double h, double E, double nu, const double* u, const double* occ) {
  ElemArgs A{};
  A.g = make_grid(nx, ny, nz);
  A.D = elastic(E, nu);
  A.inv4h = 1.0 / (4.0 * h);
  A.u = u;
  A.occ = occ;
  return A;
}

size_t tvb_elem_ws_bytes(int nx, int ny, int nz) {
  if (bad_dims(nx, ny, nz)) return 0;
  const long long ne = (long long)nx * ny * nz;
  return sizeof(double) * (2 * (size_t)elem_grid(ne) + 8);
}

int tvb_element_state(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                      double* d_strains, double* d_stresses, double* d_vm, double* d_tj, int p, double* d_pn_sums,
                      void* d_ws, size_t ws_bytes, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_u || !d_occ || !(h > 0.0)) return kStatusBadArg;
  ElemArgs A = elem_args(nx, ny, nz, h, E, nu, d_u, d_occ);
  A.strains = d_strains;
  A.stresses = d_stresses;
  A.vm = d_vm;
  A.tj = d_tj;
  A.p = p;
  cudaStream_t s = (cudaStream_t)stream;
  if (d_pn_sums) {
    if (!d_ws || ws_bytes < tvb_elem_ws_bytes(nx, ny, nz) || p < 1) return kStatusWorkspace;
    A.pnorm_partials = (double*)d_ws;
  }
  if (int st = check(launch_element_state(A, s))) return st;
  if (d_pn_sums) return check(launch_sum_pairs((const double*)d_ws, elem_state_ctas(A.g), d_pn_sums, s));
  return kStatusOk;
}

int tvb_adjoint_rhs(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                    const uint8_t* d_nflags, int p, const double* d_pn_sums, double* d_rhs, void* d_ws,
                    size_t ws_bytes, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_u || !d_occ || !d_pn_sums || !d_rhs || p < 2) return kStatusBadArg;
  ElemArgs A = elem_args(nx, ny, nz, h, E, nu, d_u, d_occ);
  A.p = p;
  if (!d_ws || ws_bytes < sizeof(double) * 6 * (size_t)A.g.ne) return kStatusWorkspace;
  return check(launch_adjoint(A, d_pn_sums, (double*)d_ws, d_nflags, d_rhs, (cudaStream_t)stream));
}

int tvb_sens_stress(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_lam,
                    const double* d_occ, double* d_ts, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_u || !d_lam || !d_occ || !d_ts) return kStatusBadArg;
  const ElemArgs A = elem_args(nx, ny, nz, h, E, nu, d_u, d_occ);
  return check(launch_stress_sens(A, d_lam, d_ts, (cudaStream_t)stream));
}

int tvb_maxabs(const double* d_t, long long n, double* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_t || !d_out || n < 0) return kStatusBadArg;
  if (!d_ws || ws_bytes < sizeof(double) * 1184) return kStatusWorkspace;
  return check(launch_maxabs(d_t, n, (double*)d_ws, d_out, (cudaStream_t)stream));
}

int tvb_combine(int k, const double* const* h_fields, const double* h_w, const double* d_maxabs, long long n,
                double* d_out, void* stream) {
  if (k < 1 || k > kMaxFields || !h_fields || !h_w || !d_maxabs || !d_out) return kStatusBadArg;
  CombineArgs C{};
  C.k = k;
  for (int i = 0; i < k; ++i) {
    C.f[i] = h_fields[i];
    C.w[i] = h_w[i];
  }
  C.maxabs = d_maxabs;
  return check(launch_combine(C, n, d_out, (cudaStream_t)stream));
}

size_t tvb_select_ws_bytes(long long n) { return select_ws_bytes(n); }

int tvb_threshold_select_ex(const double* d_ls, const uint8_t* d_design, long long n, long long k, double ersatz,
                            double nondesign, int flags, double* d_occ, void* d_ws, size_t ws_bytes,
                            unsigned long long* h_state4, void* stream) {
  if (!d_ls || !d_occ || n < 1 || k < 0 || k > n || (flags & ~1)) return kStatusBadArg;
  if (!d_ws || ws_bytes < select_ws_bytes(n)) return kStatusWorkspace;
  cudaStream_t s = (cudaStream_t)stream;
  if (int st = check(launch_select(d_ls, d_design, n, k, ersatz, nondesign, d_occ, d_ws, h_state4, s, flags & 1)))
    return st;
  if (h_state4) return check(cudaStreamSynchronize(s));
  return kStatusOk;
}

int tvb_threshold_select(const double* d_ls, const uint8_t* d_design, long long n, long long k, double ersatz,
                         double nondesign, double* d_occ, void* d_ws, size_t ws_bytes, unsigned long long* h_state4,
                         void* stream) {
  return tvb_threshold_select_ex(d_ls, d_design, n, k, ersatz, nondesign, 0, d_occ, d_ws, ws_bytes, h_state4,
                                 stream);
}

int tvb_casting_project(int nx, int ny, int nz, int axis, int parting, const double* d_in, double* d_out,
                        void* stream) {
  if (bad_dims(nx, ny, nz) || axis < 0 || axis > 2 || !d_in || !d_out) return kStatusBadArg;
  const Grid G = make_grid(nx, ny, nz);
  const int na = axis == 0 ? nx : axis == 1 ? ny : nz;
  if (parting < 0 || parting > na) return kStatusBadArg;
  return check(launch_casting_project(G, axis, parting, d_in, d_out, (cudaStream_t)stream));
}

/* ---- eigen / buckling ---------------------------------------- */
int tvb_nodal_block8(int nx, int ny, int nz, const double* d_u, double* d_out, const double* d_blocks, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_u || !d_out || !d_blocks) return kStatusBadArg;
  GeoArgs A{};
  A.g = make_grid(nx, ny, nz);
  A.u = d_u;
  A.y = d_out;
  A.blocks = d_blocks;
  A.accumulate = 1;  // apply_nodal_block8 accumulates into out
  A.scale = 1.0;
  return check(launch_geo_matvec(A, (cudaStream_t)stream));
}

int tvb_geo_matvec(int nx, int ny, int nz, const double* d_Bk, const double* d_stress, const double* d_u,
                   double* d_out, const uint8_t* d_nflags, int flags, double scale, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_Bk || !d_stress || !d_u || !d_out) return kStatusBadArg;
  GeoArgs A{};
  A.g = make_grid(nx, ny, nz);
  A.u = d_u;
  A.y = d_out;
  A.stress = d_stress;
  A.Bk = d_Bk;
  A.nflags = d_nflags;
  A.mask_in = (flags & 1) != 0;
  A.mask_out = (flags & 2) != 0;
  A.accumulate = (flags & 4) != 0;
  A.scale = scale;
  return check(launch_geo_matvec(A, (cudaStream_t)stream));
}

int tvb_lumped_mass(int nx, int ny, int nz, double coef, const double* d_occ, double* d_mass, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_occ || !d_mass) return kStatusBadArg;
  return check(launch_lumped_mass(make_grid(nx, ny, nz), coef, d_occ, d_mass, (cudaStream_t)stream));
}

int tvb_eigen_sens(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                   double omega2rho, double* d_out, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_u || !d_occ || !d_out || !(h > 0.0)) return kStatusBadArg;
  const ElemArgs A = elem_args(nx, ny, nz, h, E, nu, d_u, d_occ);
  return check(launch_eigen_sens(A, omega2rho, d_out, (cudaStream_t)stream));
}

int tvb_buckling_sens(int nx, int ny, int nz, const double* d_k0, const double* d_Bk, const double* d_stress,
                      const double* d_u, const double* d_occ, double lambda, double* d_out, void* stream) {
  if (bad_dims(nx, ny, nz) || !d_k0 || !d_Bk || !d_stress || !d_u || !d_occ || !d_out) return kStatusBadArg;
  return check(launch_buckling_sens(make_grid(nx, ny, nz), d_k0, d_Bk, d_stress, d_u, d_occ, lambda, d_out,
                                    (cudaStream_t)stream));
}

}  // extern "C"
