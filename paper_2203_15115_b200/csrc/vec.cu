// K2/K3: Jacobi diagonal, fused PCG vector updates and deterministic
// reductions (replaces diag_block24, topovox/backends/numba_kernels.py:49-58,
// and the numpy/OpenBLAS vector algebra of solve_static, topovox/fea.py:241-291).
//
// Every reduction is two-stage and order-fixed: each CTA reduces a fixed
// contiguous slice with a warp-shuffle tree, writes its partial, and the last
// CTA to finish (device counter) sums the partials in index order. Results are
// therefore bitwise reproducible for a given launch geometry.
#include <algorithm>
#include <cstdlib>

#include "vec.cuh"

namespace tvb {

// Last-CTA finaliser: sums `nparts` partial vectors of width W (laid out
// [part][W]) in index order and hands the totals to `fin` in thread 0.
template <int W, typename Fin>
__device__ void finalize_last(double* partials, int nparts, unsigned int* counter, double* red, Fin fin) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == (unsigned)(gridDim.x * gridDim.y - 1));
  __syncthreads();
  if (!last) return;
  __threadfence();
  double tot[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += ((volatile double*)partials)[(size_t)i * W + w];
    tot[w] = block_sum(s, red);
  }
  if (threadIdx.x == 0) {
    *counter = 0u;
    fin(tot);
  }
}

// ---------------------------------------------------------------------------
// inverse Jacobi diagonal: diag(K)[3n+a] = k0[a,a] * sum_{e ∋ n} occ_e
// ---------------------------------------------------------------------------
__global__ void k_inv_diag(Grid G, const double* occ, const uint8_t* nflags, double3 kd,
                           double* inv_d, double* diag_out, int accumulate, int* zero_free) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= G.nn) return;
  const int x = (int)(n % G.px);
  const int y = (int)((n / G.px) % G.py);
  const int z = (int)(n / ((long long)G.px * G.py));
  double s = 0.0;
  // fixed element order: dz, dy, dx in {-1, 0}
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int ex = x + dx, ey = y + dy, ez = z + dz;
        if (ex >= 0 && ex < G.nx && ey >= 0 && ey < G.ny && ez >= 0 && ez < G.nz) s += occ[G.elem(ex, ey, ez)];
      }
  const uint8_t fl = nflags ? nflags[n] : 0;
  const double kk[3] = {kd.x, kd.y, kd.z};
  for (int a = 0; a < 3; ++a) {
    const double d = kk[a] * s;
    if (diag_out) diag_out[3 * n + a] = accumulate ? diag_out[3 * n + a] + d : d;
    const bool fixed = (fl >> a) & 1;
    if (inv_d) inv_d[3 * n + a] = fixed ? 0.0 : (d != 0.0 ? 1.0 / d : 0.0);
    if (!fixed && d == 0.0 && zero_free) atomicAdd(zero_free, 1);
  }
}

// ---------------------------------------------------------------------------
// generic deterministic dot products
// ---------------------------------------------------------------------------
__global__ void k_dot(const double* a, const double* b, const double* wmask, long long n, double* partials,
                      unsigned int* counter, double* out) {
  __shared__ double red[32];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double v = a[i] * b[i];
    if (wmask) v *= wmask[i];
    s += v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  finalize_last<1>(partials, gridDim.x, counter, red, [&](double* t) { *out = t[0]; });
}

// ---------------------------------------------------------------------------
// PCG iteration kernels (state lives on the device; see vec.cuh)
// ---------------------------------------------------------------------------

// alpha = rz / pq ; x += alpha p ; r -= alpha q ; z = inv_d r ; rr, rz partials.
// The last CTA decides convergence exactly like topovox/fea.py:277-291.
__global__ void k_pcg_update(long long n, double* x, double* r, double* z, const double* p, const double* q,
                             const double* inv_d, SolverState* st, double* partials) {
  __shared__ double red[32];
  if (st->done) return;
  const double alpha = st->rz / st->pq;
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  double rr = 0.0, rz = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (x != nullptr) x[i] = fma(alpha, p[i], x[i]);
    // inv_d == 0 marks a fixed DOF: r stays 0 there whatever q holds (the
    // iteration's matvecs do not mask their output, see k_pcg_update_v2)
    const double di = inv_d[i];
    const double ri = di == 0.0 ? 0.0 : fma(-alpha, q[i], r[i]);
    r[i] = ri;
    const double zi = di * ri;
    z[i] = zi;
    rr = fma(ri, ri, rr);
    rz = fma(ri, zi, rz);
  }
  rr = block_sum(rr, red);
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = rr;
    partials[2 * blockIdx.x + 1] = rz;
  }
  finalize_last<2>(partials, gridDim.x, &st->counter, red, [&](double* t) {
    st->alpha = alpha;
    st->iter += 1;
    st->rr = t[0];
    st->res = sqrt(t[0]) / st->fnorm;
    if (st->res <= st->tol) {
      st->done = 1;
    } else if (st->iter >= st->max_iters) {
      st->done = 2;
    } else {
      st->beta = t[1] / st->rz;
      st->rz = t[1];
    }
  });
}

// Same update, 16-byte vector accesses (all six vectors 16-byte aligned),
// grid-strided so that all CTAs sweep the vectors together. Identical
// arithmetic per element; the partial sums run in a different (still fixed)
// order. WX = false: x is not touched (the deflated solver folds x += alpha p
// into the prolongation, which reads p anyway).
template <bool WX>
__global__ void __launch_bounds__(256) k_pcg_update_v2(long long n, double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ z, const double* __restrict__ p,
                                                       const double* __restrict__ q,
                                                       const double* __restrict__ inv_d, SolverState* st,
                                                       double* partials, const double* pq_parts, int n_parts) {
  pdl_entry();
  __shared__ double red[32];
  __shared__ double s_pq;
  if (st->done) return;
  const long long n2 = n >> 1;
  const long long hi = n2;  // grid-strided: all CTAs sweep the vectors together
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* z2 = reinterpret_cast<double2*>(z);
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  const double2* d2 = reinterpret_cast<const double2*>(inv_d);
  // Software pipeline over pairs (i, i + blockDim.x), i += 2 * blockDim.x:
  // the operands of pair k+1 are loaded before pair k is processed, and the
  // first pair's loads are issued before the p.q reduction so their DRAM
  // latency overlaps the partial-sum reads. Same elements in the same order
  // per thread as a plain loop (bitwise identical partial sums).
  struct Ops {
    double2 p, x, q, r, d;
  };
  auto load = [&](long long k, Ops& o) {
    if (WX) {
      o.p = p2[k];
      o.x = x2[k];
    }
    o.q = q2[k];
    o.r = r2[k];
    o.d = __ldg(d2 + k);
  };
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long step = (long long)gridDim.x * blockDim.x;
  Ops a{}, b{};
  if (i < hi) load(i, a);
  if (i + step < hi) load(i + step, b);
  // p.q from the matvec's per-CTA partials, summed by every CTA in the same
  // fixed order (replaces a separate finaliser launch)
  if (pq_parts != nullptr) {
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int j = threadIdx.x; j < n_parts; j += 32) s += __ldcg(pq_parts + j);
      s = warp_sum(s);
      if (threadIdx.x == 0) s_pq = s;
    }
    __syncthreads();
  } else if (threadIdx.x == 0) {
    s_pq = st->pq;
  }
  __syncthreads();
  const double pq = s_pq;
  const double alpha = st->rz / pq;
  double rr = 0.0, rz = 0.0;
  auto one = [&](const Ops& o, long long k) {
    if (WX) {
      double2 xi = o.x;
      xi.x = fma(alpha, o.p.x, xi.x);
      xi.y = fma(alpha, o.p.y, xi.y);
      __stcs(x2 + k, xi);  // x and r are next read one iteration later: evict first
    }
    // inv_d == 0 marks a fixed DOF (k_inv_diag; a zero diagonal on a free DOF
    // aborts the solve before the loop): r stays exactly 0 there whatever q
    // holds, so the iteration's matvecs need no output mask (3.7 us per K.u
    // at C4) -- r, z and both sums are bitwise those of the masked form
    double2 ri = o.r;
    ri.x = o.d.x == 0.0 ? 0.0 : fma(-alpha, o.q.x, ri.x);
    ri.y = o.d.y == 0.0 ? 0.0 : fma(-alpha, o.q.y, ri.y);
    double2 zi;
    zi.x = o.d.x * ri.x;
    zi.y = o.d.y * ri.y;
    __stcs(r2 + k, ri);
    z2[k] = zi;
    rr = fma(ri.x, ri.x, rr);
    rz = fma(ri.x, zi.x, rz);
    rr = fma(ri.y, ri.y, rr);
    rz = fma(ri.y, zi.y, rz);
  };
  while (i < hi) {
    const long long inext = i + 2 * step;
    Ops na{}, nb{};
    if (inext < hi) load(inext, na);
    if (inext + step < hi) load(inext + step, nb);
    one(a, i);
    if (i + step < hi) one(b, i + step);
    a = na;
    b = nb;
    i = inext;
  }
  if ((n & 1) && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {  // odd tail element
    const long long k = n - 1;
    if (WX) x[k] = fma(alpha, p[k], x[k]);
    const double rk = inv_d[k] == 0.0 ? 0.0 : fma(-alpha, q[k], r[k]);
    r[k] = rk;
    const double zk = inv_d[k] * rk;
    z[k] = zk;
    rr = fma(rk, rk, rr);
    rz = fma(rk, zk, rz);
  }
  rr = block_sum(rr, red);
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = rr;
    partials[2 * blockIdx.x + 1] = rz;
  }
  finalize_last<2>(partials, gridDim.x, &st->counter, red, [&](double* t) {
    st->pq = pq;
    st->alpha = alpha;
    st->iter += 1;
    st->rr = t[0];
    st->res = sqrt(t[0]) / st->fnorm;
    if (st->res <= st->tol) {
      st->done = 1;
    } else if (st->iter >= st->max_iters) {
      st->done = 2;
    } else {
      st->beta = t[1] / st->rz;
      st->rz = t[1];
    }
  });
}

__global__ void k_x_finish(long long n, double* x, const double* p, const SolverState* st) {
  const double alpha = st->alpha;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = fma(alpha, p[i], x[i]);
}

cudaError_t launch_x_finish(long long n, double* x, const double* p, const SolverState* st, cudaStream_t s) {
  k_x_finish<<<reduce_grid(n) * 4, 256, 0, s>>>(n, x, p, st);
  return cudaGetLastError();
}

// plain PCG direction update p = z + beta p
__global__ void k_pcg_pupdate(long long n, double* p, const double* z, const SolverState* st) {
  pdl_entry();
  if (st->done) return;
  const double beta = st->beta;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], z[i]);
}

// matvec dot finaliser: pq = sum partials (written by k_matvec)
__global__ void k_finalize_pq(const double* partials, int nparts, SolverState* st) {
  __shared__ double red[32];
  if (st->done) return;
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) st->pq = s;
}

// r = f - A x0 (Ax already in r), r[fixed] = 0, z = inv_d r; rr, rz.
__global__ void k_pcg_init(long long n, const double* f, double* r, double* z, const double* inv_d,
                           const uint8_t* nflags, int have_ax, double* partials, SolverState* st) {
  __shared__ double red[32];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  double rr = 0.0, rz = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double ri = have_ax ? f[i] - r[i] : f[i];
    if (nflags && ((nflags[i / 3] >> (i % 3)) & 1)) ri = 0.0;
    r[i] = ri;
    const double zi = inv_d[i] * ri;
    z[i] = zi;
    rr = fma(ri, ri, rr);
    rz = fma(ri, zi, rz);
  }
  rr = block_sum(rr, red);
  rz = block_sum(rz, red);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = rr;
    partials[2 * blockIdx.x + 1] = rz;
  }
  finalize_last<2>(partials, gridDim.x, &st->counter, red, [&](double* t) {
    st->rr = t[0];
    st->rz = t[1];
    st->res = sqrt(t[0]) / st->fnorm;
    st->iter = 0;
    st->done = (st->res <= st->tol) ? 1 : 0;
  });
}

// ||f_free||^2 into st->fnorm (sqrt applied)
__global__ void k_free_norm(long long n, const double* f, const uint8_t* nflags, double* partials, SolverState* st) {
  __shared__ double red[32];
  const long long per = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(n, lo + per);
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const bool fixed = nflags && ((nflags[i / 3] >> (i % 3)) & 1);
    if (!fixed) s = fma(f[i], f[i], s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  finalize_last<1>(partials, gridDim.x, &st->counter, red, [&](double* t) { st->fnorm = sqrt(t[0]); });
}

// x[fixed] = 0 (final clean-up, topovox/fea.py:298)
__global__ void k_zero_fixed(long long nn, double* x, const uint8_t* nflags) {
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= nn) return;
  const uint8_t f = nflags[n];
  for (int a = 0; a < 3; ++a)
    if ((f >> a) & 1) x[3 * n + a] = 0.0;
}

// ---------------------------------------------------------------------------
// host wrappers
// ---------------------------------------------------------------------------
int reduce_grid(long long n) {
  long long b = (n + 4095) / 4096;
  if (b < 1) b = 1;
  if (b > kMaxReduceCtas) b = kMaxReduceCtas;
  return (int)b;
}

cudaError_t launch_inv_diag(const Grid& G, const double* occ, const uint8_t* nflags, const double kd[3],
                            double* inv_d, double* diag_out, int* zero_free, cudaStream_t s, int accumulate) {
  const int nt = 256;
  const long long nb = (G.nn + nt - 1) / nt;
  k_inv_diag<<<(unsigned)nb, nt, 0, s>>>(G, occ, nflags, make_double3(kd[0], kd[1], kd[2]), inv_d, diag_out,
                                          accumulate, zero_free);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* a, const double* b, const double* w, long long n, double* ws,
                       unsigned int* counter, double* out, cudaStream_t s) {
  k_dot<<<reduce_grid(n), 256, 0, s>>>(a, b, w, n, ws, counter, out);
  return cudaGetLastError();
}

cudaError_t launch_pcg_update(long long n, double* x, double* r, double* z, const double* p, const double* q,
                              const double* inv_d, SolverState* st, double* partials, const double* pq_parts,
                              int n_parts, cudaStream_t s) {
  const bool vec16 = (((x ? reinterpret_cast<uintptr_t>(x) : 0) | reinterpret_cast<uintptr_t>(r) |
                       reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(p) |
                       reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(inv_d)) & 15) == 0;
  // grid: at most 2 CTAs per SM (an exact multiple of the SM count for large
  // vectors). Measured with the grid-strided prefetching kernel: C4 203.7 us
  // per DPCG iteration (592 CTAs: 207.7; the previous contiguous-range kernel
  // at 592 CTAs: 204.5), C3 111.8 (116.3), C5 1584 (1600); TVB_UPD_CTAS
  // overrides (A/B experiments)
  static int upd_ctas = -1;
  if (upd_ctas < 0) {
    upd_ctas = getenv("TVB_UPD_CTAS") ? atoi(getenv("TVB_UPD_CTAS")) : 0;
    if (upd_ctas <= 0) {
      int dev = 0, nsm = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      upd_ctas = 2 * nsm;
    }
  }
  const int g = std::min(std::min(upd_ctas, kMaxReduceCtas), reduce_grid(n));
  if (vec16 && x != nullptr) {
    launch_k(k_pcg_update_v2<true>, g, 256, 0, s, n, x, r, z, p, q, inv_d, st, partials, pq_parts, n_parts);
  } else if (vec16) {
    launch_k(k_pcg_update_v2<false>, g, 256, 0, s, n, x, r, z, p, q, inv_d, st, partials, pq_parts, n_parts);
  } else {
    if (pq_parts != nullptr) k_finalize_pq<<<1, 256, 0, s>>>(pq_parts, n_parts, st);
    k_pcg_update<<<reduce_grid(n), 256, 0, s>>>(n, x, r, z, p, q, inv_d, st, partials);
  }
  return cudaGetLastError();
}

cudaError_t launch_pcg_pupdate(long long n, double* p, const double* z, const SolverState* st, cudaStream_t s) {
  launch_k(k_pcg_pupdate, reduce_grid(n) * 4, 256, 0, s, n, p, z, st);
  return cudaGetLastError();
}

cudaError_t launch_finalize_pq(const double* partials, int nparts, SolverState* st, cudaStream_t s) {
  k_finalize_pq<<<1, 256, 0, s>>>(partials, nparts, st);
  return cudaGetLastError();
}

cudaError_t launch_pcg_init(long long n, const double* f, double* r, double* z, const double* inv_d,
                            const uint8_t* nflags, int have_ax, double* partials, SolverState* st, cudaStream_t s) {
  k_pcg_init<<<reduce_grid(n), 256, 0, s>>>(n, f, r, z, inv_d, nflags, have_ax, partials, st);
  return cudaGetLastError();
}

cudaError_t launch_free_norm(long long n, const double* f, const uint8_t* nflags, double* partials, SolverState* st,
                             cudaStream_t s) {
  k_free_norm<<<reduce_grid(n), 256, 0, s>>>(n, f, nflags, partials, st);
  return cudaGetLastError();
}

cudaError_t launch_zero_fixed(long long nn, double* x, const uint8_t* nflags, cudaStream_t s) {
  k_zero_fixed<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(nn, x, nflags);
  return cudaGetLastError();
}

}  // namespace tvb
