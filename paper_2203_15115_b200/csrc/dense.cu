// K6: numeric factorisation of the deflation coarse operator E = W^T K W on
// the device, replacing the reference's dense scipy.linalg.cho_factor
// (topovox/fea.py:197-205) and round 1's cuSOLVER / cuBLAS calls.
//
// Every front of the nested-dissection tree (coarse.py) -- and the dense
// "top" Schur complement, and the whole of E for small coarse spaces -- is
// reduced by the block SWEEP operator over its separator: for every 64-wide
// pivot block p of the separator, with P = A_pp^-1,
//     A_ij <- A_ij - A_ip P A_pj      (i, j != p)
//     A_ip <- A_ip P,  A_pj <- P A_pj,  A_pp <- -P.
// After all separator pivots the front holds exactly what the per-iteration
// solve needs (coarse.cu): A_SS = -F_SS^-1 = -Z, A_US = F_US F_SS^-1 = G and
// A_UU = F_UU - F_US F_SS^-1 F_SU, the update passed to the parent front.
// (Sweeping is order-independent and, on an SPD matrix, every pivot block is
// a Schur complement of an SPD matrix: SPD, so no pivoting.)
//
// Kernels, batched over all fronts of one tree height (one launch each):
//   k_front_assemble  build the fronts: symmetrised E entries 0.5 (E + E^T)
//                     (fea.py:198) gathered from the block stencil, plus the
//                     children's updates gathered through per-child position
//                     maps (no atomics, fixed order)
//   k_front_pivot     P = A_pp^-1 by a 2x2-block sweep of the 64x64 pivot
//                     tile in registers (pivot blocks checked SPD)
//   k_front_panel     CT_k = A_pk and R_k = P A_pk for every tile column k
//   k_front_update    A_ik -= CT_i^T R_k on every lower tile (64x64x64 DFMA
//                     tile GEMM, 8x4 register block per thread), and the
//                     pivot row / column / block replaced
// then k_front_pack / k_front_pack_top write G, [Z | -G^T] and the top
// inverse in the layouts the solve kernels read.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "dense.cuh"

namespace tvb {

constexpr int kGemmThreads = 128;

// unpadded front position of padded index R (-1: padding)
__device__ __forceinline__ long long front_unpad(const FrontRec& F, long long R) {
  if (R < F.s_pad) return R < F.s ? R : -1;
  const long long r = F.s + (R - F.s_pad);
  return r < F.s + F.u ? r : -1;
}

__global__ void __launch_bounds__(256) k_front_assemble(FrontFactor Fx, const int* tiles) {
  const int* tr = tiles + 3 * (long long)blockIdx.x;
  const int f = tr[0], I = tr[1], J = tr[2];
  const FrontRec R = Fx.fronts[f];
  double* A = Fx.pool + R.a_off;
  const int ns = (int)(R.s / 6);
  const int* blk = Fx.blocks + R.blk_off;
  const int mx = Fx.mx, mxy = Fx.mx * Fx.my;
  for (int e = threadIdx.x; e < kFT * kFT; e += 256) {
    const long long Rr = (long long)I * kFT + e / kFT, Cc = (long long)J * kFT + e % kFT;
    const long long r = front_unpad(R, Rr), c = front_unpad(R, Cc);
    double v = 0.0;
    if (r < 0 || c < 0) {
      v = (Rr == Cc && Rr < R.s_pad) ? 1.0 : 0.0;
    } else {
      const int br = (int)(r / 6), bc = (int)(c / 6);
      if (br < ns || bc < ns) {
        const int Br = blk[br], Bc = blk[bc];
        const int dx = Bc % mx - Br % mx, dy = (Bc / mx) % Fx.my - (Br / mx) % Fx.my, dz = Bc / mxy - Br / mxy;
        if (dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 && dz <= 1) {
          const int d = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
          const int i = (int)(r % 6), j = (int)(c % 6);
          v = 0.5 * (Fx.Es[((long long)Br * 27 + d) * 36 + i * 6 + j] +
                     Fx.Es[((long long)Bc * 27 + (26 - d)) * 36 + j * 6 + i]);
        }
      }
      for (long long k = 0; k < R.nchild; ++k) {
        const long long* ch = Fx.children + 2 * (R.child_off + k);
        const int* gm = Fx.gmap + ch[1];
        const int gi = gm[r], gj = gm[c];
        if (gi >= 0 && gj >= 0) {
          const FrontRec C = Fx.fronts[ch[0]];
          const long long a = C.s_pad + (gi >= gj ? gi : gj), b = C.s_pad + (gi >= gj ? gj : gi);
          v += Fx.pool[C.a_off + a * C.nf + b];
        }
      }
    }
    A[Rr * R.nf + Cc] = v;
  }
}

// P = A_pp^-1 of every front of the level that still has pivot block p:
// a sweep of the 64x64 pivot tile in 2x2 pivot blocks (32 steps). Thread t
// keeps the 16 entries (rows t/64 + 4q, column t%64) in registers; per step
// only the two pivot columns and rows travel through double-buffered shared
// arrays, so a step costs one barrier. Pivot blocks are checked SPD.
__global__ void __launch_bounds__(256) k_front_pivot(FrontFactor Fx, const int* fronts, int p) {
  __shared__ double2 colb[2][kFT];  // a[i][k], a[i][k+1]
  __shared__ double rowb[2][2][kFT];  // a[k][j], a[k+1][j]
  const FrontRec R = Fx.fronts[fronts[blockIdx.x]];
  if ((long long)p * kFT >= R.s_pad) return;
  const double* A = Fx.pool + R.a_off + (long long)p * kFT * R.nf + (long long)p * kFT;
  const int t = threadIdx.x, j = t % kFT, i0 = t / kFT;  // rows i0 + 4q, column j
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = A[(long long)(i0 + 4 * q) * R.nf + j];
  auto publish = [&](int k, int b) {  // pivot columns / rows k, k+1 into buffer b
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = i0 + 4 * q;
      if (j == k) colb[b][i].x = v[q];
      if (j == k + 1) colb[b][i].y = v[q];
      if (i == k) rowb[b][0][j] = v[q];
      if (i == k + 1) rowb[b][1][j] = v[q];
    }
  };
  publish(0, 0);
  __syncthreads();
  bool bad = false;
  for (int k = 0; k < kFT; k += 2) {
    const int b = (k >> 1) & 1;
    const double2 pk = colb[b][k], pk1 = colb[b][k + 1];  // (a_kk, a_k,k+1), (a_k+1,k, a_k+1,k+1)
    const double det = pk.x * pk1.y - pk.y * pk1.x;
    bad = bad || !(pk.x > 0.0) || !(det > 0.0) || !isfinite(det);
    const double id = 1.0 / det;
    const double p00 = pk1.y * id, p01 = -pk.y * id, p10 = -pk1.x * id, p11 = pk.x * id;  // inv 2x2
    const double rk = rowb[b][0][j], rk1 = rowb[b][1][j];
    // (P [a_kj; a_k+1,j]) for this column
    const double w0 = p00 * rk + p01 * rk1, w1 = p10 * rk + p11 * rk1;
    const bool jk = j == k || j == k + 1;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = i0 + 4 * q;
      const bool ik = i == k || i == k + 1;
      const double2 c = colb[b][i];
      double nv;
      if (!ik && !jk) {
        nv = fma(-c.x, w0, fma(-c.y, w1, v[q]));
      } else if (!ik) {  // column k or k+1: [a_ik a_ik+1] P
        nv = j == k ? c.x * p00 + c.y * p10 : c.x * p01 + c.y * p11;
      } else if (!jk) {  // row k or k+1: P [a_kj; a_k+1,j]
        nv = i == k ? w0 : w1;
      } else {
        nv = -(i == k ? (j == k ? p00 : p01) : (j == k ? p10 : p11));
      }
      v[q] = nv;
    }
    if (k + 2 < kFT) publish(k + 2, b ^ 1);
    __syncthreads();
  }
  if (bad && t == 0) atomicOr(Fx.d_err, 1);
  double* P = Fx.scratch + R.scr_off;
#pragma unroll
  for (int q = 0; q < 16; ++q) P[(i0 + 4 * q) * kFT + j] = -v[q];
}

// smem[m * ldb + b] = tile element (row m, col b) of the pivot row block A_pk
// (stored tile (p, k) when p >= k, else the transpose of stored tile (k, p))
__device__ __forceinline__ void load_row_tile(const FrontRec& R, const double* A, int p, int k, double* sm,
                                              int ldb) {
  if (p >= k) {
    const double* src = A + (long long)p * kFT * R.nf + (long long)k * kFT;
    for (int e = threadIdx.x; e < kFT * kFT / 2; e += kGemmThreads) {
      const int m = e / (kFT / 2), b2 = e % (kFT / 2);
      const double2 v = *reinterpret_cast<const double2*>(src + (long long)m * R.nf + 2 * b2);
      sm[m * ldb + 2 * b2] = v.x;
      sm[m * ldb + 2 * b2 + 1] = v.y;
    }
  } else {
    const double* src = A + (long long)k * kFT * R.nf + (long long)p * kFT;  // tile (k, p): [b][m]
    for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) {
      const int b = e / kFT, m = e % kFT;
      sm[m * ldb + b] = src[(long long)b * R.nf + m];
    }
  }
}

// acc[r][c] += sum_m As[m][ty + 8r] * Bs[m][tx + 16c]
__device__ __forceinline__ void tile_gemm(const double* As, const double* Bs, int ldb, double (&acc)[8][4]) {
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll 4
  for (int m = 0; m < kFT; ++m) {
    double a[8], b[4];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = As[m * kFT + ty + 8 * r];
#pragma unroll
    for (int c = 0; c < 4; ++c) b[c] = Bs[m * ldb + tx + 16 * c];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
  }
}

constexpr int kLdb = kFT + 1;
constexpr size_t kGemmSmem = sizeof(double) * (kFT * kFT + kFT * kLdb);

// for every tile column k != p: CT_k = A_pk, R_k = P A_pk
__global__ void __launch_bounds__(kGemmThreads) k_front_panel(FrontFactor Fx, const int* cols, int p) {
  extern __shared__ __align__(16) double sm[];
  const int f = cols[2 * (long long)blockIdx.x], k = cols[2 * (long long)blockIdx.x + 1];
  const FrontRec R = Fx.fronts[f];
  if ((long long)p * kFT >= R.s_pad || k == p) return;
  double* As = sm;
  double* Bs = sm + kFT * kFT;
  const double* A = Fx.pool + R.a_off;
  const double* P = Fx.scratch + R.scr_off;
  for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) As[e] = P[e];  // P symmetric: As[m][a] = P[a][m]
  load_row_tile(R, A, p, k, Bs, kLdb);
  __syncthreads();
  double* CT = Fx.scratch + R.scr_off + (long long)kFT * kFT * (1 + k);
  double* RK = Fx.scratch + R.scr_off + (long long)kFT * kFT * (1 + R.ntf + k);
  for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) CT[e] = Bs[(e / kFT) * kLdb + e % kFT];
  double acc[8][4] = {};
  tile_gemm(As, Bs, kLdb, acc);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) RK[(ty + 8 * r) * kFT + tx + 16 * c] = acc[r][c];
}

// every lower tile (I, J): the sweep update of pivot block p
__global__ void __launch_bounds__(kGemmThreads) k_front_update(FrontFactor Fx, const int* tiles, int p) {
  extern __shared__ __align__(16) double sm[];
  const int* tr = tiles + 3 * (long long)blockIdx.x;
  const int f = tr[0], I = tr[1], J = tr[2];
  const FrontRec R = Fx.fronts[f];
  if ((long long)p * kFT >= R.s_pad) return;
  double* A = Fx.pool + R.a_off + (long long)I * kFT * R.nf + (long long)J * kFT;
  const double* scr = Fx.scratch + R.scr_off;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  if (I == p && J == p) {  // A_pp <- -P
    for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) A[(long long)(e / kFT) * R.nf + e % kFT] = -scr[e];
    return;
  }
  if (J == p) {  // A_ip <- A_ip P = R_i^T
    const double* Ri = scr + (long long)kFT * kFT * (1 + R.ntf + I);
    for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) {
      const int a = e / kFT, b = e % kFT;
      A[(long long)a * R.nf + b] = Ri[b * kFT + a];
    }
    return;
  }
  if (I == p) {  // A_pj <- P A_pj = R_j
    const double* Rj = scr + (long long)kFT * kFT * (1 + R.ntf + J);
    for (int e = threadIdx.x; e < kFT * kFT; e += kGemmThreads) A[(long long)(e / kFT) * R.nf + e % kFT] = Rj[e];
    return;
  }
  // A_IJ -= A_Ip P A_pJ = CT_I^T R_J
  double* As = sm;
  double* Bs = sm + kFT * kFT;
  const double2* ct = reinterpret_cast<const double2*>(scr + (long long)kFT * kFT * (1 + I));
  const double2* rj = reinterpret_cast<const double2*>(scr + (long long)kFT * kFT * (1 + R.ntf + J));
  for (int e = threadIdx.x; e < kFT * kFT / 2; e += kGemmThreads) {
    const double2 v = ct[e];
    As[2 * e] = v.x;
    As[2 * e + 1] = v.y;
    const double2 w = rj[e];
    const int m = (2 * e) / kFT, b = (2 * e) % kFT;
    Bs[m * kLdb + b] = w.x;
    Bs[m * kLdb + b + 1] = w.y;
  }
  __syncthreads();
  double acc[8][4];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = A[(long long)(ty + 8 * r) * R.nf + tx + 16 * c];
  // acc -= CT^T R: negate one operand's contribution via the accumulate order
#pragma unroll 4
  for (int m = 0; m < kFT; ++m) {
    double a[8], b[4];
#pragma unroll
    for (int r = 0; r < 8; ++r) a[r] = As[m * kFT + ty + 8 * r];
#pragma unroll
    for (int c = 0; c < 4; ++c) b[c] = Bs[m * kLdb + tx + 16 * c];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = fma(-a[r], b[c], acc[r][c]);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) A[(long long)(ty + 8 * r) * R.nf + tx + 16 * c] = acc[r][c];
}

cudaError_t launch_front_level(const FrontFactor& F, const FrontLevel& L, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_front_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
    cudaFuncSetAttribute(k_front_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGemmSmem);
    attr = true;
  }
  if (L.n_tiles > 0) k_front_assemble<<<L.n_tiles, 256, 0, s>>>(F, L.tiles);
  for (int p = 0; p < L.max_steps; ++p) {
    k_front_pivot<<<L.n_fronts, 256, 0, s>>>(F, L.fronts, p);
    k_front_panel<<<L.n_cols, kGemmThreads, kGemmSmem, s>>>(F, L.cols, p);
    k_front_update<<<L.n_tiles, kGemmThreads, kGemmSmem, s>>>(F, L.tiles, p);
  }
  return cudaGetLastError();
}

// G[a][b] = A[s_pad + a][b] (u x s); B[a][b] = Z[a][b] = -A[max][min] (b < s), B[a][s + c] = -G[c][a]
__global__ void k_front_pack(FrontFactor Fx, int f, double* G, double* B) {
  const FrontRec R = Fx.fronts[f];
  const double* A = Fx.pool + R.a_off;
  const long long s = R.s, u = R.u;
  const long long nG = u * s, nB = s * (s + u);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nG + nB;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nG) {
      const long long a = e / s, b = e % s;
      G[e] = A[(R.s_pad + a) * R.nf + b];
    } else {
      const long long q = e - nG, a = q / (s + u), b = q % (s + u);
      double v;
      if (b < s) v = -(a >= b ? A[a * R.nf + b] : A[b * R.nf + a]);
      else v = -A[(R.s_pad + (b - s)) * R.nf + a];
      B[q] = v;
    }
  }
}

// out = Z = -A (order n): tiles > 0: lower 64x64 tiles, tile I (I + 1) / 2 + J row-major, zero padded;
// tiles == 0: dense rows
__global__ void k_front_pack_top(FrontFactor Fx, int f, long long n, int tiles, double* out) {
  const FrontRec R = Fx.fronts[f];
  const double* A = Fx.pool + R.a_off;
  const long long total = tiles > 0 ? (long long)tiles * (tiles + 1) / 2 * kFT * kFT : n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r, c;
    if (tiles > 0) {
      const long long t = e / (kFT * kFT), w = e % (kFT * kFT);
      long long I = (long long)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      while (I * (I + 1) / 2 > t) --I;
      const long long J = t - I * (I + 1) / 2;
      r = I * kFT + w / kFT;
      c = J * kFT + w % kFT;
    } else {
      r = e / n;
      c = e % n;
    }
    double v = 0.0;
    if (r < n && c < n) v = -(r >= c ? A[r * R.nf + c] : A[c * R.nf + r]);
    out[e] = v;
  }
}

cudaError_t launch_front_pack(const FrontFactor& F, int front, double* G, double* B, long long s_, long long u_,
                              cudaStream_t s) {
  const long long n = u_ * s_ + s_ * (s_ + u_);
  const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148 * 16);
  k_front_pack<<<grid, 256, 0, s>>>(F, front, G, B);
  return cudaGetLastError();
}

cudaError_t launch_front_pack_top(const FrontFactor& F, int front, long long n, int tiles, double* out,
                                  cudaStream_t s) {
  const long long total = tiles > 0 ? (long long)tiles * (tiles + 1) / 2 * kFT * kFT : n * n;
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148 * 16);
  k_front_pack_top<<<grid, 256, 0, s>>>(F, front, n, tiles, out);
  return cudaGetLastError();
}

}  // namespace tvb
