// K1: assembly-free hex stiffness matvec  y = M_out * sum_e occ_e P_e^T k0 P_e * M_in u
//
// Replaces the numba kernel apply_block24 (topovox/backends/numba_kernels.py:12-28)
// called from StiffnessOperator.apply (topovox/fea.py:49-65).
//
// Design:
//  * z-marching node-owner tiles. A CTA owns a (wx-1) x (wy-1) column of nodes
//    over a chunk of z-planes; each thread owns one element column of the
//    wx x wy tile (one-element halo on the low x/y side) and walks it in z.
//    Every output node is written by exactly one thread, which sums its 8
//    element contributions in a fixed order: the result is bitwise
//    deterministic and needs no atomics.
//  * u is staged plane by plane into a 3-deep shared-memory ring with cp.async,
//    one plane ahead of the compute.
//  * k0 is applied in the Walsh-Hadamard mode basis of the cube (45 nonzeros
//    instead of 576, gen_modal.py), as H3 * Mh * H3^T with butterflies.
//  * the z-direction node sum is done in mode space in registers (the "carry"
//    of the upper face), the x/y sums through one shared-memory exchange.
#include "matvec.cuh"

namespace tvb {

__device__ __forceinline__ void modal_apply(const double* __restrict__ mh, const double (&c)[24], double (&g)[24]) {
#include "modal_apply.inc"
}

template <int NT>
__global__ void __launch_bounds__(NT, (NT <= 256 ? 2 : 1)) k_matvec(MatvecParams P, Modal M) {
  extern __shared__ double smem[];
  if (P.stop != nullptr && *P.stop) return;
  const Grid& G = P.g;
  const int wx = P.wx, wy = P.wy;
  const int PW = wx + 1, PH = wy + 1, PN = PW * PH;  // node tile of one plane
  const int tile = blockIdx.x;
  const int x0 = (tile % P.ntx) * (wx - 1);
  const int y0 = (tile / P.ntx) * (wy - 1);
  const int kz0 = blockIdx.y * P.zc;
  const int kz1 = min(kz0 + P.zc, G.pz);  // owned planes [kz0, kz1)

  double* Up = smem;                 // [3][PN*3] plane ring
  double* Xc = smem + 9 * PN;        // [NT][9] face-node exchange
  double* red = Xc + 9 * NT;         // [NT/32] reduction scratch

  const int t = threadIdx.x;
  const bool active = t < wx * wy;
  const int tx = active ? t % wx : 0, ty = active ? t / wx : 0;
  const int ex = x0 - 1 + tx, ey = y0 - 1 + ty;
  const bool col_in = active && ex >= 0 && ex < G.nx && ey >= 0 && ey < G.ny;
  const bool owner = active && tx < wx - 1 && ty < wy - 1 && (x0 + tx) < G.px && (y0 + ty) < G.py;

  auto load_plane = [&](int k) {
    double* dst = Up + ((k + 3) % 3) * (3 * PN);
    const bool kin = (k >= 0 && k < G.pz);
    const int rowlen = 3 * PW;
    for (int idx = t; idx < 3 * PN; idx += NT) {
      const int jy = idx / rowlen, r = idx - jy * rowlen;
      const int gx = x0 - 1 + r / 3, gy = y0 - 1 + jy;
      if (kin && gx >= 0 && gx < G.px && gy >= 0 && gy < G.py) {
        const long long off = 3 * G.node(x0 - 1, gy, k) + r;
        cp_async8(dst + idx, P.u + off);
      } else {
        dst[idx] = 0.0;
      }
    }
    cp_async_commit();
  };
  auto mask_plane = [&](int k) {
    if (!P.mask_in || P.fixed == nullptr || k < 0 || k >= G.pz) return;
    double* dst = Up + ((k + 3) % 3) * (3 * PN);
    const int rowlen = 3 * PW;
    for (int idx = t; idx < 3 * PN; idx += NT) {
      const int jy = idx / rowlen, r = idx - jy * rowlen;
      const int gx = x0 - 1 + r / 3, gy = y0 - 1 + jy;
      if (gx >= 0 && gx < G.px && gy >= 0 && gy < G.py) {
        if ((P.fixed[G.node(gx, gy, k)] >> (r % 3)) & 1) dst[idx] = 0.0;
      }
    }
  };

  double carry[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) carry[i] = 0.0;
  double dot = 0.0;

  load_plane(kz0 - 1);
  load_plane(kz0);
  double occ_next = 0.0;
  if (col_in && kz0 - 1 >= 0 && kz0 - 1 < G.nz) occ_next = P.occ[G.elem(ex, ey, kz0 - 1)];

  for (int k = kz0 - 1; k < kz1; ++k) {
    cp_async_wait_all();
    if (k == kz0 - 1) mask_plane(k);
    mask_plane(k + 1);
    __syncthreads();
    if (k + 2 <= kz1) load_plane(k + 2);

    const double occ_e = occ_next;
    if (col_in && k + 1 >= 0 && k + 1 < G.nz) occ_next = P.occ[G.elem(ex, ey, k + 1)];
    else occ_next = 0.0;

    // gather the 8 nodes (binary local index b = ox + 2 oy + 4 oz) -> c[3b + a]
    double c[24];
    {
      const double* lo = Up + ((k + 3) % 3) * (3 * PN);
      const double* hi = Up + ((k + 4) % 3) * (3 * PN);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = 3 * ((ty + (b >> 1)) * PW + tx + (b & 1));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          c[3 * b + a] = lo[j + a];
          c[3 * (b + 4) + a] = hi[j + a];
        }
      }
    }
    // forward Walsh-Hadamard (H^T): butterflies over the x, y, z bits
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1) {
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        if (b & bit) continue;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double v0 = c[3 * b + a], v1 = c[3 * (b | bit) + a];
          c[3 * b + a] = v0 + v1;
          c[3 * (b | bit) + a] = v1 - v0;
        }
      }
    }
    double gm[24];
    modal_apply(M.mh, c, gm);
    // z-stage of the inverse transform, faces in xy-mode space
    double face[12];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double g0 = occ_e * gm[3 * m + a], g1 = occ_e * gm[3 * (m + 4) + a];
        face[3 * m + a] = (g0 - g1) + carry[3 * m + a];
        carry[3 * m + a] = g0 + g1;
      }
    }
    if (k >= kz0) {
      // xy inverse transform: mode (mx,my) -> node (ox,oy)
#pragma unroll
      for (int bit = 1; bit < 4; bit <<= 1) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b & bit) continue;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double g0 = face[3 * b + a], g1 = face[3 * (b | bit) + a];
            face[3 * b + a] = g0 - g1;
            face[3 * (b | bit) + a] = g0 + g1;
          }
        }
      }
      double* xs = Xc + 9 * t;
#pragma unroll
      for (int i = 0; i < 9; ++i) xs[i] = face[i];  // nodes (0,0), (1,0), (0,1)
      __syncthreads();
      if (owner) {
        // node (x0+tx, y0+ty) = local (1,1) of this column, (0,1) of column
        // tx+1, (1,0) of column ty+1 and (0,0) of column (tx+1, ty+1).
        const double* e10 = Xc + 9 * (t + 1);
        const double* e01 = Xc + 9 * (t + wx);
        const double* e11 = Xc + 9 * (t + wx + 1);
        const long long n = G.node(x0 + tx, y0 + ty, k);
        const uint8_t fx = (P.fixed != nullptr) ? P.fixed[n] : 0;
        const double* us = Up + ((k + 3) % 3) * (3 * PN) + 3 * ((ty + 1) * PW + tx + 1);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double v = face[9 + a] + e10[6 + a];
          v += e01[3 + a];
          v += e11[a];
          if (P.mask_out && ((fx >> a) & 1)) v = 0.0;
          if (P.accumulate) v += P.y[3 * n + a];
          P.y[3 * n + a] = v;
          dot = fma(us[a], v, dot);
        }
      }
    }
  }
  if (P.dot_partial != nullptr) {
    const double s = block_sum(dot, red);
    if (t == 0) P.dot_partial[blockIdx.x + gridDim.x * blockIdx.y] = s;
  }
}

// Host-side launch planning -------------------------------------------------

static size_t matvec_smem(int nt, int wx, int wy) {
  const int PN = (wx + 1) * (wy + 1);
  return sizeof(double) * (9 * (size_t)PN + 9 * (size_t)nt + nt / 32 + 1);
}

// Pick the tile that minimises (waves x per-CTA work); a CTA's work is
// (zc + 1) layers of wx*wy element columns.
MatvecPlan plan_matvec(const Grid& g, int num_sms) {
  MatvecPlan best{};
  double best_cost = 1e300;
  const int nt = 256;
  const int ctas_per_sm = 2;
  for (int wx = 12; wx <= 64; ++wx) {
    for (int wy = 3; wx * wy <= nt; ++wy) {
      if (wx * wy < nt - 32) continue;  // keep warps full
      const int ntx = (g.px + wx - 2) / (wx - 1);
      const int nty = (g.py + wy - 2) / (wy - 1);
      const long long tiles = (long long)ntx * nty;
      for (int nzc = 1; nzc <= g.pz; ++nzc) {
        const int zc = (g.pz + nzc - 1) / nzc;
        const int nzc_eff = (g.pz + zc - 1) / zc;
        const long long ctas = tiles * nzc_eff;
        const long long slots = (long long)num_sms * ctas_per_sm;
        const long long waves = (ctas + slots - 1) / slots;
        // fill fraction of the last wave still costs a full wave per SM
        const double cost = (double)waves * (zc + 1) * 1.0 + 0.02 * (double)ctas / slots;
        if (cost < best_cost) {
          best_cost = cost;
          best = MatvecPlan{nt, wx, wy, ntx, nty, nzc_eff, zc, matvec_smem(nt, wx, wy)};
        }
        if (ctas > 8 * slots) break;
      }
    }
  }
  return best;
}

cudaError_t launch_matvec(const MatvecPlan& pl, MatvecParams P, const Modal& M, cudaStream_t s) {
  P.wx = pl.wx;
  P.wy = pl.wy;
  P.ntx = pl.ntx;
  P.zc = pl.zc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_matvec<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
  dim3 grid(pl.ntx * pl.nty, pl.nzc);
  k_matvec<256><<<grid, 256, pl.smem, s>>>(P, M);
  return cudaGetLastError();
}

}  // namespace tvb
