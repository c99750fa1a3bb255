// K1: assembly-free hex stiffness matvec  y = M_out * sum_e occ_e P_e^T k0 P_e * u
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
//  * node planes of u and occupancy layers are staged into shared-memory rings
//    with cp.async, kAhead planes ahead of the compute (enough bytes in flight
//    per SM to cover DRAM latency); one __syncthreads per z-step.
//  * k0 is applied in the Walsh-Hadamard mode basis of the cube: butterflies
//    H3^T, a 33-flop mode-space operator (8 structural constants), butterflies
//    H3 -- ~150 fp64 ops per element instead of 576 FMAs.
//  * the bottom face's xy-transform is reused from the previous step and the
//    z-direction node sum is done in mode space in registers ("carry"); the
//    x/y node sums go through one double-buffered shared-memory exchange.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "matvec.cuh"

namespace tvb {

// Element operator in the Walsh-Hadamard mode basis (binary local numbering,
// modal DOF 3*mode + axis). The 45 nonzeros of Mh (gen_modal.py) take only 8
// structurally distinct values (cube symmetry, any E, nu, h); with
// s = occ * {k0-k1, k1, k2, k3, k4, k5-k6, k6, k7} the product is 33 flops:
//   {3,7,14} and {11,16,18}: diagonal + rank-one coupling,
//   {4,6} {5,12} {8,13}: all four entries equal (shear pairs),
//   {9,20} {10,17} {15,19}: symmetric 2x2, {21},{22},{23}: diagonal.
__device__ __forceinline__ void modal_apply8(const double (&s)[8], const double (&c)[24], double (&g)[24]) {
  g[0] = g[1] = g[2] = 0.0;
  const double tA = s[1] * ((c[3] + c[7]) + c[14]);
  g[3] = fma(s[0], c[3], tA);
  g[7] = fma(s[0], c[7], tA);
  g[14] = fma(s[0], c[14], tA);
  g[4] = g[6] = s[2] * (c[4] + c[6]);
  g[5] = g[12] = s[2] * (c[5] + c[12]);
  g[8] = g[13] = s[2] * (c[8] + c[13]);
  g[9] = fma(s[3], c[9], s[4] * c[20]);
  g[20] = fma(s[3], c[20], s[4] * c[9]);
  g[10] = fma(s[3], c[10], s[4] * c[17]);
  g[17] = fma(s[3], c[17], s[4] * c[10]);
  g[15] = fma(s[3], c[15], s[4] * c[19]);
  g[19] = fma(s[3], c[19], s[4] * c[15]);
  const double tB = s[6] * ((c[11] + c[16]) + c[18]);
  g[11] = fma(s[5], c[11], tB);
  g[16] = fma(s[5], c[16], tB);
  g[18] = fma(s[5], c[18], tB);
  g[21] = s[7] * c[21];
  g[22] = s[7] * c[22];
  g[23] = s[7] * c[23];
}

// smem row stride (doubles) of a staged node plane: 3*wx + 16 makes the
// element-column gather conflict-free even where a warp wraps to the next
// tile row (stride == 3*wx mod 16 in 8-byte words).
__host__ __device__ inline int plane_row_stride(int wx) { return 3 * wx + 16; }

__device__ __forceinline__ void xy_forward(double (&f)[12]) {
  // face node (ox,oy) -> face mode (mx,my); per bit: (v0,v1) -> (v0+v1, v1-v0)
#pragma unroll
  for (int bit = 1; bit < 4; bit <<= 1)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (b & bit) continue;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double v0 = f[3 * b + a], v1 = f[3 * (b | bit) + a];
        f[3 * b + a] = v0 + v1;
        f[3 * (b | bit) + a] = v1 - v0;
      }
    }
}

__device__ __forceinline__ void xy_inverse(double (&f)[12]) {
  // face mode -> face node; per bit: (g0,g1) -> (g0-g1, g0+g1)
#pragma unroll
  for (int bit = 1; bit < 4; bit <<= 1)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      if (b & bit) continue;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double g0 = f[3 * b + a], g1 = f[3 * (b | bit) + a];
        f[3 * b + a] = g0 - g1;
        f[3 * (b | bit) + a] = g0 + g1;
      }
    }
}

// TVB_MATVEC_DEBUG (compile-time): enables the TVB_MV_DEBUG stage switches
// of the tuning experiments; compiled out otherwise (each was a per-step
// uniform branch in the hot loop)
#ifdef TVB_MATVEC_DEBUG
#define TVB_MV_DBG(P) ((P).debug)
#else
#define TVB_MV_DBG(P) 0
#endif

constexpr int kStage = 4;   // max staged node-plane doubles per thread ((wy+1)*3(wx+1) <= kStage*NT)
constexpr int kXcPad = 64;  // exchange rows past NT read (harmlessly) by edge threads
// doubles per thread slot of the face exchange (9 used): 80-byte slots keep
// every 16-byte access aligned and a quarter-warp of them bank-conflict free
constexpr int kXw = 10;
constexpr int kAhead = 4;   // node planes in flight ahead of the compute (cp.async groups)
constexpr int kRing = kAhead + 1;

// One CTA = a (wx-1) x (wy-1) column of owned nodes over z-planes [kz0, kz1).
// Step k (element layer k between node planes k and k+1), per thread:
//   gather the 4 top-face nodes of its element column from staged plane k+1,
//   xy-transform them (the bottom face's transform is kept from step k-1),
//   apply the element operator in mode space, z-accumulate the node sums of
//   plane k in mode space (carry), and exchange the 3 non-owned face nodes of
//   plane k through shared memory; the owner thread finishes the node.
// WX, WY > 0: the tile shape as compile-time constants (every index and
// shared-memory offset of the hot loop becomes an immediate); 0: runtime shape.
// MASKIN: zero the fixed DOFs of u as it is staged (the public API's
// TVB_MASK_IN, fea.py:55-57): each thread loads the fixed-axis flags of the
// doubles it stages with the copy and clears them in shared memory once they
// have landed, before the step barrier -- no separate masked copy of u.
template <int NT, int MINB, bool DOT, bool MASKOUT, int WX = 0, int WY = 0, bool MASKIN = false>
__global__ void __launch_bounds__(NT, MINB) k_matvec(MatvecParams P, Modal M) {
  pdl_entry();
  extern __shared__ double smem[];
  if (P.stop != nullptr && *P.stop) return;
  const Grid& G = P.g;
  const int wx = WX > 0 ? WX : P.wx, wy = WY > 0 ? WY : P.wy;
  const int PW = wx + 1, PH = wy + 1;
  const int S = plane_row_stride(wx);
  const int PS = PH * S;   // doubles per staged node plane
  const int OS = wx * wy;  // doubles per staged occupancy layer
  const long long plane_stride = 3LL * G.px * G.py;
  const long long layer_stride = (long long)G.nx * G.ny;

  double* Up = smem;                  // [kRing][PS] node plane ring
  double* Oc = Up + kRing * PS;       // [kRing][OS] occupancy layer ring
  double* Xc = smem + ((kRing * PS + kRing * OS + 1) & ~1);  // [2][NT + kXcPad][kXw] face exchange (16-B aligned)
  const int XS = kXw * (NT + kXcPad);
  double* red = Xc + 2 * XS;
  // [kStage][NT] staging lists: (smem byte offset, in-plane global byte offset)
  int2* st_list = reinterpret_cast<int2*>(red + NT / 32 + 1);

  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const bool active = t < wx * wy;
  const int tx = active ? t % wx : 0, ty = active ? t / wx : 0;
  double dot = 0.0;

  // Balanced persistent split: the work is tiles x pz node planes, flattened
  // tile-major; CTA b takes the contiguous range [w0, w1) and walks it as
  // (tile, plane range) pieces.
  const int zlo = P.zlo, zhi = P.zhi < 0 ? G.pz : P.zhi, npl = zhi - zlo;  // output node planes
  // Every piece pays a fixed overhead (its halo layer and the fill of the
  // staging pipeline, ~piece_cost plane-steps), and a range that crosses a
  // tile boundary pays it twice: split a virtual length in which each tile is
  // preceded by piece_cost overhead units, so such CTAs get fewer planes.
  const long long VT = npl + P.piece_cost, V = (long long)P.ntiles * VT;
  auto to_work = [&](long long v) {
    const long long tl = v / VT, r = v - tl * VT;
    return tl * npl + (r > P.piece_cost ? r - P.piece_cost : 0);
  };
  const long long w0 = to_work(V * blockIdx.x / gridDim.x), w1 = to_work(V * (blockIdx.x + 1) / gridDim.x);
  for (long long w = w0; w < w1;) {
    const int tile = (int)(w / npl);
    const int kz0 = zlo + (int)(w % npl);
    const int kz1 = (int)min((long long)zhi, kz0 + (w1 - w));  // owned node planes [kz0, kz1)
    w += kz1 - kz0;
    const int x0 = (tile % P.ntx) * (wx - 1);
    const int y0 = (tile / P.ntx) * (wy - 1);
    const bool owner = active && tx < wx - 1 && ty < wy - 1 && (x0 + tx) < G.px && (y0 + ty) < G.py;
    __syncthreads();  // previous piece fully consumed the rings
    // parts of a staged row inside the grid: node doubles [r_lo, r_hi), element columns [e_lo, e_hi)
    const int r_lo = 3 * max(0, 1 - x0);
    const int r_hi = 3 * min(PW, G.px - x0 + 1);
    const int e_lo = max(0, 1 - x0), e_hi = min(wx, G.nx - x0 + 1);
    // zero the staged halo outside the grid once (those slots are never written again)
    for (int jy = warp; jy < PH; jy += NT / 32) {
      const int gy = y0 - 1 + jy;
      const bool yin = gy >= 0 && gy < G.py;
      for (int r = lane; r < 3 * PW; r += 32)
        if (!yin || r < r_lo || r >= r_hi)
          for (int b = 0; b < kRing; ++b) Up[b * PS + jy * S + r] = 0.0;
    }
    for (int jy = warp; jy < wy; jy += NT / 32) {
      const int ey = y0 - 1 + jy;
      const bool yin = ey >= 0 && ey < G.ny;
      for (int j = lane; j < wx; j += 32)
        if (!yin || j < e_lo || j >= e_hi)
          for (int b = 0; b < kRing; ++b) Oc[b * OS + jy * wx + j] = 0.0;
    }

    // Per-thread staging assignment, fixed for all planes of the piece: the
    // in-grid doubles of a staged node plane (rows x [r_lo, r_hi)) are dealt
    // out round-robin, thread t taking elements t, t + NT, ...; each keeps the
    // smem byte offset and the in-plane global offset of its <= kStage
    // elements, so staging one plane is kStage predicated cp.async per thread
    // (no per-plane row/column index arithmetic). Likewise one occupancy
    // element per thread (wx * wy <= NT).
    // (kept in shared memory, [kStage][NT] each: registers are the kernel's
    // limiting resource)
    int ncnt = 0;
    {
      const int rw = r_hi - r_lo;
      const int jy_lo = max(0, 1 - y0), jy_hi = min(PH, G.py - y0 + 1);
      const int nval = (jy_hi - jy_lo) * rw;
#pragma unroll
      for (int q = 0; q < kStage; ++q) {
        const int i = t + q * NT;
        if (i < nval) {
          const int jy = jy_lo + i / rw, r = r_lo + i % rw;
          // MASKIN: the staged double's axis (r = 3 * node + axis) rides in the low bits of the smem byte offset
          st_list[q * NT + t] = make_int2(8 * (jy * S + r) | (MASKIN ? r % 3 : 0),
                                          8 * (3 * G.px * (y0 - 1 + jy) + 3 * (x0 - 1) + r));
          ncnt = q + 1;
        }
      }
    }
    unsigned ooff = 0u;
    int oeoff = 0;
    bool has_occ = false;
    {
      const int ew = e_hi - e_lo;
      const int ey_lo = max(0, 1 - y0), ey_hi = min(wy, G.ny - y0 + 1);
      if (t < (ey_hi - ey_lo) * ew) {
        const int jy = ey_lo + t / ew, j = e_lo + t % ew;
        ooff = (unsigned)(8 * (jy * wx + j));
        oeoff = G.nx * (y0 - 1 + jy) + (x0 - 1) + j;
        has_occ = true;
      }
    }
    const unsigned up_s = (unsigned)__cvta_generic_to_shared(Up), oc_s = (unsigned)__cvta_generic_to_shared(Oc);
    // MASKIN: FIFO of 4-bit masks (bit q = "list entry q of this thread is a fixed DOF"), one per staged plane
    // in plane order: a plane's mask is pushed when its copies are issued and popped two steps later, when they
    // have landed -- at fixed nibble positions (see the z-loop), so no variable shifts. flp: flags of the next
    // plane to be staged (planes are staged in consecutive order).
    unsigned pend = 0u;
    const long long plane_nodes = (long long)G.px * G.py;
    const uint8_t* flp = MASKIN ? P.fixed + plane_nodes * (kz0 - 1) : nullptr;

    // stage node plane k and occupancy layer k into ring slot sl (zero-filled outside the grid)
    auto load_layer = [&](int k, int sl, int nib) {  // nib: FIFO position of this plane's mask (MASKIN)
      if (k >= 0 && k < G.pz) {
        const char* src = reinterpret_cast<const char*>(P.u + plane_stride * k);
        const unsigned base = up_s + (unsigned)(8 * sl * PS);
        // all list entries first (unused slots are read but never followed),
        // then the predicated copies: no LDS -> LDGSTS pairs in the stream
        int2 e[kStage];
#pragma unroll
        for (int q = 0; q < kStage; ++q) e[q] = st_list[q * NT + t];
#pragma unroll
        for (int q = 0; q < kStage; ++q)
          if (q < ncnt) cp_async8_s(base + (MASKIN ? (unsigned)e[q].x & ~7u : (unsigned)e[q].x), src + e[q].y);
        if (MASKIN) {
          unsigned bits = 0u;
#pragma unroll
          for (int q = 0; q < kStage; ++q)
            if (q < ncnt)  // node = in-plane byte offset / 24, axis from the entry's low bits
              bits |= (((unsigned)flp[(unsigned)e[q].y / 24u] >> ((unsigned)e[q].x & 3u)) & 1u) << q;
          pend |= bits << (4 * nib);
        }
      } else {  // halo plane above / below the grid (first / last piece only)
        double* dst = Up + sl * PS;
#pragma unroll
        for (int q = 0; q < kStage; ++q)
          if (q < ncnt) dst[st_list[q * NT + t].x / 8] = 0.0;
      }
      if (MASKIN) flp += plane_nodes;
      if (has_occ) {
        if (k >= 0 && k < G.nz) cp_async8_s(oc_s + (unsigned)(8 * sl * OS) + ooff, P.occ + layer_stride * k + oeoff);
        else Oc[sl * OS + ooff / 8] = 0.0;
      }
      cp_async_commit();
    };

    const int j00 = ty * S + 3 * tx;
    auto gather_face = [&](int sl, double (&f)[12]) {
      const double* pl = Up + sl * PS + j00;
  #pragma unroll
      for (int b = 0; b < 4; ++b)
  #pragma unroll
        for (int a = 0; a < 3; ++a) f[3 * b + a] = pl[(b >> 1) * S + 3 * (b & 1) + a];
    };

    // MASKIN: clear this thread's fixed staged doubles of ring slot sl (after they landed)
    auto apply_mask = [&](int sl, unsigned bits) {
      if (!MASKIN) return;
      if (bits == 0u) return;
      double* dst = Up + sl * PS;
#pragma unroll
      for (int q = 0; q < kStage; ++q)
        if ((bits >> q) & 1u) dst[st_list[q * NT + t].x / 8] = 0.0;
    };

    double carry[12];
  #pragma unroll
    for (int i = 0; i < 12; ++i) carry[i] = 0.0;
    const long long own_node = G.node(min(x0 + tx, G.px - 1), min(y0 + ty, G.py - 1), kz0);
    double* yrow = P.y + 3 * own_node;
    const uint8_t* frow = MASKOUT ? P.fixed + own_node : nullptr;
    // fixed-DOF flags of the owned node, loaded one output plane ahead (the
    // byte load's latency is covered by a whole z-step)
    uint8_t fnext = (MASKOUT && owner && kz0 < kz1) ? *frow : (uint8_t)0;

    // sk = ring slot of plane / layer k; plane k+1 sits in sk+1, plane k+kAhead in sk-1 (mod kRing)
    auto step = [&](int k, int sk, const double (&bot)[12], double (&top)[12]) {
      const int sk1 = sk == kRing - 1 ? 0 : sk + 1, skl = sk == 0 ? kRing - 1 : sk - 1;
      if (k + kAhead <= kz1 && !(TVB_MV_DBG(P) & 2)) load_layer(k + kAhead, skl, 2);  // FIFO: [k+2, k+3] pending
      else cp_async_commit();  // keep one group per step
      gather_face(sk1, top);
      xy_forward(top);
      const double occ_e = Oc[sk * OS + (active ? t : 0)];
      double c[24];
  #pragma unroll
      for (int i = 0; i < 12; ++i) {
        c[i] = bot[i] + top[i];
        c[12 + i] = top[i] - bot[i];
      }
      double sc[8];
  #pragma unroll
      for (int i = 0; i < 8; ++i) sc[i] = occ_e * M.k[i];
      double gm[24];
      modal_apply8(sc, c, gm);
      double face[12];
  #pragma unroll
      for (int i = 0; i < 12; ++i) {
        face[i] = (gm[i] - gm[12 + i]) + carry[i];
        carry[i] = gm[i] + gm[12 + i];
      }
      const bool out = k >= kz0;
      double* xs = Xc + (k & 1) * XS;
      if (out) {
        xy_inverse(face);
        // nodes (0,0), (1,0), (0,1): five 16-byte stores (slot word 9 unused);
        // 8-byte accesses at an 80-byte stride would conflict 2-way
        double2* x2 = reinterpret_cast<double2*>(xs + kXw * t);
  #pragma unroll
        for (int i = 0; i < 4; ++i) x2[i] = make_double2(face[2 * i], face[2 * i + 1]);
        x2[4] = make_double2(face[8], 0.0);
      }
      // dot epilogue operand: u at the owned node, read from staged plane k
      // BEFORE the barrier (after it, a faster thread may already refill the
      // slot with plane k + kRing)
      double uo[3];
      if (DOT) {
#pragma unroll
        for (int a = 0; a < 3; ++a) uo[a] = Up[sk * PS + j00 + S + 3 + a];
      }
      cp_async_wait_group<kAhead - 2>();  // plane k+2 (and occupancy k+2) landed
      if (MASKIN) {  // pop plane k+2's mask
        if (k + 2 <= kz1) apply_mask(sk == kRing - 2 ? 0 : (sk == kRing - 1 ? 1 : sk + 2), pend & 15u);
        pend >>= 4;
      }
      if (!(TVB_MV_DBG(P) & 1)) __syncthreads();
      if (out) {
        // node (x0+tx, y0+ty) = local (1,1) of this column, (0,1) of column
        // tx+1, (1,0) of column ty+1 and (0,0) of column (tx+1, ty+1).
        const double* e10 = xs + kXw * (t + 1);
        const double* e01 = xs + kXw * (t + wx);
        const double* e11 = xs + kXw * (t + wx + 1);
        const double2 a67 = *reinterpret_cast<const double2*>(e10 + 6);
        const double2 a89 = *reinterpret_cast<const double2*>(e10 + 8);
        const double2 b23 = *reinterpret_cast<const double2*>(e01 + 2);
        const double2 b45 = *reinterpret_cast<const double2*>(e01 + 4);
        const double2 c01 = *reinterpret_cast<const double2*>(e11);
        const double2 c23 = *reinterpret_cast<const double2*>(e11 + 2);
        const double n10[3] = {a67.x, a67.y, a89.x}, n01[3] = {b23.y, b45.x, b45.y}, n11[3] = {c01.x, c01.y, c23.x};
        double v[3];
  #pragma unroll
        for (int a = 0; a < 3; ++a) v[a] = ((face[9 + a] + n10[a]) + n01[a]) + n11[a];
        if (owner) {
          const uint8_t fx = MASKOUT ? fnext : 0;
  #pragma unroll
          for (int a = 0; a < 3; ++a) {
            double w = ((fx >> a) & 1) ? 0.0 : v[a];
            if (WX == 0 && P.accumulate) w += yrow[a];  // y += A u: runtime-shape kernel only (launch_fixed_shape)
            if (!(TVB_MV_DBG(P) & 4)) yrow[a] = w;
            if (DOT) dot = fma(uo[a], w, dot);
          }
        }
        yrow += plane_stride;
        if (MASKOUT) {
          frow += (long long)G.px * G.py;
          if (owner && k + 1 < kz1) fnext = *frow;
        }
      }
    };

    const int s0 = (kz0 - 1 + kRing) % kRing;  // slot of the first staged plane kz0 - 1
#pragma unroll
    for (int j = 0; j < kAhead; ++j) {
      if (kz0 - 1 + j <= kz1) load_layer(kz0 - 1 + j, (s0 + j) % kRing, j);
      else cp_async_commit();
    }
    cp_async_wait_group<kAhead - 2>();
    if (MASKIN) {  // planes kz0 - 1 and kz0 landed: pop their masks
      apply_mask(s0, pend & 15u);
      apply_mask(s0 == kRing - 1 ? 0 : s0 + 1, (pend >> 4) & 15u);
      pend >>= 8;
    }
    __syncthreads();
    double fa[12], fb[12];
    gather_face(s0, fa);
    xy_forward(fa);
    int sk = s0;
    for (int k = kz0 - 1; k < kz1; k += 2) {
      step(k, sk, fa, fb);
      sk = sk == kRing - 1 ? 0 : sk + 1;
      if (k + 1 < kz1) step(k + 1, sk, fb, fa);
      sk = sk == kRing - 1 ? 0 : sk + 1;
    }
  }
  if (DOT) {
    const double sum = block_sum(dot, red);
    if (t == 0) P.dot_partial[blockIdx.x] = sum;
  }
}

// Host-side launch planning -------------------------------------------------

static size_t matvec_smem(int nt, int wx, int wy) {
  const int PS = (wy + 1) * plane_row_stride(wx);
  return sizeof(double) * (kRing * (size_t)PS + kRing * (size_t)wx * wy + 1 + 2 * kXw * (size_t)(nt + kXcPad) + nt / 32 + 1) +
         2 * sizeof(int) * kStage * (size_t)nt;
}

static int ctas_per_sm(int nt) { return nt == 256 ? 2 : 1; }

// Tile choice for the persistent balanced split: per-SM time ~ (tile work of
// all pz planes + one halo layer per piece) x the CTA's warps (all NT/32 warps
// stage, exchange and synchronise, even where a tile leaves threads idle) /
// CTAs. Redundant halo columns and empty tile parts count as work; ties go to
// the longer staged rows (larger wx). Measured against the previous
// active-warp count (which tied 22x10 with 24x10 at C4): C4 39.9 -> 36.9 us,
// C5 197.6 -> 187-193 us, C2 unchanged (23x11).
// TVB_MV_PLAN="nt,wx,wy[,ctas]" overrides (tuning sweeps).
MatvecPlan plan_matvec(const Grid& g, int num_sms) {
  if (const char* e = getenv("TVB_MV_PLAN")) {
    int nt = 0, wx = 0, wy = 0, nc = 0;
    const int got = sscanf(e, "%d,%d,%d,%d", &nt, &wx, &wy, &nc);
    if (got >= 3 && (nt == 256 || nt == 384 || nt == 512) && wx * wy <= nt && wx >= 2 && wy >= 2) {
      const int ntx = (g.px + wx - 2) / (wx - 1), nty = (g.py + wy - 2) / (wy - 1);
      if (got < 4 || nc < 1) nc = num_sms * ctas_per_sm(nt);
      return MatvecPlan{nt, wx, wy, ntx, nty, nc, matvec_smem(nt, wx, wy)};
    }
  }
  MatvecPlan best{};
  double best_cost = 1e300;
  auto plan_cost = [&](int nt, int wx, int wy, MatvecPlan& out) {
    const int nc = num_sms * ctas_per_sm(nt);
    const int ntx = (g.px + wx - 2) / (wx - 1);
    const int nty = (g.py + wy - 2) / (wy - 1);
    const double tiles = (double)ntx * nty;
    const int warps = nt / 32;
    const double pieces = std::max(tiles, (double)nc) + nc;  // upper bound of pieces
    out = MatvecPlan{nt, wx, wy, ntx, nty, nc, matvec_smem(nt, wx, wy)};
    return (tiles * g.pz + 1.5 * pieces) * warps / nc;
  };
  // wx < 20 loses to short staged rows and frequent warp row-wraps (measured
  // sweeps, profiles/README.md); nt = 384 / 512 never won.
  for (int nt : {256, 384}) {
    for (int wx = 20; wx <= 48; ++wx) {
      for (int wy = 3; wx * wy <= nt; ++wy) {
        if (wx * wy < nt - 48) continue;
        MatvecPlan pl;
        const double cost = plan_cost(nt, wx, wy, pl);
        if (cost < best_cost - 1e-9 || (cost <= best_cost + 1e-9 && wx > best.wx)) {
          best_cost = cost;
          best = pl;
        }
      }
    }
  }
  // The tile shapes compiled with constant geometry (launch_fixed_shape) run
  // ~1.45x faster than the runtime-shape kernel at equal tiling (C4: 25x10
  // 34.9 us, 24x10 51.2 us; 100^3: 47.3 vs 53.1 us; profiles/README.md), so a
  // grid whose best generic tiling is not one of them still takes the best
  // compiled shape unless the generic tiling is predicted to save more.
  if (getenv("TVB_MV_GENERIC") == nullptr) {
    static const int fixed_shapes[4][2] = {{23, 11}, {25, 10}, {28, 9}, {42, 6}};
    MatvecPlan fbest{};
    double fcost = 1e300;
    for (const auto& sh : fixed_shapes) {
      MatvecPlan pl;
      const double cost = plan_cost(256, sh[0], sh[1], pl);
      if (cost < fcost) {
        fcost = cost;
        fbest = pl;
      }
    }
    if (fcost <= 1.4 * best_cost) return fbest;
  }
  return best;
}

template <int NT, int MINB, int WX = 0, int WY = 0>
static void set_smem_attr(size_t bytes) {
  if (WX == 0) {
    cudaFuncSetAttribute(k_matvec<NT, MINB, false, false, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_matvec<NT, MINB, false, true, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_matvec<NT, MINB, true, false, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_matvec<NT, MINB, true, true, 0, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  if (WX != 0) {  // fused input mask with constant geometry (no-dot variants)
    cudaFuncSetAttribute(k_matvec<NT, MINB, false, false, WX, WY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(k_matvec<NT, MINB, false, true, WX, WY, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  cudaFuncSetAttribute(k_matvec<NT, MINB, false, false, WX, WY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(k_matvec<NT, MINB, false, true, WX, WY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(k_matvec<NT, MINB, true, false, WX, WY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  cudaFuncSetAttribute(k_matvec<NT, MINB, true, true, WX, WY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int NT, int MINB, int WX = 0, int WY = 0>
static void launch_nt(dim3 grid, size_t smem, cudaStream_t s, const MatvecParams& P, const Modal& M) {
  const bool dot = P.dot_partial != nullptr, mo = P.mask_out && P.fixed != nullptr;
  if (P.mask_in && P.fixed != nullptr) {  // fused input mask (with the dot epilogue: runtime-shape kernel only)
    if (!dot && WX != 0) {
      if (mo) launch_k(k_matvec<NT, MINB, false, true, WX, WY, true>, grid, NT, smem, s, P, M);
      else launch_k(k_matvec<NT, MINB, false, false, WX, WY, true>, grid, NT, smem, s, P, M);
      return;
    }
    if (dot && mo) launch_k(k_matvec<NT, MINB, true, true, 0, 0, true>, grid, NT, smem, s, P, M);
    else if (dot) launch_k(k_matvec<NT, MINB, true, false, 0, 0, true>, grid, NT, smem, s, P, M);
    else if (mo) launch_k(k_matvec<NT, MINB, false, true, 0, 0, true>, grid, NT, smem, s, P, M);
    else launch_k(k_matvec<NT, MINB, false, false, 0, 0, true>, grid, NT, smem, s, P, M);
    return;
  }
  if (dot && mo) launch_k(k_matvec<NT, MINB, true, true, WX, WY>, grid, NT, smem, s, P, M);
  else if (dot) launch_k(k_matvec<NT, MINB, true, false, WX, WY>, grid, NT, smem, s, P, M);
  else if (mo) launch_k(k_matvec<NT, MINB, false, true, WX, WY>, grid, NT, smem, s, P, M);
  else launch_k(k_matvec<NT, MINB, false, false, WX, WY>, grid, NT, smem, s, P, M);
}

// tile shapes compiled with constant geometry: the planner's choices for the
// BASELINE grids (C2 23x11, C4 25x10, C5 28x9, C1 / C3 42x6)
static bool launch_fixed_shape(const MatvecPlan& pl, dim3 grid, cudaStream_t s, const MatvecParams& P, const Modal& M) {
  static const bool off = getenv("TVB_MV_GENERIC") != nullptr;
  if (off || pl.nt != 256 || P.accumulate) return false;
#define TVB_SHAPE(X, Y)                                  \
  if (pl.wx == X && pl.wy == Y) {                        \
    launch_nt<256, 2, X, Y>(grid, pl.smem, s, P, M);     \
    return true;                                         \
  }
  TVB_SHAPE(23, 11)
  TVB_SHAPE(25, 10)
  TVB_SHAPE(28, 9)
  TVB_SHAPE(42, 6)
#undef TVB_SHAPE
  return false;
}

cudaError_t launch_matvec(const MatvecPlan& pl, MatvecParams P, const Modal& M, cudaStream_t s) {
  P.wx = pl.wx;
  P.wy = pl.wy;
  P.ntx = pl.ntx;
  P.ntiles = pl.ntx * pl.nty;
  if (const char* d = getenv("TVB_MV_DEBUG")) P.debug = atoi(d);
  // measured (scripts/gpu_piece_cost.sh, same box): charge 3 vs 0 -> C2(a) K.u 53.0 -> 51.0 us (warm),
  // C4 DPCG 215.0 -> 212.0, C3 117.3 -> 114.1 us per iteration; 2 / 4 / 6 within 0.5 us of 3
  static const int piece_cost = getenv("TVB_MV_PIECE_COST") ? atoi(getenv("TVB_MV_PIECE_COST")) : 3;
  P.piece_cost = piece_cost < 0 ? 0 : piece_cost;
  static bool attr_set = false;
  if (!attr_set) {
    set_smem_attr<256, 2>(110 * 1024);
    set_smem_attr<256, 2, 23, 11>(110 * 1024);
    set_smem_attr<256, 2, 25, 10>(110 * 1024);
    set_smem_attr<256, 2, 28, 9>(110 * 1024);
    set_smem_attr<256, 2, 42, 6>(110 * 1024);
    set_smem_attr<384, 1>(220 * 1024);
    set_smem_attr<512, 1>(220 * 1024);
    attr_set = true;
  }
  dim3 grid(pl.nctas);
  if (launch_fixed_shape(pl, grid, s, P, M)) return cudaGetLastError();
  if (pl.nt == 256) launch_nt<256, 2>(grid, pl.smem, s, P, M);
  else if (pl.nt == 384) launch_nt<384, 1>(grid, pl.smem, s, P, M);
  else launch_nt<512, 1>(grid, pl.smem, s, P, M);
  return cudaGetLastError();
}

}  // namespace tvb
