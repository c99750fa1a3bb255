/*
 * topovox_b200.h -- C-ABI of the B200-native voxel FEA hot path
 * (libtopovox_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the reference package `topovox`
 * (/root/reference/pkg/src/topovox). Each entry point names the reference
 * function it replaces. Conventions:
 *   - every pointer argument named d_* is DEVICE memory owned by the caller;
 *     h_* arguments are host memory; nothing here allocates device memory
 *     except the solve drivers' internal CUDA graph objects;
 *   - node vectors are f64[3*Nn] interleaved per node (reference numbering,
 *     topovox/mesh.py:3-6), element vectors are f64[Ne];
 *   - d_nflags is a u8[Nn] node flag array: bit a (0..2) = DOF 3n+a fixed,
 *     bit 3 = structural node (built by tvb_node_flags);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     stream-ordered and asynchronous unless stated otherwise;
 *   - every call returns a status code (TVB_OK = 0); reductions are
 *     deterministic (fixed-order two-stage trees, no float atomics).
 */
#ifndef TOPOVOX_B200_H
#define TOPOVOX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mapped to topovox/errors.py exception types by the Python host) */
#define TVB_OK 0
#define TVB_BAD_DIMS 1        /* DimensionMismatch / BadDimension */
#define TVB_CUDA_ERROR 2
#define TVB_NOT_SPD 3         /* coarse matrix not SPD (topovox/fea.py:202-205) */
#define TVB_NO_CONVERGENCE 4  /* NoConvergence (topovox/fea.py:292-297) */
#define TVB_SINGULAR 5        /* SingularSystem (topovox/fea.py:246-247) */
#define TVB_BAD_ARG 6
#define TVB_WORKSPACE 7       /* workspace too small */

/* matvec flags */
#define TVB_MASK_IN 1     /* zero fixed DOFs of u before applying (fea.py:55-57) */
#define TVB_MASK_OUT 2    /* zero fixed DOFs of the result (fea.py:63-64) */
#define TVB_ACCUMULATE 4  /* out += K u (numba seam semantics) instead of out = K u */

int tvb_version(void);
const char* tvb_last_error(void);

/* Element stiffness k0 (24x24 row-major, host) -> the 45 mode-space
 * coefficients the matvec consumes. Fails (TVB_BAD_ARG) if k0 is not the
 * stiffness of an isotropic cube (the mode pattern check). Host only. */
int tvb_modal_from_k0(const double* h_k0, double* h_mh45);

/* a3: K.u  -- replaces apply_block24 (topovox/backends/numba_kernels.py:12-28)
 * as called by StiffnessOperator.apply (topovox/fea.py:49-65).
 * d_dot (optional, device scalar) receives sum(u_masked . out) over all nodes.
 * d_ws: workspace of tvb_matvec_ws_bytes() bytes (NULL allowed when d_dot is NULL). */
size_t tvb_matvec_ws_bytes(int nx, int ny, int nz);
int tvb_matvec(int nx, int ny, int nz, const double* h_mh45, const double* d_u, double* d_out,
               const double* d_occ, const uint8_t* d_nflags, int flags, double* d_dot, void* d_ws,
               size_t ws_bytes, void* stream);

/* diagnostics: the launch plan tvb_matvec uses for this grid:
 * out7 = {threads, wx, wy, tiles_x, tiles_y, persistent CTAs, 0} */
int tvb_matvec_plan(int nx, int ny, int nz, int* h_out7);

/* a3 with HOST buffers (the reference's StiffnessOperator.apply takes and
 * returns numpy arrays, topovox/fea.py:49-65): out = K u with h_u / h_out in
 * host memory (pinned for overlap), pipelined over `slabs` z-slabs of node
 * planes (<= 0: default 6) so the host->device copy, the multiply and the
 * device->host copy of successive slabs overlap. flags: MASK_IN / MASK_OUT
 * (no ACCUMULATE). d_ws >= tvb_matvec_host_ws_bytes(). Synchronous. */
size_t tvb_matvec_host_ws_bytes(int nx, int ny, int nz);
int tvb_matvec_host(int nx, int ny, int nz, const double* h_mh45, const double* h_u, double* h_out,
                    const double* d_occ, const uint8_t* d_nflags, int flags, int slabs, void* d_ws, size_t ws_bytes,
                    void* stream);
/* A stream of nvec host vectors (h_u[v] -> h_out[v]) through the same slab
 * pipeline, double-buffered on the device so vector v's host->device copies
 * overlap vector v-1's device->host copies. Synchronous; results bitwise those
 * of tvb_matvec_host. d_ws >= tvb_matvec_host_batch_ws_bytes() (4 vectors). */
size_t tvb_matvec_host_batch_ws_bytes(int nx, int ny, int nz);
int tvb_matvec_host_batch(int nx, int ny, int nz, const double* h_mh45, int nvec, const double* const* h_u,
                          double* const* h_out, const double* d_occ, const uint8_t* d_nflags, int flags, int slabs,
                          void* d_ws, size_t ws_bytes, void* stream);

/* diagnostics: sustained fp64 FMA throughput of this GPU measured live
 * (independent DFMA chains on every SM), in TFLOP/s (2 flops per FMA);
 * the denominator of the north-star fp64 roofline. Synchronous. */
double tvb_fp64_peak_tflops(void* stream);

/* apply_block24_subset (numba_kernels.py:31-46): out += K_subset u using only
 * the listed elements (duplicates count with multiplicity). d_ws: f64[Ne] + i32[Ne]. */
int tvb_matvec_subset(int nx, int ny, int nz, const double* h_mh45, const double* d_u, double* d_out,
                      const long long* d_elems, long long n_elems_listed, const double* d_occ, void* d_ws,
                      size_t ws_bytes, void* stream);

/* a4: diag(K) -- replaces diag_block24 (numba_kernels.py:49-58) as used by
 * StiffnessOperator.diagonal (fea.py:78-85). h_kdiag3 = k0[a,a] for a=0..2.
 * d_diag (optional) receives the diagonal (accumulated if accumulate != 0);
 * d_inv (optional) receives 1/diag on free DOFs and 0 on fixed DOFs;
 * d_zero_free (optional, device int) is incremented for every free DOF with
 * a zero diagonal. */
int tvb_diag(int nx, int ny, int nz, const double* d_occ, const uint8_t* d_nflags, const double* h_kdiag3,
             double* d_diag, int accumulate, double* d_inv, int* d_zero_free, void* stream);

/* node flags from the sorted fixed-DOF list and the occupancy (structural
 * nodes touch an element with occupancy == 1.0, fea.py:119-123). */
int tvb_node_flags(int nx, int ny, int nz, const long long* d_fixed_dofs, long long n_fixed, const double* d_occ,
                   uint8_t* d_nflags, void* stream);

/* deterministic dot product a.b (optionally weighted) -> *d_out */
size_t tvb_reduce_ws_bytes(long long n);
int tvb_dot(const double* d_a, const double* d_b, const double* d_w, long long n, double* d_out, void* d_ws,
            size_t ws_bytes, void* stream);

/* a5: deflation space (DeflationSpace._build_basis, fea.py:113-183).
 * Per block B (id = bx + mx*(by + my*bz), mx = ceil(nx/block), ...):
 *   d_cen  f64[3*Nb]  structural centroid (grid units, relative to block corner)
 *   d_S    f64[36*Nb] raw-mode -> orthonormal transform (0 for dropped columns)
 *   d_keep i32[Nb]    bit j = column j kept.  Nb = mx*my*mz. */
int tvb_defl_build(int nx, int ny, int nz, int block, double h, const double* d_occ, const uint8_t* d_nflags,
                   double* d_cen, double* d_S, int* d_keep, void* stream);
/* restriction yc = W^T y (6*Nb) and prolongation out = W mu / z - W mu */
int tvb_restrict(int nx, int ny, int nz, int block, double h, const uint8_t* d_nflags, const double* d_cen,
                 const double* d_S, const int* d_keep, const double* d_y, double* d_yc, void* stream);
int tvb_prolong(int nx, int ny, int nz, int block, double h, const uint8_t* d_nflags, const double* d_cen,
                const double* d_S, const int* d_keep, const double* d_mu, double* d_out, double* d_nu_ws,
                void* stream);

/* a6: Galerkin coarse operator E = W^T A W (DeflationSpace.prepare, fea.py:185-206)
 * as a symmetrised 27-neighbour 6x6 block stencil d_Es f64[Nb*27*36];
 * dropped/inactive coarse DOFs carry a unit diagonal.
 * d_ws >= tvb_coarse_assemble_ws_bytes(). */
size_t tvb_coarse_assemble_ws_bytes(int nx, int ny, int nz, int block);
int tvb_coarse_assemble(int nx, int ny, int nz, int block, double h, const double* h_mh45, const double* d_occ,
                        const uint8_t* d_nflags, const double* d_cen, const double* d_S, const int* d_keep,
                        double* d_Es, void* d_ws, size_t ws_bytes, void* stream);
/* dense (6Nb x 6Nb, row-major) copy of the block stencil (small coarse spaces) */
int tvb_coarse_dense(int nx, int ny, int nz, int block, const double* d_Es, double* d_E, void* stream);

/* a7: exact coarse solve x = E^-1 y with the nested-dissection block-LDL^T
 * factor (paper_2203_15115_b200/coarse.py builds it). Replaces the dense
 * cho_solve of DeflationSpace.coarse_solve (fea.py:208-211). All d_* are
 * device arrays described in coarse.py; h_* are host arrays. Coarse vectors
 * of tvb_coarse_nd_solve are in ND order (natural block B at ND block
 * d_perm[B]); tvb_pcg_solve applies d_perm inside restriction/prolongation. */
typedef struct tvb_coarse_nd {
  int n_levels;             /* bottom tree heights factored node by node */
  int max_front, max_sep;
  const long long* d_meta;  /* [bottom node][8] s,u,g_off,b_off,sd_off,ud_off,gm_off,0 */
  const int* d_gmap;        /* per node (s+u) x 2: children's update-vector index per front position, -1 = none */
  const double* d_G;        /* per node u x s (G = F_US F_SS^-1) */
  const double* d_B;        /* per node s x (s+u): [F_SS^-1 | -G^T] */
  const int* d_udof;
  double* d_fS;
  double* d_cU;
  const long long* d_fwd_items;  /* [n][10]: the node's meta row (7), 0, row0, row1 */
  const long long* d_bwd_items;
  const long long* h_fwd_ptr;  /* n_levels+1 work-item group offsets */
  const long long* h_bwd_ptr;
  const int* h_fwd_wpr;     /* warps per row per group (1,2,4,8) */
  const int* h_bwd_wpr;
  const int* h_split;       /* per height: 1 = separate front-assembly launch (large fronts) */
  const int* d_asm_nodes;   /* nodes grouped by height */
  const long long* h_asm_ptr;
  int n_top;                /* dense top set (heights >= n_levels), DOFs */
  long long top_off;        /* its ND DOF offset (= 6 Nb - n_top) */
  int top_wpr;
  const double* d_ZT;       /* n_top x n_top inverse of the top Schur complement */
  double* d_fT;
  const int* d_tptr;        /* CSR over top positions of children's update-vector entries */
  const int* d_tidx;
  const int* d_perm;        /* i32[Nb]: natural block -> ND block */
  /* persistent dataflow schedule (one launch per solve); d_items = NULL -> one launch per level */
  const int* d_items;       /* [n_items][12] type, wpr, node, r0, r1, wait_idx, wait_need, done_idx, done_need,
                               rel_begin, rel_end, 0 -- topological order */
  int n_items;
  const int* d_rel;
  unsigned long long* d_cnt;  /* dependency counters, zero-initialised once */
  unsigned long long* d_ctl;  /* [3] next item, CTAs exited, epoch; zero-initialised once */
  const double* d_factor;   /* the single allocation holding G, B, ZT (L2 persistence window) */
  size_t factor_bytes;
  /* multi-RHS scratch: column c of d_fS / d_cU / d_fT at + c * fs_ld / cu_ld / ft_ld;
     max_cols columns allocated (solves of more RHS run in groups of max_cols) */
  long long fs_ld, cu_ld, ft_ld;
  int max_cols;
  /* packed symmetric top (per-level schedule only): top_tiles = ceil(n_top/64)
     > 0 -> d_ZT holds the lower 64x64 tiles (I >= J at I*(I+1)/2 + J,
     row-major, zero-padded) and d_tpart (max_cols x [nt][nt][64], column
     stride tpart_ld) receives the tile partial products; 0 -> dense rows */
  int top_tiles;
  double* d_tpart;
  long long tpart_ld;
} tvb_coarse_nd;
int tvb_coarse_nd_solve(const tvb_coarse_nd* nd, const double* d_y, double* d_x, void* stream);

/* ---- K6: numeric factorisation of the coarse operator (replaces
 * scipy.linalg.cho_factor(E), topovox/fea.py:197-205) ----------------------
 * Fronts of the nested-dissection tree (coarse.py) -- or one front holding
 * all of E for small coarse spaces -- reduced on the device by the block
 * sweep operator (csrc/dense.cu). d_fronts: int64[n][12] records
 * (a_off, nf, s, s_pad, u, blk_off, nchild, child_off, scr_off, ntf, 0, 0);
 * d_children: int64 pairs (child front, gmap offset); d_gmap: int32 parent
 * front position -> child update index or -1; d_blocks: natural block ids of
 * each front (separator, then update set); d_Es: block stencil f64[nb][27][36].
 * d_err is set nonzero when a pivot is not positive (E not SPD). */
typedef struct tvb_front_set {
  const void* d_fronts;
  double* d_pool;
  double* d_scratch;
  const int* d_blocks;
  const long long* d_children;
  const int* d_gmap;
  const double* d_Es;
  int mx, my, mz;
  int* d_err;
} tvb_front_set;

/* assemble and sweep every front of one tree height: d_level_fronts (n_fronts
 * indices), d_tiles (n_tiles (front, I, J) lower 64x64 tiles), d_cols
 * (n_cols (front, K) tile columns), max_steps = max separator tiles */
int tvb_front_level(const tvb_front_set* fs, int n_fronts, const int* d_level_fronts, int n_tiles,
                    const int* d_tiles, int n_cols, const int* d_cols, int max_steps, void* stream);
/* G (u x s) and [Z | -G^T] (s x (s + u)) of a swept front, row-major */
int tvb_front_pack(const tvb_front_set* fs, int front, double* d_G, double* d_B, long long s, long long u,
                   void* stream);
/* Z = F^-1 of a fully swept front of order n: tiles > 0 -> lower 64x64 tiles
 * (tile I (I + 1) / 2 + J, row-major, zero padded), tiles == 0 -> dense rows */
int tvb_front_pack_top(const tvb_front_set* fs, int front, long long n, int tiles, double* d_out, void* stream);

/* a8: (deflated) Jacobi PCG -- replaces solve_static (fea.py:218-299).
 * Synchronous: returns after convergence / the iteration cap. */
typedef struct tvb_pcg_desc {
  int nx, ny, nz;
  double h;
  const double* h_mh45;     /* 45 modal coefficients (host) */
  const double* h_kdiag3;   /* k0[a,a], a = 0..2 (host) */
  const double* d_occ;
  const uint8_t* d_nflags;
  const double* d_f;        /* right-hand side */
  double* d_x;              /* solution (output) */
  void* d_ws;               /* workspace, tvb_pcg_ws_bytes() */
  size_t ws_bytes;
  double tol;
  int max_iters;
  int check_every;          /* iterations per CUDA-graph launch (<= 0: default) */
  /* deflation: block <= 0 or no coarse data -> plain Jacobi PCG */
  int block;
  const double* d_cen;
  const double* d_S;
  const int* d_keep;
  const double* d_coarse;   /* coarse_kind 0: dense inverse f64[nc*nc] */
  int coarse_kind;          /* 0 = dense inverse, 1 = nested dissection (coarse_nd) */
  const tvb_coarse_nd* coarse_nd;
  /* deflated search direction (equal in exact arithmetic):
   *   0 = the reference's recurrence p = z + beta p - W E^-1 (AW)^T z (fea.py:289)
   *   1 = stabilised:               p = z + beta p - W E^-1 W^T (A z + beta A p_old),
   *       which re-imposes W^T A p = 0 every iteration (robust at tol ~1e-12) */
  int projection;
  /* node flags (fixed axes + structural bit) the deflation space was built
   * with (restriction / prolongation); NULL -> d_nflags. The reference builds
   * W from the deflation space's own Dirichlet set and topology (fea.py:113-183) */
  const uint8_t* d_defl_nflags;
  /* outputs */
  int iterations;
  double residual;
  double fnorm;
} tvb_pcg_desc;

size_t tvb_pcg_ws_bytes(int nx, int ny, int nz, int block);
int tvb_pcg_solve(tvb_pcg_desc* desc, void* stream);

/* Multi-RHS batching: nrhs (<= 8) independent solves
 * K x_c = f_c against the operator / deflation space of `desc` (its d_f, d_x
 * and outputs are ignored). One CUDA graph iterates all RHS; the coarse solve
 * reads the factor once per iteration for all of them. Each RHS keeps its own
 * stopping test and iteration count, and its result is bitwise equal to
 * tvb_pcg_solve on it alone. Per-RHS outputs: h_iterations, h_residuals,
 * h_status (0 / NoConvergence / Singular ...). Returns the first failing
 * per-RHS status, or the call's own error (bad arguments, workspace, CUDA),
 * which is then also written to every h_status entry -- no failure path leaves
 * a per-RHS status at 0. d_ws >= tvb_pcg_batch_ws_bytes(). */
size_t tvb_pcg_batch_ws_bytes(int nx, int ny, int nz, int block, int nrhs);
int tvb_pcg_solve_batch(tvb_pcg_desc* desc, int nrhs, const double* const* h_d_f, double* const* h_d_x,
                        int* h_iterations, double* h_residuals, int* h_status, void* stream);

/* a9/a10/a11: element state -- replaces batch_element_state (fea.py:302-309)
 * plus the compliance sensitivity T_J and the p-norm sums
 * (SPEC.md:292-300). Any output may be NULL. d_strains/d_stresses are
 * f64[Ne][6] (Voigt, engineering shear), d_vm/d_tj f64[Ne];
 * d_pn_sums (device f64[2]) <- (sum occ*vm^p, sum occ), which needs
 * d_ws >= tvb_elem_ws_bytes(). */
size_t tvb_elem_ws_bytes(int nx, int ny, int nz);
int tvb_element_state(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                      double* d_strains, double* d_stresses, double* d_vm, double* d_tj, int p, double* d_pn_sums,
                      void* d_ws, size_t ws_bytes, void* stream);
/* a12: adjoint right-hand side d sigma_PN / du, fixed DOFs
 * zeroed; d_pn_sums from tvb_element_state; d_ws >= 48*Ne bytes. */
int tvb_adjoint_rhs(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                    const uint8_t* d_nflags, int p, const double* d_pn_sums, double* d_rhs, void* d_ws,
                    size_t ws_bytes, void* stream);
/* a13: stress sensitivity T_sigma from u and the adjoint */
int tvb_sens_stress(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_lam,
                    const double* d_occ, double* d_ts, void* stream);
/* a14: max|t| and T_L = sum_i w_i t_i / max|t_i| (normalize_field + combine,
 * SPEC.md:375-392). h_fields: host array of k device pointers. */
int tvb_maxabs(const double* d_t, long long n, double* d_out, void* d_ws, size_t ws_bytes, void* stream);
int tvb_combine(int k, const double* const* h_fields, const double* h_w, const double* d_maxabs, long long n,
                double* d_out, void* stream);
/* a15: extract: keep the k largest level-set values among
 * design elements (ties by ascending element index) -> d_occ = 1, other
 * design elements = ersatz, non-design = nondesign. h_state4 (optional,
 * synchronous copy) <- {tau key, -, ties taken, #greater}. */
size_t tvb_select_ws_bytes(long long n);
int tvb_threshold_select(const double* d_ls, const uint8_t* d_design, long long n, long long k, double ersatz,
                         double nondesign, double* d_occ, void* d_ws, size_t ws_bytes,
                         unsigned long long* h_state4, void* stream);
/* extract with casting: flags bit 0 = retain EVERY design
 * element whose value equals the threshold (the superlevel set {v >= tau} of a
 * casting-projected field is undercut-free; the fraction may exceed the
 * target). flags = 0 is tvb_threshold_select. */
int tvb_threshold_select_ex(const double* d_ls, const uint8_t* d_design, long long n, long long k, double ersatz,
                            double nondesign, int flags, double* d_occ, void* d_ws, size_t ws_bytes,
                            unsigned long long* h_state4, void* stream);
/* casting_project (PAPER §3.7): along each element column
 * parallel to axis (0 = x, 1 = y, 2 = z), running minimum moving away from the
 * parting plane. Element layers i >= parting form the +axis mold half, i <
 * parting the -axis half; parting in [0, n_axis] (0 = one +axis half, n_axis =
 * one -axis half). d_in == d_out allowed. Replaces no reference code (the
 * reference ships none); oracle/topovox_oracle.py:casting_project. */
int tvb_casting_project(int nx, int ny, int nz, int axis, int parting, const double* d_in, double* d_out,
                        void* stream);

/* ---- eigen / buckling ---------- */
/* apply_nodal_block8 (topovox/backends/numba_kernels.py:61-76; seam
 * topovox/backends/__init__.py:52): d_out += sum_e P_e^T (B_e (x) I3) P_e d_u
 * with d_blocks f64[Ne][8][8] in the element's local (VTK) node order. */
int tvb_nodal_block8(int nx, int ny, int nz, const double* d_u, double* d_out, const double* d_blocks, void* stream);
/* geometric stiffness K_G u with B_e = sum_k stress[e][k] * Bk[k] (Bk = the
 * 6 Voigt components of geometric_tensor, elements.py:141-153, device
 * f64[6][8][8]); flags: 1 zero fixed DOFs of u, 2 zero fixed rows of the
 * output, 4 accumulate; output scaled by `scale`. */
int tvb_geo_matvec(int nx, int ny, int nz, const double* d_Bk, const double* d_stress, const double* d_u,
                   double* d_out, const uint8_t* d_nflags, int flags, double scale, void* stream);
/* MassOperator: d_mass f64[3*Nn] = coef * sum of the
 * occupancies of the node's elements, coef = rho h^3 / 8. */
int tvb_lumped_mass(int nx, int ny, int nz, double coef, const double* d_occ, double* d_mass, void* stream);
/* eigen_sensitivity T_lambda = sigma(u):eps(u) - omega2rho * occ_e * |u(centroid)|^2
 * (omega2rho = omega_n^2 rho). */
int tvb_eigen_sens(int nx, int ny, int nz, double h, double E, double nu, const double* d_u, const double* d_occ,
                   double omega2rho, double* d_out, void* stream);
/* buckling_sensitivity T_p = u_e^T K^e u_e - lambda u_e^T K_sigma^e u_e with
 * K^e = occ_e k0 (d_k0 device f64[24][24]) and K_sigma = -K_G (compression
 * positive): = occ_e u_e^T k0 u_e + lambda sum_a u_ea^T B_e u_ea. */
int tvb_buckling_sens(int nx, int ny, int nz, const double* d_k0, const double* d_Bk, const double* d_stress,
                      const double* d_u, const double* d_occ, double lambda, double* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOPOVOX_B200_H */
