// Shared definitions for the sm_100a voxel-FEA kernels.
//
// Layout in HBM (all fp64 unless noted), reference numbering
// (topovox/mesh.py:3-6):
//   node vectors   f64[3*Nn]   interleaved (x,y,z) per node, node n = ix + px*(iy + py*iz)
//   element data   f64[Ne]     occupancy, e = ix + nx*(iy + ny*iz)
//   fixed mask     u8[Nn]      bit a set <=> DOF 3n+a is Dirichlet-fixed
// No index table is ever read: every index is arithmetic in (nx, ny, nz).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

namespace tvb {

struct Grid {
  int nx, ny, nz;      // elements per axis
  int px, py, pz;      // nodes per axis (= n + 1)
  long long ne, nn;    // element / node counts
  __host__ __device__ long long node(int x, int y, int z) const {
    return (long long)x + (long long)px * ((long long)y + (long long)py * z);
  }
  __host__ __device__ long long elem(int x, int y, int z) const {
    return (long long)x + (long long)nx * ((long long)y + (long long)ny * z);
  }
};

inline Grid make_grid(int nx, int ny, int nz) {
  Grid g;
  g.nx = nx; g.ny = ny; g.nz = nz;
  g.px = nx + 1; g.py = ny + 1; g.pz = nz + 1;
  g.ne = (long long)nx * ny * nz;
  g.nn = (long long)g.px * g.py * g.pz;
  return g;
}

// The element stiffness in mode space reduced to its 8 structurally distinct
// constants {k0-k1, k1, k2, k3, k4, k5-k6, k6, k7} (see modal_apply8 and
// modal_reduce in capi.cu). sm_100 DFMA cannot read the constant bank, so
// these 8 doubles are held in registers for the whole kernel.
struct Modal {
  double k[8];
};

constexpr int kStatusOk = 0;
constexpr int kStatusBadDims = 1;
constexpr int kStatusCuda = 2;
constexpr int kStatusNotSpd = 3;
constexpr int kStatusNoConvergence = 4;
constexpr int kStatusSingular = 5;
constexpr int kStatusBadArg = 6;
constexpr int kStatusWorkspace = 7;

// Deterministic block reduction helpers -----------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Sum over the CTA in a fixed order (warp tree, then warp 0 over warp sums).
// Result valid in thread 0. `scratch` must hold blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : 0.0;
    r = warp_max(r);
  }
  return r;
}

// cp.async helpers (LDGSTS) ------------------------------------------------
// smem given as a shared-window byte address (precomputed by the caller)
__device__ __forceinline__ void cp_async8_s(unsigned smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Programmatic dependent launch (sm_90+) ------------------------------------
// Every kernel of the solver iteration starts with pdl_entry(): it lets the
// next kernel in the stream launch as soon as all of this grid's CTAs are
// resident (launch_dependents), then blocks until the previous grid has
// completed and its writes are visible (wait). So the next kernel's launch
// and CTA rasterisation overlap this kernel's run instead of following its
// completion, and no kernel touches its predecessor's data early. Both
// instructions are no-ops for a grid launched without the PDL attribute.
// All CTAs of a grid are resident before its dependents can launch, so
// early-launched CTAs can never starve their predecessor of SM slots.
__device__ __forceinline__ void pdl_entry() {
#ifdef TVB_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

// TVB_PDL=0 launches without the attribute (A/B experiments).
inline bool pdl_enabled() {
  static const int on = getenv("TVB_PDL") ? atoi(getenv("TVB_PDL")) : 1;
  return on != 0;
}

// kernel<<<grid, block, smem, s>>>(args...) with the programmatic-stream-
// serialization attribute (captured into graphs as programmatic edges)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace tvb
