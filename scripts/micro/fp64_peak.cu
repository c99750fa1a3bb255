// FP64 pipe microbenchmark: throughput (many independent chains) and latency
// (one dependent chain) of DFMA / DADD on this GPU. Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, bool ADD>
__global__ void k_tput(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = ADD ? (x[i] + a) : fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_lat(double* out, int iters, double a, double b, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int pass = 0; pass < 2; ++pass) {
    for (int blocks_per_sm : {4, 8}) {
      dim3 grid(sms * blocks_per_sm), block(256);
      k_tput<8, false><<<grid, block>>>(out, 16, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      if (pass == 0) k_tput<8, false><<<grid, block>>>(out, iters, 1.0000001, 1e-9);
      else k_tput<8, true><<<grid, block>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)grid.x * block.x * iters * 8;
      printf(", \"%s_per_s_bps%d\": %.4g", pass == 0 ? "dfma" : "dadd", blocks_per_sm, ops / (ms * 1e-3));
    }
  }
  k_lat<<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf(", \"dfma_latency_cycles\": %.2f}\n", (double)h / iters);
  return 0;
}
