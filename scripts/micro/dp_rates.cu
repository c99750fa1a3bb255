// fp64 pipe rates on this GPU: DADD vs DMUL vs DFMA vs "add as fma(a, 1, b)".
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dp_rates dp_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double a) {
  double v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(v[i]) : "d"(a));
      if (OP == 1) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(v[i]) : "d"(a));
      if (OP == 2) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(v[i]) : "d"(a));
      if (OP == 3) asm volatile("fma.rn.f64 %0, %0, 0d3FF0000000000000, %1;" : "+d"(v[i]) : "d"(a));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  const char* names[4] = {"DADD", "DMUL", "DFMA", "add as fma(x,1,y)"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 4096;
  for (int op = 0; op < 4; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (op == 0) k<0><<<148 * 8, 256>>>(out, iters, 1.0000001);
      if (op == 1) k<1><<<148 * 8, 256>>>(out, iters, 1.0000001);
      if (op == 2) k<2><<<148 * 8, 256>>>(out, iters, 1.0000001);
      if (op == 3) k<3><<<148 * 8, 256>>>(out, iters, 1.0000001);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 148.0 * 8 * 256 * iters * 8;
      if (rep) printf("%-20s %.2f T instr-lanes/s\n", names[op], ops / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
