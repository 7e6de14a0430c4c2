// dmma_concurrency.cu -- does the FP64 tensor-core instruction (DMMA,
// mma.sync.m8n8k4.f64) run beside the FP64 CUDA-core pipe on the B200, or on
// it?  Three kernels with 8 warps x 148 x 8 CTAs: DADD chains only, DMMA
// chains only, and both interleaved 4 : 1 (the ratio a DD multiply-accumulate
// with its cross terms on the tensor cores would have).  If the mixed
// kernel's time is max(dadd, dmma) the pipes are separate; if it is the sum
// they are one.   nvcc -arch=sm_100a -O3 -o dmma_concurrency dmma_concurrency.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int kDadd, int kDmma>
__global__ void __launch_bounds__(256) k(double* out, int iters, double seed) {
  double x[8], c[4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + i + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = seed * i;
  const double a = seed * 0.5 + (threadIdx.x & 3), b = seed * 0.25 + (threadIdx.x >> 2);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (kDadd) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(x[i], seed);  // 8 independent DADDs
      }
      if (kDmma) {
        dmma(c[r & 3], a, b);  // every DMMA = 256 FMAs = 8 DFMA instructions' worth
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int A, int B>
float run(double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<A, B><<<148 * 8, 256>>>(out, iters, 1e-300);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<A, B><<<148 * 8, 256>>>(out, iters, 1e-300);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 256);
  const int iters = 20000;
  const float d = run<1, 0>(out, iters), m = run<0, 1>(out, iters), both = run<1, 1>(out, iters);
  const double warps = 148.0 * 8 * 8, dadd_instr = warps * iters * 32.0, dmma_instr = warps * iters * 4.0;
  printf("DADD only : %8.3f ms  %.2f T lane-ops/s\n", d, dadd_instr * 32 / (d * 1e-3) / 1e12);
  printf("DMMA only : %8.3f ms  %.2f T FMA/s (256 per instruction)\n", m, dmma_instr * 256 / (m * 1e-3) / 1e12);
  printf("both      : %8.3f ms  (sum %.3f, max %.3f)\n", both, d + m, d > m ? d : m);
  printf(cudaGetLastError() == cudaSuccess ? "ok\n" : "CUDA error\n");
  return 0;
}
