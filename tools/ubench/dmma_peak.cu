// FP64 tensor-pipe (DMMA m8n8k4) peak: independent mma.sync chains from registers only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void k(double* out, int iters) {
  double acc[8][2];
  for (int i = 0; i < 8; i++) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 20000;
    k<<<148 * 2, 32 * warps / 2>>>(o, 100);
    cudaEventRecord(e0);
    k<<<148 * 2, 32 * warps / 2>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * (148 * 2) * (warps / 2);  // 256 FMA per DMMA (per warp)
    printf("warps/SM %2d: %.2f TF/s\n", warps, flops / ms / 1e9);
  }
  return 0;
}
