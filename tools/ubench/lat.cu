// Latency microbenchmarks (cycles) for the building blocks of the latency-bound kernels.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k(double* out, long long* cyc, double x0, int iters) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double x = x0 + tid * 1e-12;
  long long t0, t1;
  // (0) dependent DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = fma(x, 0.999999, 1e-7);
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / iters;
  // (1) sqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = sqrt(x + 1.0);
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / iters;
  // (2) div chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = 1.0 / (x + 1.5);
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / iters;
  // (3) rsqrt chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = rsqrt(x + 1.0);
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / iters;
  // (4) warp_sum (double, 5 xor shuffles) chain
  t0 = clock64();
  for (int i = 0; i < iters; i++) x = warp_sum(x) * 0.03125;
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0) / iters;
  // (5) dependent LDS chain
  int idx = tid & 255;
  t0 = clock64();
  for (int i = 0; i < iters; i++) {
    double v = sm[idx];
    idx = ((int)(v * 1e9) + i) & 511;
    x += v;
  }
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / iters;
  // (6) __syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (tid == (i & 31)) sm[i & 1023] = x;
  }
  t1 = clock64();
  if (tid == 0) cyc[6] = (t1 - t0) / iters;
  out[tid] = x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"dfma", "sqrt", "div", "rsqrt", "warp_sum(double)", "lds(dep)",
                         "syncthreads(512)"};
  for (int threads : {32, 512}) {
    k<<<1, threads>>>(out, cyc, 0.5, 1000);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 7; i++) printf("  %-18s %lld cycles\n", names[i], cyc[i]);
  }
  return 0;
}
