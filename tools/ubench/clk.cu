// Effective SM clock of a single-CTA latency-bound kernel: clock64 cycles vs globaltimer ns.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, int iters) {
  long long c0 = clock64();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double x = threadIdx.x;
  for (int i = 0; i < iters; i++) x = fma(x, 0.999, 1e-3);
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = (long long)(t1 - t0); out[2] = (long long)x; }
}
int main() {
  long long* o; cudaMallocManaged(&o, 24);
  for (int g : {1, 1, 148, 1}) {
    k<<<g, 512>>>(o, 2000000); cudaDeviceSynchronize();
    printf("grid %3d: %lld cycles in %lld ns -> %.0f MHz\n", g, o[0], o[1], 1e3 * o[0] / (double)o[1]);
  }
  return 0;
}
