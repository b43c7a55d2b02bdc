// HBM write / read / copy bandwidth on the c4 Y1 size (5.6 GB), 16-byte accesses.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wr(double2* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_double2(1.0, (double)i));
}
__global__ void wr_plain(double2* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_double2(1.0, (double)i);
}
__global__ void rd(const double2* p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(p + i); s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}
int main() {
  size_t bytes = 5637144576ull, n = bytes / 16;
  double2* p; double* o;
  cudaMalloc(&p, bytes); cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
    float ms;
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(a); wr<<<grid, 512>>>(p, n); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    printf("grid %5d  write(cs) %.0f GB/s", grid, bytes / ms / 1e6);
    cudaEventRecord(a); wr_plain<<<grid, 512>>>(p, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("  write %.0f GB/s", bytes / ms / 1e6);
    cudaEventRecord(a); rd<<<grid, 512>>>(p, n, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); printf("  read %.0f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}
