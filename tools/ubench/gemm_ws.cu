// Experiment: warp-specialised DMMA GEMM fed by TMA bulk copies (cp.async.bulk + mbarrier)
// vs the library's cp.async GEMM (tk_dgemm) on the c4 form_W shape
// C (M x N) = A (M x K, row-major) * B (K x N, row-major).  Diagnostic only.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gemm_ws \
//        tools/ubench/gemm_ws.cu -Lpaper_1906_06785_b200 -lttk -Xlinker -rpath=$PWD/paper_1906_06785_b200
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>

#include "../../paper_1906_06785_b200/csrc/ttk_internal.h"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned smaddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(phase) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// CTA tile BM x BN x BK; CW consumer warps (WM x WN) each (BM/WM) x (BN/WN); 1 producer warp.
template <int BM, int BN, int BK, int WM, int WN, int STAGES>
__global__ void __launch_bounds__(32 * (WM * WN + 1)) gemm_ws(int64_t M, int64_t N, int64_t K,
                                                              const double* __restrict__ A, int64_t lda,
                                                              const double* __restrict__ B, int64_t ldb,
                                                              double* __restrict__ C, int64_t ldc) {
  constexpr int CW = WM * WN, FM = BM / WM / 8, FN = BN / WN / 8;
  constexpr int LDA = BK + 4;   // A tile [BM][BK+4]   (rows of BK doubles, padded)
  constexpr int LDB = BN + 4;   // B tile [BK][BN+4]
  constexpr int ASZ = BM * LDA, BSZ = BK * LDB;
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) unsigned long long bars[2 * STAGES];
  double* As = sm;
  double* Bs = sm + STAGES * ASZ;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t nk = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      mbar_init(smaddr(&bars[s]), 1);            // full: producer arrive + tx
      mbar_init(smaddr(&bars[STAGES + s]), CW);  // empty: one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {  // producer
    for (int64_t t = 0; t < nk; t++) {
      const int s = (int)(t % STAGES);
      const unsigned ph = (unsigned)((t / STAGES) & 1);
      if (t >= STAGES) mbar_wait(smaddr(&bars[STAGES + s]), ph ^ 1);
      const unsigned full = smaddr(&bars[s]);
      if (lane == 0) mbar_expect_tx(full, (unsigned)((BM * BK + BK * BN) * 8));
      __syncwarp();
      const int64_t k0 = t * BK;
      for (int r = lane; r < BM; r += 32)
        bulk_g2s(smaddr(As + s * ASZ + r * LDA), A + (m0 + r) * lda + k0, BK * 8, full);
      for (int r = lane; r < BK; r += 32)
        bulk_g2s(smaddr(Bs + s * BSZ + r * LDB), B + (k0 + r) * ldb + n0, BN * 8, full);
    }
    return;
  }
  const int wm = warp / WN, wn = warp % WN, lr = lane >> 2, lc = lane & 3;
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; i++)
#pragma unroll
    for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int64_t t = 0; t < nk; t++) {
    const int s = (int)(t % STAGES);
    mbar_wait(smaddr(&bars[s]), (unsigned)((t / STAGES) & 1));
    const double* as = As + s * ASZ;
    const double* bs = Bs + s * BSZ;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; i++) a[i] = as[(wm * (BM / WM) + i * 8 + lr) * LDA + kk + lc];
#pragma unroll
      for (int j = 0; j < FN; j++) b[j] = bs[(kk + lc) * LDB + wn * (BN / WN) + j * 8 + lr];
#pragma unroll
      for (int i = 0; i < FM; i++)
#pragma unroll
        for (int j = 0; j < FN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smaddr(&bars[STAGES + s]));
  }
#pragma unroll
  for (int i = 0; i < FM; i++) {
    const int64_t gm = m0 + wm * (BM / WM) + i * 8 + lr;
#pragma unroll
    for (int j = 0; j < FN; j++) {
      const int64_t gn = n0 + wn * (BN / WN) + j * 8 + 2 * lc;
      *(double2*)(C + gm * ldc + gn) = make_double2(acc[i][j][0], acc[i][j][1]);
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
float run_ws(int64_t M, int64_t N, int64_t K, const double* A, const double* B, double* C, int reps) {
  constexpr int LDA = BK + 4, LDB = BN + 4;
  size_t smem = (size_t)STAGES * (BM * LDA + BK * LDB) * 8;
  auto kern = gemm_ws<BM, BN, BK, WM, WN, STAGES>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (WM * WN + 1), smem);
  dim3 grid(N / BN, M / BM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, 32 * (WM * WN + 1), smem>>>(M, N, K, A, K, B, N, C, N);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; r++) kern<<<grid, 32 * (WM * WN + 1), smem>>>(M, N, K, A, K, B, N, C, N);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("ws %3dx%3dx%2d warps %dx%d stages %d  ctas/SM %d  smem %5.1f KB: %7.3f ms  %6.2f TF/s\n", BM, BN, BK,
         WM, WN, STAGES, per_sm, smem / 1024.0, ms, 2.0 * M * N * K / ms / 1e9);
  return ms;
}

__global__ void fill_k(double* p, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffff) / 65536.0 - 0.5;
  }
}

int main(int argc, char** argv) {
  const int64_t M = 786432, K = 896, N = 640;
  const int reps = argc > 1 ? atoi(argv[1]) : 5;
  double *A, *B, *C, *C2;
  CK(cudaMalloc(&A, M * K * 8));
  CK(cudaMalloc(&B, K * N * 8));
  CK(cudaMalloc(&C, M * N * 8));
  CK(cudaMalloc(&C2, M * N * 8));
  fill_k<<<1024, 256>>>(A, M * K, 1);
  fill_k<<<1024, 256>>>(B, K * N, 2);
  CK(cudaDeviceSynchronize());
  // library GEMM
  tk_ctx* ctx;
  tk_ctx_create(&ctx, nullptr);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  tk_dgemm(ctx, false, false, M, N, K, 1.0, A, K, B, N, 0.0, C, N);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < reps; r++) tk_dgemm(ctx, false, false, M, N, K, 1.0, A, K, B, N, 0.0, C, N);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("library tk_dgemm (cp.async):                              %7.3f ms  %6.2f TF/s\n", ms, 2.0 * M * N * K / ms / 1e9);
  auto check = [&]() {
    std::vector<double> h1(4096), h2(4096);
    double md = 0, mx = 0;
    for (int64_t off : {(int64_t)0, M * N / 2, M * N - 4096}) {
      cudaMemcpy(h1.data(), C + off, 4096 * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(h2.data(), C2 + off, 4096 * 8, cudaMemcpyDeviceToHost);
      for (int i = 0; i < 4096; i++) { md = fmax(md, fabs(h1[i] - h2[i])); mx = fmax(mx, fabs(h1[i])); }
    }
    printf("   max |diff| %.3e (max |C| %.3e)\n", md, mx);
  };
  run_ws<64, 64, 16, 2, 2, 3>(M, N, K, A, B, C2, reps); check();
  run_ws<64, 64, 16, 2, 2, 4>(M, N, K, A, B, C2, reps); check();
  run_ws<64, 64, 16, 2, 2, 6>(M, N, K, A, B, C2, reps); check();
  run_ws<64, 64, 32, 2, 2, 3>(M, N, K, A, B, C2, reps); check();
  run_ws<128, 64, 16, 4, 2, 4>(M, N, K, A, B, C2, reps); check();
  run_ws<128, 64, 16, 2, 2, 4>(M, N, K, A, B, C2, reps); check();
  run_ws<64, 128, 16, 2, 2, 4>(M, N, K, A, B, C2, reps); check();
  run_ws<128, 128, 16, 4, 4, 3>(M, N, K, A, B, C2, reps); check();
  run_ws<128, 128, 16, 2, 4, 3>(M, N, K, A, B, C2, reps); check();
  return 0;
}
