// Experiment: tile configurations of the library's DMMA GEMM kernel (k_gemm.cu, included here
// under another name) on the c4 GEMM shapes: form_W, gram_W (symmetric, split-K), form_U1.
// Diagnostic only.
#include <cstdio>
#include <cstdlib>
#define tk_dgemm tk_dgemm_copy
#define tk_anchor_k_gemm tk_anchor_k_gemm_copy
#define tk_anchor_k_gemm_k tk_anchor_k_gemm_copy_k
#include "../../paper_1906_06785_b200/csrc/k_gemm.cu"
#undef tk_dgemm

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill_k(double* p, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffff) / 65536.0 - 0.5;
  }
}

static tk_ctx* g_ctx;
static int g_reps = 5;

template <typename F>
float timeit(F f) {
  f();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < g_reps; r++) f();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / g_reps;
}

template <int BM_, int BN_, int WM, int WN, bool AK, bool BK_>
void variant(const char* name, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
             const double* B, int64_t ldb, double* C, int64_t ldc, int sym, int64_t splits,
             double flops) {
  const int64_t tm = (M + BM_ - 1) / BM_, tn = (N + BN_ - 1) / BN_;
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  splits = (K + kchunk - 1) / kchunk;
  double* partial = nullptr;
  if (splits > 1) CK(cudaMalloc(&partial, sizeof(double) * splits * M * N));
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)splits);
  using GA = TileGeom<AK, BM_>;
  using GB = TileGeom<BK_, BN_>;
  const size_t smem = (size_t)STAGES * (GA::SIZE + GB::SIZE) * sizeof(double);
  cudaFuncSetAttribute(dgemm_kernel<BM_, BN_, WM, WN, AK, BK_, true, false>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dgemm_kernel<BM_, BN_, WM, WN, AK, BK_, true, false>,
                                                32 * WM * WN, smem);
  float ms = timeit([&]() {
    launch_t<BM_, BN_, WM, WN, AK, BK_, true, false>(g_ctx, grid, M, N, K, A, lda, B, ldb, C, ldc,
                                                     1.0, 0.0, kchunk, sym, partial, nullptr);
    if (splits > 1) {
      int64_t total = M * N;
      splitk_reduce<<<(int)std::min<int64_t>((total + 255) / 256, 8LL * 148), 256>>>(
          M, N, (int)splits, partial, C, ldc, 1.0, 0.0, sym, nullptr);
    }
  });
  printf("  %-10s %3dx%3d warps %dx%d splits %4lld ctas/SM %d: %8.3f ms %6.2f TF/s\n", name, BM_, BN_, WM,
         WN, (long long)splits, per_sm, ms, flops / ms / 1e9);
  if (partial) cudaFree(partial);
}

int main(int argc, char** argv) {
  g_reps = argc > 1 ? atoi(argv[1]) : 5;
  tk_ctx_create(&g_ctx, nullptr);
  const int64_t nx = 786432, R1 = 896, k2 = 640, r1 = 160;
  double *Y, *P, *W, *G, *F, *U;
  CK(cudaMalloc(&Y, nx * R1 * 8));
  CK(cudaMalloc(&P, R1 * k2 * 8));
  CK(cudaMalloc(&W, nx * k2 * 8));
  CK(cudaMalloc(&G, k2 * k2 * 8));
  CK(cudaMalloc(&F, k2 * r1 * 8));
  CK(cudaMalloc(&U, nx * r1 * 8));
  fill_k<<<1024, 256>>>(Y, nx * R1, 1);
  fill_k<<<1024, 256>>>(P, R1 * k2, 2);
  fill_k<<<1024, 256>>>(W, nx * k2, 3);
  fill_k<<<1024, 256>>>(F, k2 * r1, 4);
  CK(cudaDeviceSynchronize());

  printf("form_W  (%lld x %lld x %lld)\n", (long long)nx, (long long)k2, (long long)R1);
  double fl = 2.0 * nx * k2 * R1;
  printf("  library: %.3f ms\n", timeit([&]() { tk_dgemm_copy(g_ctx, false, false, nx, k2, R1, 1.0, Y, R1, P, k2, 0.0, W, k2); }));
  variant<64, 64, 2, 2, false, true>("64x64", nx, k2, R1, Y, R1, P, k2, W, k2, 0, 1, fl);
  variant<64, 128, 2, 4, false, true>("64x128", nx, k2, R1, Y, R1, P, k2, W, k2, 0, 1, fl);
  variant<128, 64, 4, 2, false, true>("128x64/8w", nx, k2, R1, Y, R1, P, k2, W, k2, 0, 1, fl);
  variant<64, 160, 2, 4, false, true>("64x160", nx, k2, R1, Y, R1, P, k2, W, k2, 0, 1, fl);

  printf("gram_W  (sym %lld x %lld x %lld)\n", (long long)k2, (long long)k2, (long long)nx);
  fl = (double)k2 * (k2 + 1) * nx;
  printf("  library: %.3f ms\n", timeit([&]() { tk_dgemm_copy(g_ctx, true, false, k2, k2, nx, 1.0, W, k2, W, k2, 0.0, G, k2, true); }));
  for (int64_t s : {16, 32, 64, 128})
    variant<64, 64, 2, 2, true, true>("64x64", k2, k2, nx, W, k2, W, k2, G, k2, 1, s, fl);
  for (int64_t s : {32, 64, 128})
    variant<128, 128, 4, 4, true, true>("128x128", k2, k2, nx, W, k2, W, k2, G, k2, 1, s, fl);
  for (int64_t s : {32, 64, 128})
    variant<64, 128, 2, 4, true, true>("64x128", k2, k2, nx, W, k2, W, k2, G, k2, 0, s, 2.0 * k2 * k2 * nx);

  printf("form_U1 (%lld x %lld x %lld)\n", (long long)nx, (long long)r1, (long long)k2);
  fl = 2.0 * nx * r1 * k2;
  printf("  library: %.3f ms\n", timeit([&]() { tk_dgemm_copy(g_ctx, false, false, nx, r1, k2, 1.0, W, k2, F, r1, 0.0, U, r1); }));
  variant<128, 80, 2, 2, false, true>("128x80", nx, r1, k2, W, k2, F, r1, U, r1, 0, 1, fl);
  variant<64, 80, 2, 2, false, true>("64x80", nx, r1, k2, W, k2, F, r1, U, r1, 0, 1, fl);
  variant<64, 160, 2, 4, false, true>("64x160", nx, r1, k2, W, k2, F, r1, U, r1, 0, 1, fl);
  variant<128, 160, 4, 4, false, true>("128x160", nx, r1, k2, W, k2, F, r1, U, r1, 0, 1, fl);
  variant<32, 160, 1, 4, false, true>("32x160", nx, r1, k2, W, k2, F, r1, U, r1, 0, 1, fl);
  return 0;
}
