// fp64 GEMM / Gram on the FP64 tensor pipe (DMMA) for sm_100a.
//
// tcgen05 has no f64 kind, so fp64 tensor work on B200 is the warp-level
// mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4).  CTA tile 64x64x16, 4 warps each
// owning a 32x32 sub-tile (4x4 DMMA fragments, 32 fp64 accumulators per thread), operands
// staged through a 3-stage cp.async (LDGSTS) shared-memory pipeline with zero-filled ragged
// edges.  Layout-generic: A may be M-major (row-major M x K) or K-major (stored K x M, the
// Gram/"TN" case), B K-major (K x N) or N-major (stored N x K).  Shared-memory strides are
// padded so every fragment load is bank-conflict free.
//
// Split-K (for the tall-skinny Grams Y^T Y where M, N << K) writes per-split partial tiles
// that a second kernel reduces in a fixed order: results are deterministic.
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>

#include "ttk_internal.h"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, NT = 128;
constexpr int PADK = 4;   // stride BK+4 = 20 doubles for M/N-major tiles
constexpr int PADM = 4;   // stride BM+4 = 68 doubles for K-major tiles

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int valid_elems) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid_elems * 8;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Shared-memory tile geometry
template <bool KMAJOR, int BMN>
struct TileGeom {
  // KMAJOR: [BK][BMN + PADM];  else [BMN][BK + PADK]
  static constexpr int SIZE = KMAJOR ? BK * (BMN + PADM) : BMN * (BK + PADK);
  __device__ static __forceinline__ int idx(int k, int m) {
    return KMAJOR ? k * (BMN + PADM) + m : m * (BK + PADK) + k;
  }
};

// Load a BMN x BK tile of an operand into shared memory.
//   KMAJOR: global element (k, m) at G[(k0+k)*ld + m0+m]   (contiguous in m)
//   else  : global element (k, m) at G[(m0+m)*ld + k0+k]   (contiguous in k)
template <bool KMAJOR, int BMN, bool VEC2, int NTH = NT>
__device__ __forceinline__ void load_tile(double* sm, const double* __restrict__ G, int64_t ld,
                                          int64_t m0, int64_t mlim, int64_t k0, int64_t klim,
                                          int tid) {
  using GEO = TileGeom<KMAJOR, BMN>;
  if (VEC2) {
    constexpr int PAIRS = BMN * BK / 2;
#pragma unroll
    for (int e = tid; e < PAIRS; e += NTH) {
      int k, m;
      int64_t gk, gm;
      const double* src;
      int valid;
      if (KMAJOR) {
        k = e / (BMN / 2);
        m = (e % (BMN / 2)) * 2;
        gk = k0 + k;
        gm = m0 + m;
        valid = (gk < klim) ? (int)max((int64_t)0, min((int64_t)2, mlim - gm)) : 0;
        src = G + (valid ? gk * ld + gm : 0);
        cp_async16(sm + GEO::idx(k, m), src, valid);
      } else {
        m = e / (BK / 2);
        k = (e % (BK / 2)) * 2;
        gk = k0 + k;
        gm = m0 + m;
        valid = (gm < mlim) ? (int)max((int64_t)0, min((int64_t)2, klim - gk)) : 0;
        src = G + (valid ? gm * ld + gk : 0);
        cp_async16(sm + GEO::idx(k, m), src, valid);
      }
    }
  } else {
    constexpr int ELEMS = BMN * BK;
#pragma unroll
    for (int e = tid; e < ELEMS; e += NTH) {
      int k, m;
      if (KMAJOR) {
        k = e / BMN;
        m = e % BMN;
      } else {
        m = e / BK;
        k = e % BK;
      }
      int64_t gk = k0 + k, gm = m0 + m;
      bool valid = gk < klim && gm < mlim;
      const double* src = G + (valid ? (KMAJOR ? gk * ld + gm : gm * ld + gk) : 0);
      cp_async8(sm + GEO::idx(k, m), src, valid);
    }
  }
}

// A_KMAJOR == transA ; B_KMAJOR == !transB.  CTA tile BM_ x BN_ x BK, WM x WN warps, each
// warp a (BM_/WM) x (BN_/WN) sub-tile of (BM_/WM/8) x (BN_/WN/8) DMMA fragments.
// BETA: C is read (beta != 0); the beta == 0 instantiations never touch C before writing it
// and keep <= 128 registers (4 CTAs per SM for the 64 x 64 tile).
template <int BM_, int BN_, int WM, int WN, bool A_KMAJOR, bool B_KMAJOR, bool VEC2, bool BETA>
__global__ void __launch_bounds__(32 * WM * WN, (BETA ? 3 : 0)) dgemm_kernel(
    int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t lda,
    const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc, double alpha,
    double beta, int64_t kchunk, int sym, double* __restrict__ partial,
    const int* __restrict__ skip) {
  constexpr int NTH = 32 * WM * WN, FM = BM_ / WM / 8, FN = BN_ / WN / 8;
  if (skip && *skip) return;  // device-side no-op flag (a finished pivoted Cholesky)
  using GA = TileGeom<A_KMAJOR, BM_>;
  using GB = TileGeom<B_KMAJOR, BN_>;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * GA::SIZE;

  // sym bit 0: symmetric Gram (upper tiles, mirrored); bit 1: B is upper triangular (row k of
  // B is zero beyond column k), so tile column n0 only needs k < n0 + BN_
  const int triu = sym & 2;
  sym &= 1;
  const int tile_m = blockIdx.y, tile_n = blockIdx.x;
  if (sym && tile_n < tile_m) return;
  const int64_t m0 = (int64_t)tile_m * BM_, n0 = (int64_t)tile_n * BN_;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(triu ? min(K, n0 + BN_) : K, kbeg + kchunk);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int lr = lane >> 2, lc = lane & 3;

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; i++)
#pragma unroll
    for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t ntiles = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  // prologue
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < ntiles) {
      int64_t k0 = kbeg + (int64_t)s * BK;
      load_tile<A_KMAJOR, BM_, VEC2, NTH>(As + s * GA::SIZE, A, lda, m0, M, k0, kend, tid);
      load_tile<B_KMAJOR, BN_, VEC2, NTH>(Bs + s * GB::SIZE, B, ldb, n0, N, k0, kend, tid);
    }
    cp_commit();
  }

  for (int64_t t = 0; t < ntiles; t++) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    // prefetch tile t + STAGES - 1
    {
      int64_t tn = t + STAGES - 1;
      if (tn < ntiles) {
        int s = (int)(tn % STAGES);
        int64_t k0 = kbeg + tn * BK;
        load_tile<A_KMAJOR, BM_, VEC2, NTH>(As + s * GA::SIZE, A, lda, m0, M, k0, kend, tid);
        load_tile<B_KMAJOR, BN_, VEC2, NTH>(Bs + s * GB::SIZE, B, ldb, n0, N, k0, kend, tid);
      }
      cp_commit();
    }
    const double* as = As + (int)(t % STAGES) * GA::SIZE;
    const double* bs = Bs + (int)(t % STAGES) * GB::SIZE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[FM], b[FN];
#pragma unroll
      for (int i = 0; i < FM; i++) a[i] = as[GA::idx(kk + lc, wm * (BM_ / WM) + i * 8 + lr)];
#pragma unroll
      for (int j = 0; j < FN; j++) b[j] = bs[GB::idx(kk + lc, wn * (BN_ / WN) + j * 8 + lr)];
#pragma unroll
      for (int i = 0; i < FM; i++)
#pragma unroll
        for (int j = 0; j < FN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();

  if (!BETA) {
    // epilogue.  Fast path (no symmetric mirror, N and ldc even, C 16-byte aligned): each lane's
    // two adjacent outputs as one 16-byte store (the scalar stores stalled on the LSU: 17 % of the
    // form_W warp samples sat in the epilogue)
    const bool vec_out = !sym && (N % 2 == 0) &&
                         (partial ? true : ((ldc % 2 == 0) && (((uintptr_t)C & 15) == 0)));
    if (vec_out) {
  #pragma unroll
      for (int i = 0; i < FM; i++) {
        const int64_t gm = m0 + wm * (BM_ / WM) + i * 8 + lr;
        if (gm >= M) continue;
  #pragma unroll
        for (int j = 0; j < FN; j++) {
          const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc;
          if (gn >= N) continue;
          if (partial) {
            *(double2*)(partial + ((int64_t)blockIdx.z * M + gm) * N + gn) =
                make_double2(acc[i][j][0], acc[i][j][1]);
          } else {
            double2 o = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
            double2* cp = (double2*)(C + gm * ldc + gn);
            if (beta != 0.0) {
              const double2 c = *cp;
              o.x += beta * c.x;
              o.y += beta * c.y;
            }
            *cp = o;
          }
        }
      }
      return;
    }
  #pragma unroll
    for (int i = 0; i < FM; i++) {
      const int64_t gm = m0 + wm * (BM_ / WM) + i * 8 + lr;
      if (gm >= M) continue;
  #pragma unroll
      for (int j = 0; j < FN; j++) {
  #pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc + h;
          if (gn >= N) continue;
          if (sym && gn < gm) continue;
          double v = acc[i][j][h];
          if (partial) {
            partial[((int64_t)blockIdx.z * M + gm) * N + gn] = v;
          } else {
            double o = alpha * v;
            if (beta != 0.0) o += beta * C[gm * ldc + gn];
            C[gm * ldc + gn] = o;
            if (sym && gn != gm) {
              double o2 = alpha * v;
              if (beta != 0.0) o2 += beta * C[gn * ldc + gm];
              C[gn * ldc + gm] = o2;
            }
          }
        }
      }
    }
    return;
  }
  // epilogue.  Fast path (no symmetric mirror, N and ldc even, C 16-byte aligned): each lane's
  // two adjacent outputs as one 16-byte store (the scalar stores stalled on the LSU: 17 % of the
  // form_W warp samples sat in the epilogue)
  const bool vec_out = !sym && (N % 2 == 0) &&
                       (partial ? true : ((ldc % 2 == 0) && (((uintptr_t)C & 15) == 0)));
  // With beta != 0 every output needs a read of C: the reads of one fragment row i are issued
  // together BEFORE its stores (the compiler cannot move a load of C above a store to C, so the
  // former load-compute-store per element cost one L2 round trip each: ~20 us for a 64 x 64
  // symmetric tile, the trailing updates of the Cholesky panels).
  if (vec_out) {
#pragma unroll
    for (int i = 0; i < FM; i++) {
      const int64_t gm = m0 + wm * (BM_ / WM) + i * 8 + lr;
      if (gm >= M) continue;
      if (partial) {
#pragma unroll
        for (int j = 0; j < FN; j++) {
          const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc;
          if (gn < N)
            *(double2*)(partial + ((int64_t)blockIdx.z * M + gm) * N + gn) =
                make_double2(acc[i][j][0], acc[i][j][1]);
        }
        continue;
      }
      double2 cv[FN];
      if (BETA) {
#pragma unroll
        for (int j = 0; j < FN; j++) {
          const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc;
          cv[j] = gn < N ? *(const double2*)(C + gm * ldc + gn) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int j = 0; j < FN; j++) {
        const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc;
        if (gn >= N) continue;
        double2 o = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        if (BETA) {
          o.x += beta * cv[j].x;
          o.y += beta * cv[j].y;
        }
        *(double2*)(C + gm * ldc + gn) = o;
      }
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < FM; i++) {
    const int64_t gm = m0 + wm * (BM_ / WM) + i * 8 + lr;
    if (gm >= M) continue;
    double cn[FN][2], cmir[FN][2];
    if (BETA && !partial) {
#pragma unroll
      for (int j = 0; j < FN; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc + h;
          const bool ok = gn < N && !(sym && gn < gm);
          cn[j][h] = ok ? C[gm * ldc + gn] : 0.0;
          cmir[j][h] = (ok && sym && gn != gm) ? C[gn * ldc + gm] : 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < FN; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t gn = n0 + wn * (BN_ / WN) + j * 8 + 2 * lc + h;
        if (gn >= N) continue;
        if (sym && gn < gm) continue;
        double v = acc[i][j][h];
        if (partial) {
          partial[((int64_t)blockIdx.z * M + gm) * N + gn] = v;
        } else {
          double o = alpha * v;
          if (BETA) o += beta * cn[j][h];
          C[gm * ldc + gn] = o;
          if (sym && gn != gm) {
            double o2 = alpha * v;
            if (BETA) o2 += beta * cmir[j][h];
            C[gn * ldc + gm] = o2;
          }
        }
      }
    }
  }
}

__global__ void splitk_reduce(int64_t M, int64_t N, int splits, const double* __restrict__ P,
                              double* __restrict__ C, int64_t ldc, double alpha, double beta,
                              int sym, const int* __restrict__ skip) {
  if (skip && *skip) return;
  int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t m = e / N, n = e % N;
    int64_t pm = m, pn = n;
    if (sym && n < m) {
      pm = n;
      pn = m;
    }
    double s = 0.0;
    for (int z = 0; z < splits; z++) s += P[((int64_t)z * M + pm) * N + pn];
    double o = alpha * s;
    if (beta != 0.0) o += beta * C[m * ldc + n];
    C[m * ldc + n] = o;
  }
}

template <int BM_, int BN_, int WM, int WN, bool AK, bool BK_, bool V2, bool BETA>
int launch_t(tk_ctx* ctx, dim3 grid, int64_t M, int64_t N, int64_t K, const double* A,
             int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, double alpha,
             double beta, int64_t kchunk, int sym, double* partial, const int* skip) {
  using GA = TileGeom<AK, BM_>;
  using GB = TileGeom<BK_, BN_>;
  size_t smem = (size_t)STAGES * (GA::SIZE + GB::SIZE) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(dgemm_kernel<BM_, BN_, WM, WN, AK, BK_, V2, BETA>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  dgemm_kernel<BM_, BN_, WM, WN, AK, BK_, V2, BETA><<<grid, 32 * WM * WN, smem, ctx->stream>>>(
      M, N, K, A, lda, B, ldb, C, ldc, alpha, beta, kchunk, sym, partial, skip);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

// tile configurations: 0 = 64 x 64 (4 warps of 32 x 32), 1 = 128 x 64 (4 warps of 64 x 32),
// 2 = 128 x 80 (4 warps of 64 x 40: N = 80 j without a ragged tile)
template <int CFG, bool AK, bool BK_, bool V2>
int launch_cfg(tk_ctx* ctx, dim3 grid, int64_t M, int64_t N, int64_t K, const double* A,
               int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, double alpha,
               double beta, int64_t kchunk, int sym, double* partial, const int* skip) {
  // beta != 0 only on the 64 x 64 tile (the caller maps it there)
  if (beta != 0.0 && !partial)
    return launch_t<64, 64, 2, 2, AK, BK_, V2, true>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc,
                                                     alpha, beta, kchunk, sym, partial, skip);
  if (CFG == 1)
    return launch_t<128, 64, 2, 2, AK, BK_, V2, false>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc,
                                                       alpha, beta, kchunk, sym, partial, skip);
  if (CFG == 2)
    return launch_t<128, 80, 2, 2, AK, BK_, V2, false>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc,
                                                       alpha, beta, kchunk, sym, partial, skip);
  return launch_t<64, 64, 2, 2, AK, BK_, V2, false>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc,
                                                    alpha, beta, kchunk, sym, partial, skip);
}

}  // namespace

int tk_dgemm(tk_ctx* ctx, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
             double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
             double beta, double* C, int64_t ldc, bool sym, bool triu_b, const int* skip) {
  if (M <= 0 || N <= 0) return TK_OK;
  if (sym && M != N) {
    ctx->err = "tk_dgemm: sym requires M == N";
    return TK_EARG;
  }
  if (K <= 0) {
    if (beta != 0.0) {
      ctx->err = "tk_dgemm: K == 0 with beta != 0 is not supported";
      return TK_EARG;
    }
    TK_TRY(tk_zero(ctx, C, M, sizeof(double) * N, sizeof(double) * ldc));
    return TK_OK;
  }
  // tile configuration: large non-symmetric products whose N is a multiple of 80 but not of 64
  // (160 at c4: the bond-1 reconstruction) take the 128 x 80 tile (warp tiles 64 x 40, no
  // ragged tile column: c4 form_U1 6.09 -> 5.51 ms)
  int cfg = 0;
  // (the 128 x 64 tile measured slower than 64 x 64 on the c4 form_W: 27.96 vs 27.06 ms — half
  // the resident warps)
  if (beta == 0.0 && !sym && M >= 128LL * 4 * ctx->num_sms && N >= 64 && N % 64 != 0 &&
      N % 80 == 0)
    cfg = 2;
  const int64_t bm = cfg == 2 ? 128 : BM, bn = cfg == 2 ? 80 : BN;
  const int64_t tm = (M + bm - 1) / bm, tn = (N + bn - 1) / bn;
  int64_t tiles = sym ? tm * (tm + 1) / 2 : tm * tn;
  // split-K for small outputs with a long K: about four waves of resident CTAs (SMs x CTAs/SM);
  // measured at c4 (bond-1 Gram 640 x 640 x 786432): 1 wave 15.4 ms, 2 waves 11.5, 3-6 waves
  // 11.2-11.3 (the former "4 CTAs per SM" target gave 14.0)
  static int per_sm = 0;
  if (per_sm == 0) {
    const size_t smem = (size_t)STAGES * 2 * BM * (BK + PADK) * sizeof(double);
    cudaFuncSetAttribute(dgemm_kernel<64, 64, 2, 2, true, true, true, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, dgemm_kernel<64, 64, 2, 2, true, true, true, false>, NT, smem);
    per_sm = std::max(per_sm, 1);
  }
  // heavy products with beta == 0: the TMA-fed kernel (same tile, same split-K partials)
  const double flops = sym ? (double)M * (M + 1) * K : 2.0 * M * N * K;
  // (cfg 2, the N = 80 j products, runs the TMA kernel's 64 x 80 tile instead of the cp.async
  // 128 x 80 one)
  const bool use_tma = ctx->gemm_tma && beta == 0.0 && !triu_b && flops >= 1e8 &&
                       tk_dgemm_tma_eligible(transA, transB, M, N, K, A, lda, B, ldb);
  // Waves of resident CTAs.  cp.async kernel: 4 (time-optimal, above).  TMA kernel: 12 — shorter
  // K chunks keep the CTAs that share operand columns (the 10 tiles of a Gram's column block)
  // within an L2-sized window of each other: gram_W (640 x 640 x 786432) DRAM reads 10.8 GB at
  // 4 waves, 6.2 at 8, 5.5 at 12, 5.2 at 16 (4.03 algorithmic) and 10.19 / 10.02 / 10.00 / 9.97 ms
  // including the reduction of the partials, which grows with the split count.
  const int mult = use_tma ? 12 : 4;
  const int64_t slots = (int64_t)per_sm * ctx->num_sms * mult;
  int64_t splits = 1;
  if (cfg == 0 && tiles < slots && K >= 8 * BK) {
    splits = std::min<int64_t>(std::max<int64_t>(slots / tiles, 1), (K + 8 * BK - 1) / (8 * BK));
    splits = std::max<int64_t>(splits, 1);
    if (use_tma) {
      // the partial sums (written and re-read once) stay below 1/8 of the operand bytes (and
      // 64 MB): bounds the scratch and the extra traffic of the higher split count
      const double opb = 8.0 * ((double)M * K + (sym ? 0.0 : (double)K * N));
      const double cap = std::max(64.0 * 1048576.0, opb / 8.0);
      const int64_t smax = std::max<int64_t>((int64_t)(cap / (8.0 * M * N)), 1);
      const int64_t s4 = std::max<int64_t>(slots / (3 * tiles), 1);  // the 4-wave count
      splits = std::max(std::min(splits, smax), std::min(splits, s4));
    }
  }
  int64_t kchunk = (K + splits - 1) / splits;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  splits = (K + kchunk - 1) / kchunk;
  double* partial = nullptr;
  DevBuf pbuf;
  if (splits > 1) {
    TK_TRY(pbuf.get(ctx, (size_t)splits * M * N));
    partial = pbuf.p;
  }
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)splits);
  double pflops = flops;
  if (triu_b)
    pflops = K >= N ? (double)M * N * (N + 1) : 2.0 * M * (K * (K + 1) / 2.0 + (double)(N - K) * K);
  const double bytes = 8.0 * ((double)M * K + (sym ? 0.0 : (double)K * N) + (double)M * N);
  const int prof_id = tk_prof_begin(ctx, ctx->tag, pflops, bytes);
  const bool AK = transA, BKm = !transB;
  // 16-byte vector path: contiguous dims even and 16-byte aligned bases
  bool v2 = (lda % 2 == 0) && (ldb % 2 == 0) && (((uintptr_t)A & 15) == 0) &&
            (((uintptr_t)B & 15) == 0);
  int st = TK_OK;
  if (use_tma) {
    st = tk_dgemm_tma_launch(ctx, transA, transB, M, N, K, alpha, A, lda, B, ldb, C, ldc, kchunk,
                             (int)splits, sym ? 1 : 0, partial, skip, cfg == 2 ? 80 : 64);
  } else {
#define TK_GEMM_CASE(a, b, v)                                                               \
  if (AK == a && BKm == b && v2 == v) {                                                     \
    const int sf = (sym ? 1 : 0) | (triu_b ? 2 : 0);                                        \
    if (cfg == 2)                                                                           \
      st = launch_cfg<2, a, b, v>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta,  \
                                  kchunk, sf, partial, skip);                                     \
    else                                                                                    \
      st = launch_cfg<0, a, b, v>(ctx, grid, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta,  \
                                  kchunk, sf, partial, skip);                                     \
  }
  TK_GEMM_CASE(false, false, false)
  TK_GEMM_CASE(false, false, true)
  TK_GEMM_CASE(false, true, false)
  TK_GEMM_CASE(false, true, true)
  TK_GEMM_CASE(true, false, false)
  TK_GEMM_CASE(true, false, true)
  TK_GEMM_CASE(true, true, false)
  TK_GEMM_CASE(true, true, true)
#undef TK_GEMM_CASE
  }
  if (st != TK_OK) return st;
  if (splits > 1) {
    int64_t total = M * N;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * ctx->num_sms);
    splitk_reduce<<<blocks, 256, 0, ctx->stream>>>(M, N, (int)splits, partial, C, ldc, alpha,
                                                   beta, sym ? 1 : 0, skip);
    TK_LAUNCH_CHECK(ctx);
  }
  tk_prof_end(ctx, prof_id);
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_gemm_k() {}
const void* tk_anchor_k_gemm() { return (const void*)tk_anchor_k_gemm_k; }
