// fp64 DMMA GEMM / Gram fed by TMA tensor tiles (cp.async.bulk.tensor + mbarrier), sm_100a.
//
// Same math and CTA shape as k_gemm.cu (tile 64 x 64 x 16, 4 warps of 32 x 32, DMMA.8x8x4,
// 3 stages, 4 CTAs per SM) but the operand tiles are brought in by the TMA unit: one elected
// thread arms the stage's mbarrier and issues the tensor copies; the 128 threads spend their
// issue slots on fragment loads and DMMAs only (the cp.async kernel spends ~1/4 of its
// instructions on LDGSTS and their address/predicate arithmetic).
//
// Shared-memory layout: dense 128-byte rows with the hardware 128B swizzle (16-byte chunk index
// XOR row index mod 8).  A plain (consecutive-index) DMMA fragment read of such a tile is 2-way
// bank conflicted for either operand orientation: the fragment's 4 consecutive k (or m) map to
// the same 16-byte chunks.  The fix is an index permutation, not padding:
//   fragment row/col r (0..7)  <->  tile index mu(r) = {0,1,4,5,2,3,6,7}[r]
//   fragment k-lane q (0..3)   <->  k offset {0,1,4,5}[q] (+2 for the second MMA of a k-octet)
// The sum over k is order independent and a row permutation only relabels which rows an MMA
// produces, so C is unchanged; with it the 16 lanes of a half-warp touch 16 distinct 8-byte
// bank pairs for K-contiguous ([m][16 k]) and K-major ([k][16 m] boxes) tiles alike:
//   K-contiguous  byte(m, k)  = m*128 + (((k>>1) ^ (m&7)) << 4) + ((k&1) << 3)
//   K-major       byte(m, k)  = (m>>4)*2048 + k*128 + ((((m&15)>>1) ^ (k&7)) << 4) + ((m&1) << 3)
// (half-warp: m&7 in {0,1,4,5} or {2,3,6,7}, k&7 in {0,1,4,5} or {2,3,6,7}: the XOR of a chunk
// pair {c, c^2} with four indices pairwise different in bits 0 and 2 gives 8 distinct chunks.)
//
// Ragged edges: the TMA zero-fills out-of-bounds elements (M, N and K tails).
// Eligibility (tk_dgemm falls back to the cp.async kernel otherwise): beta == 0, no
// triangular-B mode, 16-byte aligned bases, even leading dimensions.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "ttk_internal.h"

namespace {

constexpr int BM = 64, BK = 16, STAGES = 3, NT = 128;
constexpr int TILE_BYTES = BM * BK * 8;            // 8 KB: the A tile (and the B tile for BN = 64)

__device__ __forceinline__ unsigned smaddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// byte offset of element (m, k) of a swizzled operand tile (see the header comment)
template <bool KMAJOR>
__device__ __forceinline__ int tile_off(int m, int k) {
  if (KMAJOR)
    return ((m >> 4) << 11) + (k << 7) + ((((m & 15) >> 1) ^ (k & 7)) << 4) + ((m & 1) << 3);
  return (m << 7) + (((k >> 1) ^ (m & 7)) << 4) + ((k & 1) << 3);
}

// One stage's operand tile of ROWS rows.  K-contiguous operand (row-major [rows][K]): one
// 16 x ROWS box at (k0, r0); K-major operand ([K][rows]): ROWS / 16 boxes of 16 x 16 at
// (r0 + 16 b, k0).
template <bool KMAJOR, int ROWS>
__device__ __forceinline__ void issue_tile(unsigned dst, const CUtensorMap* map, int r0, int k0,
                                           unsigned bar) {
  if (KMAJOR) {
#pragma unroll
    for (int b = 0; b < ROWS / 16; b++) tma_load_2d(dst + b * 2048, map, r0 + 16 * b, k0, bar);
  } else {
    tma_load_2d(dst, map, k0, r0, bar);
  }
}

// BN_: tile columns, 64 or 80 (N = 80 j products such as the c4 reconstruction, N = 160: warp
// tiles 32 x 40, no ragged tile column).
template <bool A_KMAJOR, bool B_KMAJOR, int BN_>
__global__ void __launch_bounds__(NT, 4) dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB,
                                                       int64_t M, int64_t N, int64_t K,
                                                       double* __restrict__ C, int64_t ldc,
                                                       double alpha, int64_t kchunk, int sym,
                                                       double* __restrict__ partial,
                                                       const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int tile_m = blockIdx.y, tile_n = blockIdx.x;
  if (sym && tile_n < tile_m) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bars[2 * STAGES];  // full[s], empty[s]
  constexpr int FN = BN_ / 16, WN_COLS = BN_ / 2;
  constexpr int TILE_BYTES_B = BN_ * BK * 8, STAGE_BYTES = TILE_BYTES + TILE_BYTES_B;
  const unsigned sbase = smaddr(smem_raw);
  if (sbase & 1023u) __trap();  // the 128B swizzle pattern repeats every 1024 bytes
  const unsigned bar0 = smaddr(bars);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int lr = lane >> 2, lc = lane & 3;
  const int64_t m0 = (int64_t)tile_m * BM, n0 = (int64_t)tile_n * BN_;
  const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) {
      mbar_init(bar0 + 8 * s, 1);
      mbar_init(bar0 + 8 * (STAGES + s), NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++)
      if (s < ntiles) {
        const unsigned fb = bar0 + 8 * s, dst = sbase + s * STAGE_BYTES;
        const int k0 = (int)(kbeg + (int64_t)s * BK);
        mbar_expect_tx(fb, STAGE_BYTES);
        issue_tile<A_KMAJOR, BM>(dst, &tmA, (int)m0, k0, fb);
        issue_tile<B_KMAJOR, BN_>(dst + TILE_BYTES, &tmB, (int)n0, k0, fb);
      }
  }

  // fragment index permutation
  const int mu = (lr & 1) | ((lr & 2) << 1) | ((lr & 4) >> 1);  // {0,1,4,5,2,3,6,7}[lr]
  const int kq = (lc & 1) | ((lc & 2) << 1);                    // {0,1,4,5}[lc]
  // Fragment addresses.  With k = 8 g + kq + 2 j (step st = 2 g + j) and rows m + 8 i the
  // swizzled offsets are the base offset with a few bits flipped plus a constant:
  //   K-contiguous: (base ^ (j << 4) ^ (g << 6)) + 1024 i
  //   K-major     : (base ^ (j << 5) ^ ((i & 1) << 6)) + 2048 (i >> 1) + 1024 g + 256 j
  // (kq has bits 0 and 2 only and mu >> 1 bits 0.. of the chunk index, so +2 in k, +4 in
  // k >> 1 and +8 in m are XORs of single chunk-index bits) — four base registers per operand.
  const int baseA = tile_off<A_KMAJOR>(wm * 32 + mu, kq);
  const int baseB = tile_off<B_KMAJOR>(wn * WN_COLS + mu, kq);
  // (K-major B with 40-column warp tiles: 8 j + 40 wn crosses the 16-wide boxes irregularly, so
  // every fragment keeps its own base offset; + 2 in k is still the XOR of byte-offset bit 5)
  int oB[FN];
#pragma unroll
  for (int j = 0; j < FN; j++) oB[j] = tile_off<B_KMAJOR>(wn * WN_COLS + 8 * j + mu, kq);
  int vA[4], vB[4];
#pragma unroll
  for (int v = 0; v < 4; v++) {
    vA[v] = baseA ^ (A_KMAJOR ? (((v & 1) << 5) ^ ((v >> 1) << 6)) : (((v & 1) << 4) ^ ((v >> 1) << 6)));
    vB[v] = baseB ^ (B_KMAJOR ? (((v & 1) << 5) ^ ((v >> 1) << 6)) : (((v & 1) << 4) ^ ((v >> 1) << 6)));
  }
  double acc[4][FN][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const char* sgen = (const char*)__cvta_shared_to_generic((size_t)sbase);
  for (int t = 0; t < ntiles; t++) {
    const int s = t % STAGES;
    const unsigned ph = (unsigned)(t / STAGES) & 1u;
    // refill the stage freed by tile t - 1 with tile t - 1 + STAGES
    if (tid == 0 && t >= 1 && t - 1 + STAGES < ntiles) {
      const int sp = (t - 1) % STAGES;
      const unsigned php = (unsigned)((t - 1) / STAGES) & 1u;
      mbar_wait(bar0 + 8 * (STAGES + sp), php);
      const unsigned fb = bar0 + 8 * sp, dst = sbase + sp * STAGE_BYTES;
      const int k0 = (int)(kbeg + (int64_t)(t - 1 + STAGES) * BK);
      mbar_expect_tx(fb, STAGE_BYTES);
      issue_tile<A_KMAJOR, BM>(dst, &tmA, (int)m0, k0, fb);
      issue_tile<B_KMAJOR, BN_>(dst + TILE_BYTES, &tmB, (int)n0, k0, fb);
    }
    __syncwarp();
    mbar_wait(bar0 + 8 * s, ph);
    const char* as = sgen + s * STAGE_BYTES;
    const char* bs = as + TILE_BYTES;
#pragma unroll
    for (int st = 0; st < 4; st++) {
      double a[4], b[FN];
      const int g = st >> 1, j2 = st & 1;
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int off = A_KMAJOR ? vA[j2 | ((i & 1) << 1)] + 2048 * (i >> 1) + 1024 * g + 256 * j2
                                 : vA[j2 | (g << 1)] + 1024 * i;
        a[i] = *(const double*)(as + off);
      }
#pragma unroll
      for (int j = 0; j < FN; j++) {
        int off;
        if (B_KMAJOR && BN_ != 64)
          off = (oB[j] ^ (j2 << 5)) + 1024 * g + 256 * j2;
        else
          off = B_KMAJOR ? vB[j2 | ((j & 1) << 1)] + 2048 * (j >> 1) + 1024 * g + 256 * j2
                         : vB[j2 | (g << 1)] + 1024 * j;
        b[j] = *(const double*)(bs + off);
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < FN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    // The stage is about to be overwritten by the TMA (async proxy) while it was read through
    // the generic proxy: the release needs a cross-proxy fence.  Without it a warp's fragment
    // loads were occasionally overtaken by the refill when the CTA shared its SM with
    // higher-priority kernels (bond-1 reconstruction on the side stream: a few wrong 32 x 32
    // warp tiles per run; a CTA barrier instead of the fence did not help).
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(bar0 + 8 * (STAGES + s));
  }

  // epilogue: fragment (i, j) holds row m = 8 i + mu(lr), columns 8 j + mu(2 lc) + {0, 1}
  const int nc = ((lc & 1) << 2) | (lc & 2);
  const bool vec_out = !sym && (N % 2 == 0) &&
                       (partial ? true : ((ldc % 2 == 0) && (((uintptr_t)C & 15) == 0)));
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const int64_t gm = m0 + wm * 32 + i * 8 + mu;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < FN; j++) {
      const int64_t gn = n0 + wn * WN_COLS + j * 8 + nc;
      if (vec_out) {
        if (gn >= N) continue;
        if (partial)
          *(double2*)(partial + ((int64_t)blockIdx.z * M + gm) * N + gn) =
              make_double2(acc[i][j][0], acc[i][j][1]);
        else
          *(double2*)(C + gm * ldc + gn) = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
      } else {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t g = gn + h;
          if (g >= N || (sym && g < gm)) continue;
          const double v = acc[i][j][h];
          if (partial) {
            partial[((int64_t)blockIdx.z * M + gm) * N + g] = v;
          } else {
            C[gm * ldc + g] = alpha * v;
            if (sym && g != gm) C[g * ldc + gm] = alpha * v;
          }
        }
      }
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  });
  return fn;
}

// rows x K operand: kmajor = stored [K][rows] (rows contiguous), else [rows][K] (K contiguous)
bool make_map(CUtensorMap* map, const double* base, bool kmajor, int64_t rows, int64_t K,
              int64_t ld, int tile_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2], estr[2] = {1, 1};
  if (kmajor) {
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)K;
    box[0] = 16;
    box[1] = 16;
  } else {
    dims[0] = (cuuint64_t)K;
    dims[1] = (cuuint64_t)rows;
    box[0] = 16;
    box[1] = (cuuint32_t)tile_rows;
  }
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool AK, bool BKm, int BN_>
int launch(tk_ctx* ctx, dim3 grid, const CUtensorMap& ta, const CUtensorMap& tb, int64_t M,
           int64_t N, int64_t K, double* C, int64_t ldc, double alpha, int64_t kchunk, int sym,
           double* partial, const int* skip) {
  const size_t smem = (size_t)STAGES * (TILE_BYTES + BN_ * BK * 8);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(dgemm_tma_kernel<AK, BKm, BN_>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_set = true;
  }
  dgemm_tma_kernel<AK, BKm, BN_><<<grid, NT, smem, ctx->stream>>>(ta, tb, M, N, K, C, ldc, alpha,
                                                                  kchunk, sym, partial, skip);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
template <int BN_>
int launch_bn(tk_ctx* ctx, bool AK, bool BKm, dim3 grid, const CUtensorMap& ta,
              const CUtensorMap& tb, int64_t M, int64_t N, int64_t K, double* C, int64_t ldc,
              double alpha, int64_t kchunk, int sym, double* partial, const int* skip) {
  if (AK && BKm) return launch<true, true, BN_>(ctx, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
  if (AK && !BKm) return launch<true, false, BN_>(ctx, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
  if (!AK && BKm) return launch<false, true, BN_>(ctx, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
  return launch<false, false, BN_>(ctx, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
}

}  // namespace

bool tk_dgemm_tma_eligible(bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                           const double* A, int64_t lda, const double* B, int64_t ldb) {
  if (!encode_fn()) return false;
  if ((lda & 1) || (ldb & 1) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15)) return false;
  if (M >= (1LL << 31) || N >= (1LL << 31) || K >= (1LL << 31)) return false;
  (void)transA;
  (void)transB;
  return true;
}

// The TMA-fed kernel proper (split-K decided by tk_dgemm).  sym: symmetric Gram flag; bn: tile
// columns (64, or 80 for N = 80 j).
int tk_dgemm_tma_launch(tk_ctx* ctx, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C, int64_t ldc, int64_t kchunk, int splits, int sym,
                        double* partial, const int* skip, int bn) {
  CUtensorMap ta, tb;
  const bool AK = transA, BKm = !transB;
  if (!make_map(&ta, A, AK, M, K, lda, BM) || !make_map(&tb, B, BKm, N, K, ldb, bn)) {
    ctx->err = "tk_dgemm: cuTensorMapEncodeTiled failed";
    return TK_ECUDA;
  }
  dim3 grid((unsigned)((N + bn - 1) / bn), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  if (bn == 80)
    return launch_bn<80>(ctx, AK, BKm, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
  return launch_bn<64>(ctx, AK, BKm, grid, ta, tb, M, N, K, C, ldc, alpha, kchunk, sym, partial, skip);
}

__global__ void tk_anchor_k_gemm_tma_k() {}
const void* tk_anchor_k_gemm_tma() { return (const void*)tk_anchor_k_gemm_tma_k; }
