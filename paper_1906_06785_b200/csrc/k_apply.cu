// Operator apply  y = sum_k (T_k (x) G_k (x) K_k) x  on TT cores (eq:Xz).
//
//  spmm_multi : Y1[:, k r1:(k+1) r1] = K_k U1 for ALL k in one sweep over the spatial rows.
//               One warp per row; the row's T*r1 outputs are written once, contiguously
//               (the write stream is 87% of the apply's HBM bytes at c4).  U1 rows are
//               gathered through the read-only path (L1/L2 reuse across neighbouring rows
//               of the stencil-like K_k).  The row's CSR entries of all terms are staged
//               in shared memory as (val, col | term << 32) pairs (lane k copies term k's) and
//               read back as broadcasts: no per-entry shuffles on the MIO pipe.
//  stoch_apply: Y2 = blockdiag_k (G_k x_2 U2), written densely (zeros off the blocks).
//  time_apply : Y3[k r2 + b, :] = U3[b, :] T_k^T with T_k in LAPACK band storage.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "ttk_internal.h"

namespace {

// V2: lane owns column pairs (16-byte loads/stores; needs r even and RPL even), else single
// columns lane + 32 u.
template <int RPL, bool V2>
__global__ void __launch_bounds__(256, (RPL <= 2 ? 4 : (RPL <= 3 ? 3 : 1))) spmm_multi_k(int64_t n_x, int T, int r,
                                                    const int32_t* __restrict__ rowptr,
                                                    const int32_t* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const int64_t* __restrict__ nnz_off,
                                                    const double* __restrict__ U1,
                                                    double* __restrict__ Y1) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t R = (int64_t)T * r;
  constexpr int CW = 32 * RPL;  // columns per chunk
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int UNR = 4;        // entries whose U1 rows are loaded together (memory-level parallelism)
  constexpr int STEP = V2 ? 2 : 1;
  constexpr int ECAP = 128;     // staged entries per warp (rows with more take the slow path)
  __shared__ double2 ent_all[256 / 32][ECAP];
  double2* ent = ent_all[threadIdx.x >> 5];
  auto colof = [lane](int u) { return V2 ? (64 * (u >> 1) + 2 * lane + (u & 1)) : (lane + 32 * u); };
  auto put = [&](double* dst, const double* acc, int lim) {  // dst: column c0; lim = r - c0
#pragma unroll
    for (int u = 0; u < RPL; u += STEP) {
      const int cc = colof(u);
      if (V2) {
        if (cc < lim) __stcs((double2*)(dst + cc), make_double2(acc[u], acc[u + 1]));
      } else {
        if (cc < lim) __stcs(dst + cc, acc[u]);
      }
    }
  };
  for (int64_t i = warp; i < n_x; i += nwarps) {
    double* yrow = Y1 + i * R;
    // Terms in groups of 32: lane k fetches the CSR extent of term kg0 + k for this row, so the
    // T row-pointer loads are issued in parallel instead of as T dependent chains.
    for (int kg0 = 0; kg0 < T; kg0 += 32) {
      const int kn = min(32, T - kg0);
      int64_t mybeg = 0;
      int mycnt = 0;
      if (lane < kn) {
        const int32_t* rp = rowptr + (int64_t)(kg0 + lane) * (n_x + 1);
        const int b = __ldg(rp + i), e = __ldg(rp + i + 1);
        mybeg = nnz_off[kg0 + lane] + b;
        mycnt = e - b;
      }
      int myoff = mycnt;  // inclusive scan -> exclusive offsets of each term's entries
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, myoff, o);
        if (lane >= o) myoff += t;
      }
      const int E = __shfl_sync(FULL, myoff, 31);
      myoff -= mycnt;
      if (E <= ECAP) {
        // stage all of the row's entries (term-major order) in shared memory: lane k copies
        // term k's (val, col) pairs; everyone reads them back as broadcasts
        if (lane < kn) {
          for (int g = 0; g < mycnt; g++) {
            const int64_t src = mybeg + g;
            ent[myoff + g] = make_double2(__ldg(val + src),
                                          __longlong_as_double((long long)__ldg(col + src)));
          }
        }
        __syncwarp();
        for (int c0 = 0; c0 < r; c0 += CW) {
          for (int k = 0; k < kn; k++) {
            const int ck = __shfl_sync(FULL, mycnt, k), ok = __shfl_sync(FULL, myoff, k);
            double acc[RPL];
#pragma unroll
            for (int u = 0; u < RPL; u++) acc[u] = 0.0;
            for (int q0 = 0; q0 < ck; q0 += UNR) {
              double uv[UNR][RPL];
              double vv[UNR];
#pragma unroll
              for (int s = 0; s < UNR; s++) {
                const bool live = q0 + s < ck;  // warp-uniform
                const double2 en = ent[ok + min(q0 + s, ck - 1)];
                const int c = (int)__double_as_longlong(en.y);
                vv[s] = live ? en.x : 0.0;
                const double* urow = U1 + (int64_t)c * r + c0;
#pragma unroll
                for (int u = 0; u < RPL; u += STEP) {
                  const int cc = colof(u);
                  const bool okc = live && c0 + cc < r;
                  if (V2) {
                    const double2 t =
                        okc ? __ldg((const double2*)(urow + cc)) : make_double2(0.0, 0.0);
                    uv[s][u] = t.x;
                    uv[s][u + 1] = t.y;
                  } else {
                    uv[s][u] = okc ? __ldg(urow + cc) : 0.0;
                  }
                }
              }
#pragma unroll
              for (int s = 0; s < UNR; s++)
#pragma unroll
                for (int u = 0; u < RPL; u++) acc[u] = fma(vv[s], uv[s][u], acc[u]);
            }
            put(yrow + (int64_t)(kg0 + k) * r + c0, acc, r - c0);
          }
        }
        __syncwarp();
      } else {
        // long row (more than ECAP entries over the group's terms): term by term from global
        for (int c0 = 0; c0 < r; c0 += CW) {
          for (int k = 0; k < kn; k++) {
            const int ck = __shfl_sync(FULL, mycnt, k);
            const int64_t bk = __shfl_sync(FULL, mybeg, k);
            double acc[RPL];
#pragma unroll
            for (int u = 0; u < RPL; u++) acc[u] = 0.0;
            for (int g = 0; g < ck; g++) {
              const int c = __ldg(col + bk + g);
              const double v = __ldg(val + bk + g);
              const double* urow = U1 + (int64_t)c * r + c0;
#pragma unroll
              for (int u = 0; u < RPL; u++) {
                const int cc = colof(u);
                if (c0 + cc < r) acc[u] = fma(v, __ldg(urow + cc), acc[u]);
              }
            }
            put(yrow + (int64_t)(kg0 + k) * r + c0, acc, r - c0);
          }
        }
      }
    }
  }
}

// Column-merged variant (T <= TM terms).  All T terms of a spatial row are merged by column
// (host side, tk_op_create): for each DISTINCT column c of the row, one word col | mask << 32
// (bit k of mask = term k has an entry at (i, c)) and, in (c, k) order, the values.  A warp
// loads each U1 row ONCE for all the terms that touch it (the per-term kernel above loads it
// once per term: at c4 44 U1-row gathers per spatial row become ~7).  Lane j expands distinct
// column j's values into a dense, zero-padded TM-vector in shared memory, so the inner loop is
// branch-free: per distinct column one U1 row load, TM/2 16-byte broadcast loads of values and
// 2 TM FMAs into the T x RPL register accumulators (k a compile-time index).  Per term the
// entries are still summed in ascending column order, as in each term's sorted CSR row (the
// zero padding adds exact zeros).  The row's T r outputs are streamed once at the end.
//
// Each row is ONE contiguous record in `rec` (int64 words): [row | gn << 32][gn words
// col | mask << 32][values as doubles], at rec + recptr[i].  Record i is NOT row i: the host
// stores the rows in a breadth-first (Cuthill-McKee) order of the merged pattern, so rows that
// gather the same U1 rows (at c4 a velocity row and the pressure rows it couples to, 2 N^2
// apart in the natural order) are processed at the same time and U1 is read from DRAM about
// once instead of twice.  The row loop is software-pipelined: while row i is
// computed, the record of the warp's next row (RW words per lane, one coalesced load) and the
// record pointer of the row after it are already in flight, so the dependent global loads
// (pointer -> record) leave the critical path; only the U1 row gathers (L2) remain on it.
//
// Output map.  The records merge the op's spatial GROUPS (terms with bitwise-proportional K_k
// share a group, and so do the r2 terms of the convection operator that share N(u_a)), at
// most TM per launch (a chunk of the op's groups).  MAP == false: the chunk's groups ARE
// terms k0 .. k0+nout-1 (coefficient 1).  MAP == true: group g < nout writes its terms
// tk[tg[g] .. tg[g+1]) as Y1[:, tk[t] r : (tk[t]+1) r] = tc[t] * (K_g U1) straight from its
// register accumulator: each product is computed once per group, the T r outputs (the
// HBM-bound part) are all written.  R = row stride of Y1.
template <int TM, bool V2, bool MAP>
__global__ void __launch_bounds__(256, 2) spmm_merged_k(int64_t n_x, int nout, int r, int64_t R,
                                                       const int64_t* __restrict__ recptr,
                                                       const long long* __restrict__ rec,
                                                       const double* __restrict__ U1,
                                                       double* __restrict__ Y1, int k0,
                                                       const int* __restrict__ tk,
                                                       const int* __restrict__ tg,
                                                       const double* __restrict__ tc) {
  static_assert(TM % 2 == 0, "TM even (16-byte value loads)");
  constexpr int RPL = V2 ? 2 : 1;
  constexpr int CW = 32 * RPL;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int UNR = V2 ? 2 : 8;  // U1 rows loaded together
  constexpr int RW = 3;   // record words per lane held in registers (96 per warp)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // per warp: the staged record, dense values [distinct column][term pair] and the distinct
  // columns (<= 32 per row: the host routes longer merged rows to the per-term kernel)
  __shared__ long long rec_all[256 / 32][32 * RW];
  __shared__ double2 vd_all[256 / 32][32][TM / 2];
  __shared__ int col_all[256 / 32][32];
  long long* rs = rec_all[threadIdx.x >> 5];
  double2 (*vd)[TM / 2] = vd_all[threadIdx.x >> 5];
  int* cols = col_all[threadIdx.x >> 5];

  auto load_rec = [&](int64_t row, int64_t p0, int64_t p1, long long* w) {
#pragma unroll
    for (int m = 0; m < RW; m++) {
      const int64_t e = lane + 32 * m;
      w[m] = (row < n_x && e < p1 - p0) ? __ldg(rec + p0 + e) : 0LL;
    }
  };
  int64_t i = warp;
  int64_t p0 = 0, p1 = 0, q0 = 0, q1 = 0;
  if (i < n_x) {
    p0 = __ldg(recptr + i);
    p1 = __ldg(recptr + i + 1);
  }
  if (i + nwarps < n_x) {
    q0 = __ldg(recptr + i + nwarps);
    q1 = __ldg(recptr + i + nwarps + 1);
  }
  long long cur[RW];
  load_rec(i, p0, p1, cur);
  for (; i < n_x; i += nwarps) {
    // pipeline: next row's record and the pointer of the row after it
    long long nxt[RW];
    load_rec(i + nwarps, q0, q1, nxt);
    int64_t s0 = 0, s1 = 0;
    if (i + 2 * nwarps < n_x) {
      s0 = __ldg(recptr + i + 2 * nwarps);
      s1 = __ldg(recptr + i + 2 * nwarps + 1);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < RW; m++) rs[lane + 32 * m] = cur[m];
    __syncwarp();
    const int gn = (int)(rs[0] >> 32);
    const int64_t row = (int64_t)(rs[0] & 0xffffffffLL);  // records are in locality order
    const long long w = lane < gn ? rs[1 + lane] : 0LL;
    const unsigned mask = (unsigned)(w >> 32);
    const int cnt = __popc(mask);
    int off = cnt;  // inclusive scan of the value counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, off, o);
      if (lane >= o) off += t;
    }
    off -= cnt;
    const int gp = (gn + UNR - 1) / UNR * UNR;  // padded to the unroll: pad slots hold zeros
    double* yrow = Y1 + row * R;
    for (int c0 = 0; c0 < r; c0 += CW) {
    if (c0 == 0 && lane < gp) {  // lane j: dense, zero-padded values of distinct column j
      const int64_t v0 = 1 + gn + off;
      // staged record, or (rows longer than 32 RW words) straight from global
      const long long* src = (p1 - p0 <= 32 * RW) ? rs + v0 : rec + p0 + v0;
      int q = 0;
#pragma unroll
      for (int k = 0; k < TM; k += 2) {
        double a = 0.0, b = 0.0;
        if (mask & (1u << k)) a = __longlong_as_double(src[q++]);
        if (mask & (2u << k)) b = __longlong_as_double(src[q++]);
        vd[lane][k / 2] = make_double2(a, b);
      }
      cols[lane] = lane < gn ? (int)(w & 0xffffffffLL) : 0;
    }
    __syncwarp();
      const int cc = c0 + (V2 ? 2 * lane : lane);
      const bool okc = cc < r;
      const double* ub = U1 + (okc ? cc : 0);
      double acc[TM][RPL];
#pragma unroll
      for (int k = 0; k < TM; k++)
#pragma unroll
        for (int q = 0; q < RPL; q++) acc[k][q] = 0.0;
      for (int j0 = 0; j0 < gp; j0 += UNR) {
        double u[UNR][RPL];
#pragma unroll
        for (int s = 0; s < UNR; s++) {
          const double* urow = ub + (int64_t)cols[j0 + s] * r;
          if (V2) {
            const double2 t = __ldg((const double2*)urow);
            u[s][0] = t.x;
            u[s][RPL - 1] = t.y;
          } else {
            u[s][0] = __ldg(urow);
          }
        }
#pragma unroll
        for (int s = 0; s < UNR; s++) {
#pragma unroll
          for (int k = 0; k < TM; k += 2) {
            const double2 v = vd[j0 + s][k / 2];
#pragma unroll
            for (int q = 0; q < RPL; q++) {
              acc[k][q] = fma(v.x, u[s][q], acc[k][q]);
              acc[k + 1][q] = fma(v.y, u[s][q], acc[k + 1][q]);
            }
          }
        }
      }
      if (MAP) {
        static_assert(!MAP || !V2, "MAP: scalar lanes");
        // group g's product goes to its terms tk[tg[g] .. tg[g+1]) (warp-uniform loads)
        if (okc) {
#pragma unroll
          for (int g = 0; g < TM; g++) {
            if (g < nout) {
              const int t1 = __ldg(tg + g + 1);
              for (int t = __ldg(tg + g); t < t1; t++)
                __stcs(yrow + (int64_t)__ldg(tk + t) * r + cc, __ldg(tc + t) * acc[g][0]);
            }
          }
        }
      } else if (okc) {
        double* dst = yrow + (int64_t)k0 * r + cc;
#pragma unroll
        for (int k = 0; k < TM; k++) {
          if (k < nout) {
            if (V2)
              __stcs((double2*)dst, make_double2(acc[k][0], acc[k][RPL - 1]));
            else
              __stcs(dst, acc[k][0]);
          }
          dst += r;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < RW; m++) cur[m] = nxt[m];
    p0 = q0;
    p1 = q1;
    q0 = s0;
    q1 = s1;
  }
}

// The diagonal blocks only (the rest of Y2 is zeroed by a memset first):
//   Y2[k r1 + a, i, k r2 + b] = sum_j G_k[i, j] U2[a, j, b]
// blockIdx.y = row k r1 + a; threads over (i, b), b fastest (coalesced U2 reads and Y2 writes,
// G_k[i, :] broadcast within a warp when r2 >= 32).
// compact != 0: write the blocks densely packed, B[k r1 + a, i, b] (T r1 x n_xi x r2), for the
// fused apply+round (the zero off-diagonal blocks are never materialised).
__global__ void stoch_apply_k(int T, int r1, int n_xi, int r2, const double* __restrict__ G,
                              const double* __restrict__ U2, double* __restrict__ Y2,
                              int compact) {
  const int row = blockIdx.y;
  const int k = row / r1, a = row % r1;
  const int64_t R2 = compact ? r2 : (int64_t)T * r2;
  const double* g = G + (int64_t)k * n_xi * n_xi;
  const double* u = U2 + (int64_t)a * n_xi * r2;
  double* y = Y2 + (int64_t)row * n_xi * R2 + (compact ? 0 : (int64_t)k * r2);
  const int n = n_xi * r2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int i = e / r2, b = e - i * r2;
    const double* gi = g + (int64_t)i * n_xi;
    double v = 0.0;
    for (int j = 0; j < n_xi; j++) v = fma(__ldg(gi + j), __ldg(u + (int64_t)j * r2 + b), v);
    y[(int64_t)i * R2 + b] = v;
  }
}

__global__ void time_apply_k(int T, int r2, int n_t, const int* __restrict__ kl,
                             const int* __restrict__ ku, const int64_t* __restrict__ band_off,
                             const double* __restrict__ band, const double* __restrict__ U3,
                             double* __restrict__ Y3) {
  const int64_t n = (int64_t)T * r2 * n_t;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e % n_t);
    const int64_t row = e / n_t;
    const int k = (int)(row / r2), b = (int)(row % r2);
    const int l = kl[k], u = ku[k], ld = l + u + 1;
    const double* bd = band + band_off[k];
    const double* x = U3 + (int64_t)b * n_t;
    double v = 0.0;
    const int s0 = max(0, t - l), s1 = min(n_t - 1, t + u);
    for (int s = s0; s <= s1; s++) v = fma(bd[(int64_t)s * ld + u + t - s], x[s], v);
    Y3[e] = v;
  }
}

}  // namespace

int tk_launch_spmm_multi(tk_ctx* ctx, const tk_op* op, int r, const double* U1, double* Y1,
                         bool grouped) {
  const int64_t n_x = op->n_x;
  const int threads = 256;
  int64_t blocks = (n_x * 32 + threads - 1) / threads;
  blocks = std::min<int64_t>(blocks, 32LL * ctx->num_sms);
  if (grouped && op->gchunks.empty()) {
    ctx->err = "spmm: this operator has no group-space records";
    return TK_EARG;
  }
  if (grouped || (!op->chunks.empty() && !op->spmm_perterm)) {
    // column-merged kernel, one launch per chunk of <= 16 groups.  grouped: the group
    // representatives only (tk_op_group_space), Y1' = [K_g U1]_g with row stride G r.
    blocks = std::min<int64_t>((n_x * 32 + threads - 1) / threads, 16LL * ctx->num_sms);
    const int64_t R = (int64_t)(grouped ? op->n_groups : op->T) * r;
    for (const SpmmChunk& c : (grouped ? op->gchunks : op->chunks)) {
      const bool map = !grouped && !c.ident;
      const int nout = c.ng;  // (MAP: the chunk's groups; their terms come from c.tg / c.tk)
      const int k0 = grouped ? c.g0 : c.k0;
      const int tm = c.ng;
#define TK_SPMM_M(TM, MP)                                                                   \
  spmm_merged_k<TM, false, MP><<<(unsigned)blocks, threads, 0, ctx->stream>>>(              \
      n_x, nout, r, R, c.recptr, (const long long*)c.rec, U1, Y1, k0, c.tk, c.tg, c.tc)
#define TK_SPMM_T(TM)            \
  if (map) TK_SPMM_M(TM, true);  \
  else TK_SPMM_M(TM, false);
      if (tm <= 2) {
        TK_SPMM_T(2)
      } else if (tm <= 4) {
        TK_SPMM_T(4)
      } else if (tm <= 6) {
        TK_SPMM_T(6)
      } else if (tm <= 8) {
        TK_SPMM_T(8)
      } else if (tm <= 10) {
        TK_SPMM_T(10)
      } else if (tm <= 12) {
        TK_SPMM_T(12)
      } else if (tm <= 14) {
        TK_SPMM_T(14)
      } else {
        TK_SPMM_T(16)
      }
#undef TK_SPMM_T
#undef TK_SPMM_M
      TK_LAUNCH_CHECK(ctx);
    }
    return TK_OK;
  }
  if (!op->rowptr) {
    ctx->err = "spmm: this operator has no per-term CSR (merged kernel only)";
    return TK_EARG;
  }
  const int rpl = (r + 31) / 32;
#define TK_SPMM(R, V)                                                                       \
  spmm_multi_k<R, V><<<(unsigned)blocks, threads, 0, ctx->stream>>>(                        \
      n_x, op->T, r, op->rowptr, op->col, op->val, op->nnz_off, U1, Y1)
  // 16-byte path: r even (row starts stay 16-byte aligned) and 16-byte aligned bases
  const bool v2 = (r % 2 == 0) && (((uintptr_t)U1 & 15) == 0) && (((uintptr_t)Y1 & 15) == 0);
  if (v2) {
    if (rpl <= 2)
      TK_SPMM(2, true);
    else if (rpl <= 4)
      TK_SPMM(4, true);
    else
      TK_SPMM(8, true);
  } else if (rpl <= 1)
    TK_SPMM(1, false);
  else if (rpl == 2)
    TK_SPMM(2, false);
  else if (rpl == 3)
    TK_SPMM(3, false);
  else if (rpl == 4)
    TK_SPMM(4, false);
  else
    TK_SPMM(8, false);
#undef TK_SPMM
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

int tk_launch_stoch_apply(tk_ctx* ctx, const tk_op* op, int r1, int r2, const double* U2,
                          double* Y2, bool compact) {
  const int64_t rows = (int64_t)op->T * r1;
  const int64_t total = rows * op->n_xi * op->T * r2;
  if (!compact) TK_TRY(tk_zero(ctx, Y2, 1, sizeof(double) * total, sizeof(double) * total));
  const int n = (int)(op->n_xi * r2);
  const int bx = std::max(1, std::min((n + 255) / 256, 8));
  if (rows > 65535) {
    ctx->err = "tk_apply_op: T * r1 exceeds the stochastic kernel's grid limit";
    return TK_EARG;
  }
  stoch_apply_k<<<dim3(bx, (unsigned)rows), 256, 0, ctx->stream>>>(op->T, r1, (int)op->n_xi, r2,
                                                                    op->G, U2, Y2, compact ? 1 : 0);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

int tk_launch_time_apply(tk_ctx* ctx, const tk_op* op, int r2, const double* U3, double* Y3) {
  int64_t n = (int64_t)op->T * r2 * op->n_t;
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16LL * ctx->num_sms));
  time_apply_k<<<blocks, 256, 0, ctx->stream>>>(op->T, r2, (int)op->n_t, op->band_kl,
                                                op->band_ku, op->band_off, op->band, U3, Y3);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_apply_k() {}
const void* tk_anchor_k_apply() { return (const void*)tk_anchor_k_apply_k; }
