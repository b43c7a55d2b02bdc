// Symmetric eigen-decomposition by two-sided BLOCK Jacobi (fp64, on device).
//
// Used for the small R x R Gram matrices of the rounding: pass 1
// needs an ORTHOGONAL eigenbasis to absolute accuracy, pass 2 needs eigenvalues with
// RELATIVE accuracy on a graded matrix — Jacobi with the relative skip test
// |a_pq| <= rel * sqrt(|a_pp a_qq|) provides that (Demmel-Veselic), tridiagonal QR does not.
//
// Layout: the matrix is embedded in an n_pad x n_pad buffer (n_pad = 64 * ceil(n/64), zero
// padding — padded indices never rotate since their couplings are 0), split into
// nb = n_pad/32 blocks of 32 rows/cols.  One sweep = nb-1 rounds of a round-robin
// tournament over blocks; a round handles nb/2 disjoint block pairs (I, J):
//   inner_k      one CTA per pair: load S = G[I u J, I u J] (64 x 64) into shared memory,
//                run scalar cyclic Jacobi on it (parallel ordering, Rutishauser updates of
//                each 2x2 pivot block) accumulating Q (64 x 64); write Q and the rotated S.
//   col_update_k G[:, I u J] <- G[:, I u J] Q  and  V[:, I u J] <- V[:, I u J] Q
//   row_update_k G[I u J, :] <- Q^T G[I u J, :]  (the pair's own 64 x 64 block takes the
//                inner solver's S, so its annihilated entries stay exactly 0)
// Three launches per round; a per-sweep rotation counter (read by the host) ends the loop.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ttk_internal.h"

namespace {

constexpr int JB = 32;        // block size
constexpr int JS = 2 * JB;    // pair size (64)
constexpr int JLD = JS + 1;   // shared-memory leading dimension
constexpr int JT = 256;       // threads per CTA (update kernels)
constexpr int JTI = 512;      // threads per CTA (inner solver)

__host__ __device__ __forceinline__ int rr_player(int pos, int r, int ne) {
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (ne - 1);
}

__device__ __forceinline__ void pair_blocks(int t, int r, int nb, int& I, int& J) {
  int a = rr_player(t, r, nb), b = rr_player(nb - 1 - t, r, nb);
  I = min(a, b);
  J = max(a, b);
}
// global index of local index l (0..63) of the pair (I, J)
__device__ __forceinline__ int gidx(int l, int I, int J) {
  return l < JB ? I * JB + l : J * JB + (l - JB);
}

__global__ void __launch_bounds__(JTI) inner_k(int n_pad, const double* __restrict__ G,
                                               double* __restrict__ Qout, double* __restrict__ Sout,
                                               int* __restrict__ skip, int r, int nb,
                                               const double* __restrict__ d_maxdiag,
                                               double abs_scale, double rel_tol, int max_inner,
                                               int* __restrict__ counter) {
  extern __shared__ double sm[];
  double* S = sm;                 // [64][65]
  double* Q = sm + JS * JLD;      // [64][65]
  __shared__ double rc[JB], rs[JB], rt[JB], rapp[JB], raqq[JB], rapq[JB];
  __shared__ int rp_[JB], rq_[JB], ract[JB];
  __shared__ int nrot;
  const int t = blockIdx.x;
  int I, J;
  pair_blocks(t, r, nb, I, J);
  const double abs_tol = fmax(abs_scale * d_maxdiag[0], 1e-300);
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    int gi = gidx(i, I, J), gj = gidx(j, I, J);
    double v = 0.5 * (G[(int64_t)gi * n_pad + gj] + G[(int64_t)gj * n_pad + gi]);
    S[i * JLD + j] = v;
    Q[i * JLD + j] = (i == j) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) nrot = 0;
  __syncthreads();
  // already converged block pair (every |s_ij| below its skip threshold): no rotation
  {
    int any = 0;
    for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
      int i = e / JS, j = e % JS;
      if (j <= i) continue;
      double thr = fmax(abs_tol, rel_tol * sqrt(fabs(S[i * JLD + i] * S[j * JLD + j])));
      any |= fabs(S[i * JLD + j]) > thr;
    }
    if (!__syncthreads_or(any)) {
      if (threadIdx.x == 0) skip[t] = 1;
      return;
    }
    if (threadIdx.x == 0) skip[t] = 0;
  }
  for (int sweep = 0; sweep < max_inner; sweep++) {
    const int before = nrot;
    __syncthreads();
    for (int ir = 0; ir < JS - 1; ir++) {
      // (a) rotation parameters of the 32 disjoint pairs of this inner round
      if (threadIdx.x < JB) {
        const int k = threadIdx.x;
        int a = rr_player(k, ir, JS), b = rr_player(JS - 1 - k, ir, JS);
        int p = min(a, b), q = max(a, b);
        double app = S[p * JLD + p], aqq = S[q * JLD + q], apq = S[p * JLD + q];
        double c = 1.0, s = 0.0, tt = 0.0;
        int act = 0;
        double thr = fmax(abs_tol, rel_tol * sqrt(fabs(app * aqq)));
        if (fabs(apq) > thr) {
          double theta = (aqq - app) / (2.0 * apq);
          double at = fabs(theta);
          if (at > 1e150) {
            tt = 0.5 / theta;
          } else {
            tt = 1.0 / (at + sqrt(1.0 + at * at));
            if (theta < 0) tt = -tt;
          }
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
          act = 1;
        }
        rc[k] = c;
        rs[k] = s;
        rt[k] = tt;
        rapp[k] = app;
        raqq[k] = aqq;
        rapq[k] = apq;
        rp_[k] = p;
        rq_[k] = q;
        ract[k] = act;
        const unsigned bal = __ballot_sync(0xffffffffu, act);
        if (k == 0) nrot += __popc(bal);
      }
      __syncthreads();
      // (b) column update of S and Q:  (x_p, x_q) <- (c x_p - s x_q, s x_p + c x_q)
      for (int e = threadIdx.x; e < JB * JS; e += blockDim.x) {
        const int pr = e / JS, i = e % JS;
        if (!ract[pr]) continue;
        const int p = rp_[pr], q = rq_[pr];
        const double c = rc[pr], s = rs[pr];
        double sp = S[i * JLD + p], sq = S[i * JLD + q];
        S[i * JLD + p] = c * sp - s * sq;
        S[i * JLD + q] = s * sp + c * sq;
        double qp = Q[i * JLD + p], qq = Q[i * JLD + q];
        Q[i * JLD + p] = c * qp - s * qq;
        Q[i * JLD + q] = s * qp + c * qq;
      }
      __syncthreads();
      // (c) row update of S; the 2x2 pivot block takes Rutishauser's values
      for (int e = threadIdx.x; e < JB * JS; e += blockDim.x) {
        const int pr = e / JS, j = e % JS;
        if (!ract[pr]) continue;
        const int p = rp_[pr], q = rq_[pr];
        if (j == p) {
          S[p * JLD + p] = rapp[pr] - rt[pr] * rapq[pr];
          S[q * JLD + p] = 0.0;
        } else if (j == q) {
          S[q * JLD + q] = raqq[pr] + rt[pr] * rapq[pr];
          S[p * JLD + q] = 0.0;
        } else {
          const double c = rc[pr], s = rs[pr];
          double sp = S[p * JLD + j], sq = S[q * JLD + j];
          S[p * JLD + j] = c * sp - s * sq;
          S[q * JLD + j] = s * sp + c * sq;
        }
      }
      __syncthreads();
    }
    const bool done = (nrot == before);
    __syncthreads();
    if (done) break;
  }
  // write Q and S (rotated pair block)
  double* Qo = Qout + (int64_t)t * JS * JS;
  double* So = Sout + (int64_t)t * JS * JS;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    Qo[e] = Q[i * JLD + j];
    So[e] = S[i * JLD + j];
  }
  if (threadIdx.x == 0 && nrot) atomicAdd(counter, nrot);
}

// G[:, I u J] <- G[:, I u J] Q (z = 0),  V[:, I u J] <- V[:, I u J] Q (z = 1)
__global__ void __launch_bounds__(JT) col_update_k(int n_pad, double* __restrict__ G,
                                                   double* __restrict__ V,
                                                   const double* __restrict__ Qall,
                                                   const int* __restrict__ skip, int r, int nb) {
  extern __shared__ double dsm[];
  double(*Qs)[JS + 1] = reinterpret_cast<double(*)[JS + 1]>(dsm);
  double(*Ts)[JS + 1] = reinterpret_cast<double(*)[JS + 1]>(dsm + JS * (JS + 1));
  const int t = blockIdx.y;
  if (skip[t]) return;
  int I, J;
  pair_blocks(t, r, nb, I, J);
  double* M = blockIdx.z == 0 ? G : V;
  const int row0 = blockIdx.x * JS;
  const double* Q = Qall + (int64_t)t * JS * JS;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    Qs[i][j] = Q[e];
    Ts[i][j] = M[(int64_t)(row0 + i) * n_pad + gidx(j, I, J)];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    double acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < JS; k++) acc = fma(Ts[i][k], Qs[k][j], acc);
    M[(int64_t)(row0 + i) * n_pad + gidx(j, I, J)] = acc;
  }
}

// G[I u J, :] <- Q^T G[I u J, :]; the pair's own columns take the inner solver's S
__global__ void __launch_bounds__(JT) row_update_k(int n_pad, double* __restrict__ G,
                                                   const double* __restrict__ Qall,
                                                   const double* __restrict__ Sall,
                                                   const int* __restrict__ skip, int r, int nb) {
  extern __shared__ double dsm[];
  double(*Qs)[JS + 1] = reinterpret_cast<double(*)[JS + 1]>(dsm);
  double(*Ts)[JS + 1] = reinterpret_cast<double(*)[JS + 1]>(dsm + JS * (JS + 1));
  const int t = blockIdx.y;
  if (skip[t]) return;
  int I, J;
  pair_blocks(t, r, nb, I, J);
  const int col0 = blockIdx.x * JS;
  const double* Q = Qall + (int64_t)t * JS * JS;
  const double* S = Sall + (int64_t)t * JS * JS;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    Qs[i][j] = Q[e];
    Ts[i][j] = G[(int64_t)gidx(i, I, J) * n_pad + col0 + j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    int gc = col0 + j;
    int bc = gc / JB;
    double v;
    if (bc == I || bc == J) {
      int lj = (bc == I) ? gc - I * JB : JB + gc - J * JB;
      v = S[i * JS + lj];
    } else {
      v = 0.0;
#pragma unroll 8
      for (int k = 0; k < JS; k++) v = fma(Qs[k][i], Ts[k][j], v);
    }
    G[(int64_t)gidx(i, I, J) * n_pad + gc] = v;
  }
}

__global__ void embed_k(int n, int n_pad, const double* __restrict__ A, double* __restrict__ G,
                        double* __restrict__ V) {
  int64_t nn = (int64_t)n_pad * n_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn;
       e += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(e / n_pad), j = (int)(e % n_pad);
    G[e] = (i < n && j < n) ? A[(int64_t)i * n + j] : 0.0;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
}

// Sort eigenvalues descending (stable by index) and permute eigenvector columns.
__global__ void eig_sort_k(int n, int n_pad, const double* __restrict__ G,
                           const double* __restrict__ Vp, double* __restrict__ lam,
                           double* __restrict__ Vout) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double li = G[(int64_t)i * n_pad + i];
    int rank = 0;
    for (int j = 0; j < n; j++) {
      double lj = G[(int64_t)j * n_pad + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    lam[rank] = li;
    for (int k = 0; k < n; k++) Vout[(int64_t)k * n + rank] = Vp[(int64_t)k * n_pad + i];
  }
}

__global__ void max_abs_diag_k(int n, const double* A, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(A[(int64_t)i * n + i]));
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

}  // namespace

int tk_jacobi_eig(tk_ctx* ctx, int n, double* A, double* lam, double* V, double abs_tol_scale,
                  double rel_tol, int max_sweeps, int* sweeps_out) {
  if (n <= 0) return TK_OK;
  const int n_pad = ((n + JS - 1) / JS) * JS;
  const int nb = n_pad / JB;
  const int npairs = nb / 2;
  DevBuf Gp, Vp, Qb, Sb, scr;
  TK_TRY(Gp.get(ctx, (size_t)n_pad * n_pad));
  TK_TRY(Vp.get(ctx, (size_t)n_pad * n_pad));
  TK_TRY(Qb.get(ctx, (size_t)npairs * JS * JS));
  TK_TRY(Sb.get(ctx, (size_t)npairs * JS * JS));
  TK_TRY(scr.get(ctx, 2 + (size_t)max_sweeps));
  double* d_maxdiag = scr.p;
  int* counters = (int*)(scr.p + 1);
  TK_CUDA_TRY(ctx, cudaMemsetAsync(counters, 0, sizeof(int) * (max_sweeps + 1), ctx->stream));
  const int prof_id = tk_prof_begin(ctx, "jacobi", 0.0, 0.0);
  max_abs_diag_k<<<1, 256, 0, ctx->stream>>>(n, A, d_maxdiag);
  TK_LAUNCH_CHECK(ctx);
  {
    int64_t nn = (int64_t)n_pad * n_pad;
    int g = (int)std::min<int64_t>((nn + 255) / 256, 8LL * ctx->num_sms);
    embed_k<<<g, 256, 0, ctx->stream>>>(n, n_pad, A, Gp.p, Vp.p);
    TK_LAUNCH_CHECK(ctx);
  }
  static bool attr = false;
  const size_t ismem = 2 * (size_t)JS * JLD * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(inner_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem);
    cudaFuncSetAttribute(col_update_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem);
    cudaFuncSetAttribute(row_update_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ismem);
    attr = true;
  }
  DevBuf skipb;
  TK_TRY(skipb.get(ctx, (size_t)npairs));
  int* skip = (int*)skipb.p;
  // a single pair (n <= 64) is solved completely by the inner solver; otherwise one inner
  // sweep per block pair and round (classical block Jacobi)
  const int max_inner = (npairs == 1) ? 60 : 1;
  int sweep = 0;
  for (; sweep < max_sweeps; sweep++) {
    for (int r = 0; r < nb - 1; r++) {
      inner_k<<<npairs, JTI, ismem, ctx->stream>>>(n_pad, Gp.p, Qb.p, Sb.p, skip, r, nb,
                                                  d_maxdiag, abs_tol_scale, rel_tol, max_inner,
                                                  counters + sweep);
      TK_LAUNCH_CHECK(ctx);
      col_update_k<<<dim3(n_pad / JS, npairs, 2), JT, ismem, ctx->stream>>>(n_pad, Gp.p, Vp.p,
                                                                           Qb.p, skip, r, nb);
      TK_LAUNCH_CHECK(ctx);
      row_update_k<<<dim3(n_pad / JS, npairs), JT, ismem, ctx->stream>>>(n_pad, Gp.p, Qb.p, Sb.p,
                                                                        skip, r, nb);
      TK_LAUNCH_CHECK(ctx);
    }
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, counters + sweep, sizeof(int),
                                     cudaMemcpyDeviceToHost, ctx->stream));
    TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const int rot = *(int*)ctx->pinned;
    if (rot == 0 || (npairs == 1 && sweep == 0)) {
      sweep++;
      break;
    }
  }
  int sg = (int)std::min<int64_t>((n + 127) / 128, 4LL * ctx->num_sms);
  eig_sort_k<<<sg, 128, 0, ctx->stream>>>(n, n_pad, Gp.p, Vp.p, lam, V);
  TK_LAUNCH_CHECK(ctx);
  tk_prof_end(ctx, prof_id);
  if (sweeps_out) *sweeps_out = sweep;
  if (getenv("TTK_DEBUG")) fprintf(stderr, "[ttk] jacobi n=%d sweeps=%d rel=%g\n", n, sweep, rel_tol);
  return TK_OK;
}
