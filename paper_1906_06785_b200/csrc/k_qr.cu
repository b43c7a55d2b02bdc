// Blocked Householder QR of a square fp64 matrix, returning the explicit orthogonal Q.
//
// Used as PASS 1 of the two-pass Gram-Jacobi rounding: for the Gram
// G = Z^T Z, Q from G = Q R is one step of orthogonal iteration, i.e. an exactly orthogonal
// basis whose leading columns already follow the dominant eigenvectors; W = Z Q is then
// graded enough that pass 2 (relative Jacobi on W^T W) converges in a few sweeps.  Only the
// orthogonality of Q matters for accuracy (Householder: ||Q^T Q - I|| = O(eps)).
//
// Panel (width QB = 16) factorised by one CTA (LAPACK dgeqr2 + dlarft: reflectors v_c, tau_c
// and the compact-WY factor T with H_1..H_QB = I - V T V^T; the panel kernel also emits V T and
// V T^T); trailing update and the backward accumulation of Q are two DMMA GEMMs each:
//   A[j0:, j1:] -= (V T^T) (V^T A[j0:, j1:])        Q[j0:, j0:] -= (V T) (V^T Q[j0:, j0:])
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "ttk_internal.h"

namespace {

constexpr int QB = 16;     // panel width
constexpr int QT = 512;    // threads of the panel kernel

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Factor the m x jb panel P (row-major, leading dimension ld).  SMEM: the panel is staged in
// shared memory (stride QB+1: conflict-free column access); otherwise it is worked on in global
// memory in place.  Outputs: Vout (m x QB row-major, unit lower trapezoidal, zero padded) and
// Tout (QB x QB).  The R factor is not needed (only Q is used) and is not written back.
template <bool SMEM>
__global__ void __launch_bounds__(QT) qr_panel_k(int m, int jb, double* __restrict__ Pg,
                                                 int64_t ldg, double* __restrict__ Vout,
                                                 double* __restrict__ Tout) {
  extern __shared__ double psm[];
  __shared__ double red[QT / 32][QB + 1];
  __shared__ double s_tau[QB], s_w[QB], s_beta, s_scale;
  __shared__ double Ts[QB][QB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  double* P = SMEM ? psm : Pg;
  const int64_t ld = SMEM ? (QB + 1) : ldg;
  if (SMEM) {
    for (int e = tid; e < m * QB; e += blockDim.x) {
      const int i = e / QB, j = e % QB;
      psm[i * (QB + 1) + j] = (j < jb) ? Pg[(int64_t)i * ldg + j] : 0.0;
    }
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  for (int c = 0; c < jb; c++) {
    // ---- norm of x = P[c:, c]
    double s = 0.0;
    for (int i = c + 1 + tid; i < m; i += blockDim.x) {
      double v = P[(int64_t)i * ld + c];
      s += v * v;
    }
    s = warp_sum(s);
    if (lane == 0) red[warp][0] = s;
    __syncthreads();
    if (tid == 0) {
      double sig = 0.0;
      for (int w = 0; w < nw; w++) sig += red[w][0];
      double alpha = P[(int64_t)c * ld + c];
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (sig > 0.0) {
        double nrm = sqrt(alpha * alpha + sig);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      s_tau[c] = tau;
      s_beta = beta;
      s_scale = scale;
    }
    __syncthreads();
    const double tau = s_tau[c], scale = s_scale;
    // ---- v = [1; x[1:] * scale] into P[c:, c] (below diagonal)
    for (int i = c + 1 + tid; i < m; i += blockDim.x) P[(int64_t)i * ld + c] *= scale;
    if (tid == 0) P[(int64_t)c * ld + c] = s_beta;
    __syncthreads();
    // ---- w_j = v^T P[c:, j] for j > c  and  z_l = V[:, l]^T v for l < c (T column)
    {
      double accw[QB], accz[QB];
#pragma unroll
      for (int j = 0; j < QB; j++) accw[j] = accz[j] = 0.0;
      for (int i = c + tid; i < m; i += blockDim.x) {
        const double* row = P + (int64_t)i * ld;
        const double vi = (i == c) ? 1.0 : row[c];
#pragma unroll
        for (int j = 0; j < QB; j++) {
          if (j > c && j < jb) accw[j] += vi * row[j];
          if (j < c) accz[j] += (i == j ? 1.0 : row[j]) * vi;
        }
      }
#pragma unroll
      for (int j = 0; j < QB; j++) {
        double a = warp_sum(accw[j]);
        double b = warp_sum(accz[j]);
        if (lane == 0) red[warp][j] = (j > c) ? a : b;
      }
    }
    __syncthreads();
    if (tid < QB) {
      double t = 0.0;
      for (int w = 0; w < nw; w++) t += red[w][tid];
      s_w[tid] = t;  // j > c: w_j ; j < c: z_j
    }
    __syncthreads();
    // ---- apply H_c to the remaining panel columns: P[c:, j] -= tau v w_j
    for (int e = tid; e < (m - c) * QB; e += blockDim.x) {
      const int i = c + e / QB, j = e % QB;
      if (j <= c || j >= jb) continue;
      const double vi = (i == c) ? 1.0 : P[(int64_t)i * ld + c];
      P[(int64_t)i * ld + j] -= tau * vi * s_w[j];
    }
    // ---- T column c (dlarft, forward, columnwise): T[0:c, c] = -tau T[0:c, 0:c] z
    if (tid < c) {
      double t = 0.0;
      for (int q = tid; q < c; q++) t += Ts[tid][q] * s_w[q];
      Ts[tid][c] = -tau * t;
    }
    if (tid == 0) Ts[c][c] = tau;
    __syncthreads();
  }
  // ---- export V (unit lower trapezoidal) and T
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB, j = e % QB;
    double v = 0.0;
    if (j < jb) {
      if (i == j)
        v = 1.0;
      else if (i > j)
        v = P[(int64_t)i * ld + j];
    }
    Vout[e] = v;
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Tout[e] = Ts[e / QB][e % QB];
}

// Warp-per-column panel factorisation (panel staged in shared memory, stride QB+1): warp j owns
// column j.  Per column c: warp c forms the reflector (norm, tau, v = x / (alpha - beta)); after
// one barrier every warp j > c computes w_j = v^T P[c:, j] and updates its own column, and every
// warp j < c computes z_j = V[:, j]^T v for the T factor (dlarft); after a second barrier warp 0
// forms T[0:c, c] = -tau T[0:c, 0:c] z.  Two barriers per column, no block-wide reductions.
__global__ void __launch_bounds__(32 * QB)
    qr_panel_warp_k(int m, int jb, const double* __restrict__ Pg, int64_t ldg,
                    double* __restrict__ Vout, double* __restrict__ Tout,
                    double* __restrict__ VTout, double* __restrict__ VTtout) {
  extern __shared__ double psm[];
  __shared__ double s_tau[QB], s_z[QB];
  __shared__ double Ts[QB][QB + 1];
  constexpr int LD = QB + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB, j = e % QB;
    psm[i * LD + j] = (j < jb) ? Pg[(int64_t)i * ldg + j] : 0.0;
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  for (int c = 0; c < jb; c++) {
    if (warp == c) {
      double s = 0.0;
      for (int i = c + 1 + lane; i < m; i += 32) {
        const double v = psm[i * LD + c];
        s = fma(v, v, s);
      }
      s = warp_sum(s);
      const double alpha = psm[c * LD + c];
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (s > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, s));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int i = c + 1 + lane; i < m; i += 32) psm[i * LD + c] *= scale;
      if (lane == 0) {
        psm[c * LD + c] = beta;  // R entry (unused); v_c = 1 is implicit below
        s_tau[c] = tau;
      }
    }
    __syncthreads();
    const double tau = s_tau[c];
    if (warp > c && warp < jb) {
      const int j = warp;
      double w = lane == 0 ? psm[c * LD + j] : 0.0;  // row c (v_c = 1), counted once
      for (int i = c + 1 + lane; i < m; i += 32) w = fma(psm[i * LD + c], psm[i * LD + j], w);
      w = warp_sum(w) * tau;
      if (lane == 0) psm[c * LD + j] -= w;
      for (int i = c + 1 + lane; i < m; i += 32) psm[i * LD + j] = fma(-w, psm[i * LD + c], psm[i * LD + j]);
    } else if (warp < c) {
      const int j = warp;
      // z_j = V[:, j]^T v over rows >= c (v is zero above c; V[c, j] is stored below diag j)
      double z = lane == 0 ? psm[c * LD + j] : 0.0;  // row c (v_c = 1), counted once
      for (int i = c + 1 + lane; i < m; i += 32) z = fma(psm[i * LD + j], psm[i * LD + c], z);
      z = warp_sum(z);
      if (lane == 0) s_z[j] = z;
    }
    __syncthreads();
    if (warp == 0) {
      if (lane < c) {
        double t = 0.0;
        for (int q = lane; q < c; q++) t = fma(Ts[lane][q], s_z[q], t);
        Ts[lane][c] = -tau * t;
      }
      if (lane == 0) Ts[c][c] = tau;
    }
  }
  __syncthreads();
  // V (unit lower trapezoidal) into shared memory in place, then V, V T and V T^T out
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB, j = e % QB;
    double v = 0.0;
    if (j < jb) {
      if (i == j)
        v = 1.0;
      else if (i > j)
        v = psm[i * LD + j];
    }
    psm[i * LD + j] = v;
    Vout[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB, j = e % QB;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int q = 0; q < QB; q++) {
      const double v = psm[i * LD + q];
      a = fma(v, Ts[q][j], a);
      b = fma(v, Ts[j][q], b);
    }
    VTout[e] = a;
    VTtout[e] = b;
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Tout[e] = Ts[e / QB][e % QB];
}

}  // namespace

// Q (n x n, row-major) from the Householder QR of A (n x n, row-major; A is not modified).
int tk_householder_q(tk_ctx* ctx, int n, const double* A, double* Q) {
  if (n <= 0) return TK_OK;
  TagScope tag(ctx, "qr_pass1.gemm");
  DevBuf Aw, Vb, Tb, VTb, VTtb, W1;
  TK_TRY(Aw.get(ctx, (size_t)n * n));
  TK_CUDA_TRY(ctx, cudaMemcpyAsync(Aw.p, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
  const int np = (n + QB - 1) / QB;
  // panel p: V, V T, V T^T as (n - j0) x QB at offset p*n*QB;  T: QB x QB
  TK_TRY(Vb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTtb.get(ctx, (size_t)np * n * QB));
  TK_TRY(Tb.get(ctx, (size_t)np * QB * QB));
  TK_TRY(W1.get(ctx, (size_t)QB * n));
  for (int p = 0; p < np; p++) {
    const int j0 = p * QB, jb = std::min(QB, n - j0), m = n - j0;
    double* Vp = Vb.p + (size_t)p * n * QB;
    double* VTp = VTb.p + (size_t)p * n * QB;
    double* VTtp = VTtb.p + (size_t)p * n * QB;
    double* Tp = Tb.p + (size_t)p * QB * QB;
    const int pid = tk_prof_begin(ctx, "qr_panel", 2.0 * m * (double)jb * jb, 0.0);
    const size_t psmem = (size_t)m * (QB + 1) * sizeof(double);
    if (psmem <= 200 * 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(qr_panel_warp_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
        attr = true;
      }
      qr_panel_warp_k<<<1, 32 * QB, psmem, ctx->stream>>>(m, jb, Aw.p + (int64_t)j0 * n + j0, n,
                                                          Vp, Tp, VTp, VTtp);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
    } else {
      qr_panel_k<false><<<1, QT, 0, ctx->stream>>>(m, jb, Aw.p + (int64_t)j0 * n + j0, n, Vp, Tp);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      TK_TRY(tk_dgemm(ctx, false, false, m, QB, QB, 1.0, Vp, QB, Tp, QB, 0.0, VTp, QB));
      TK_TRY(tk_dgemm(ctx, false, true, m, QB, QB, 1.0, Vp, QB, Tp, QB, 0.0, VTtp, QB));
    }
    const int nt = n - (j0 + jb);
    if (nt > 0) {
      // A_t <- H_p^T A_t = A_t - (V T^T) (V^T A_t)
      double* At = Aw.p + (int64_t)j0 * n + j0 + jb;
      TK_TRY(tk_dgemm(ctx, true, false, QB, nt, m, 1.0, Vp, QB, At, n, 0.0, W1.p, nt));
      TK_TRY(tk_dgemm(ctx, false, false, m, nt, QB, -1.0, VTtp, QB, W1.p, nt, 1.0, At, n));
    }
  }
  // Q = H_1 ... H_np : backward accumulation from the identity, Qs <- Qs - (V T) (V^T Qs)
  TK_TRY(tk_eye(ctx, Q, n));
  for (int p = np - 1; p >= 0; p--) {
    const int j0 = p * QB, m = n - j0;
    double* Vp = Vb.p + (size_t)p * n * QB;
    double* VTp = VTb.p + (size_t)p * n * QB;
    double* Qs = Q + (int64_t)j0 * n + j0;
    TK_TRY(tk_dgemm(ctx, true, false, QB, m, m, 1.0, Vp, QB, Qs, n, 0.0, W1.p, m));
    TK_TRY(tk_dgemm(ctx, false, false, m, m, QB, -1.0, VTp, QB, W1.p, m, 1.0, Qs, n));
  }
  return TK_OK;
}
