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
// V T^T); trailing update and the backward accumulation of Q:
//   A[j0:, j1:] -= (V T^T) (V^T A[j0:, j1:])        Q[j0:, j0:] -= (V T) (V^T Q[j0:, j0:])
// each applied by one fused kernel (apply_reflector_k: a rank-16 update is too thin for DMMA
// tiles, and the two-GEMM form cost a split-K reduction and three launches per panel).
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

// sum_{i = i0 + lane, step 32, i < m} P[i][a] * P[i][b] for a shared-memory panel with leading
// dimension LD; four independent accumulators (the shared-memory latency, not the FMA, bounds a
// single chain).
template <int LD>
__device__ __forceinline__ double col_dot(const double* P, int a, int b, int i0, int m, int lane) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int i = i0 + lane;
  for (; i + 96 < m; i += 128) {
    s0 = fma(P[i * LD + a], P[i * LD + b], s0);
    s1 = fma(P[(i + 32) * LD + a], P[(i + 32) * LD + b], s1);
    s2 = fma(P[(i + 64) * LD + a], P[(i + 64) * LD + b], s2);
    s3 = fma(P[(i + 96) * LD + a], P[(i + 96) * LD + b], s3);
  }
  for (; i < m; i += 32) s0 = fma(P[i * LD + a], P[i * LD + b], s0);
  return (s0 + s1) + (s2 + s3);
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
// column j.  One barrier per column: after reflector c is published, every warp j > c applies it
// to its own column (w_j = tau v^T P[c:, j], P[:, j] -= w_j v) and warp c + 1 then immediately
// forms reflector c + 1 from its freshly updated column (look-ahead); warps j < c compute
// z_j = V[:, j]^T v_c for the T factor (dlarft; double-buffered so that warp 0 can form
// T[0:c, c] = -tau T[0:c, 0:c] z after the barrier while the next column proceeds).
__device__ __forceinline__ void make_reflector(double* psm, int c, int m, int lane, double* s_tau) {
  constexpr int LD = QB + 1;
  const double s = warp_sum(col_dot<LD>(psm, c, c, c + 1, m, lane));
  const double alpha = psm[c * LD + c];
  double tau = 0.0, scale = 0.0, beta = alpha;
  if (s > 0.0) {
    const double nrm = sqrt(fma(alpha, alpha, s));
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
#pragma unroll 4
  for (int i = c + 1 + lane; i < m; i += 32) psm[i * LD + c] *= scale;
  if (lane == 0) {
    psm[c * LD + c] = beta;  // R entry (unused); v_c = 1 is implicit below
    s_tau[c] = tau;
  }
}

__global__ void __launch_bounds__(32 * QB)
    qr_panel_warp_k(int m, int jb, const double* __restrict__ Pg, int64_t ldg,
                    double* __restrict__ Vout, double* __restrict__ Tout,
                    double* __restrict__ VTout, double* __restrict__ VTtout) {
  extern __shared__ double psm[];
  __shared__ double s_tau[QB], s_z[2][QB];
  __shared__ double Ts[QB][QB + 1];
  constexpr int LD = QB + 1;
  constexpr int NT = 32 * QB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // panel -> shared memory, 8 loads in flight per thread (thread's column j = tid % QB is fixed)
  {
    const int j = tid % QB;
    for (int i0 = tid / QB; i0 < m; i0 += 8 * (NT / QB)) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        v[u] = (i < m && j < jb) ? Pg[(int64_t)i * ldg + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        if (i < m) psm[i * LD + j] = v[u];
      }
    }
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  if (warp == 0 && jb > 0) make_reflector(psm, 0, m, lane, s_tau);
  __syncthreads();
  for (int c = 0; c < jb; c++) {
    const double tau = s_tau[c];
    if (warp > c && warp < jb) {
      const int j = warp;
      // row c counted once (v_c = 1)
      double w = col_dot<LD>(psm, c, j, c + 1, m, lane) + (lane == 0 ? psm[c * LD + j] : 0.0);
      w = warp_sum(w) * tau;
      if (lane == 0) psm[c * LD + j] -= w;
#pragma unroll 4
      for (int i = c + 1 + lane; i < m; i += 32) psm[i * LD + j] = fma(-w, psm[i * LD + c], psm[i * LD + j]);
      __syncwarp();
      if (j == c + 1) make_reflector(psm, j, m, lane, s_tau);
    } else if (warp < c) {
      const int j = warp;
      // z_j = V[:, j]^T v over rows >= c (v is zero above c; V[c, j] is stored below diag j)
      double z = col_dot<LD>(psm, j, c, c + 1, m, lane) + (lane == 0 ? psm[c * LD + j] : 0.0);
      z = warp_sum(z);
      if (lane == 0) s_z[c & 1][j] = z;
    }
    __syncthreads();
    if (warp == 0) {
      if (lane < c) {
        double t = 0.0;
        for (int q = lane; q < c; q++) t = fma(Ts[lane][q], s_z[c & 1][q], t);
        Ts[lane][c] = -tau * t;
      }
      if (lane == 0) Ts[c][c] = tau;
    }
  }
  __syncthreads();
  // V (unit lower trapezoidal) into shared memory in place, then V, V T and V T^T out; the
  // thread's column j = tid % QB is fixed, so column j and row j of T stay in registers
  const int j = tid % QB;
  double tc[QB], tr[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) {
    tc[q] = Ts[q][j];
    tr[q] = Ts[j][q];
  }
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB;
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
    const int i = e / QB;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int q = 0; q < QB; q++) {
      const double v = psm[i * LD + q];
      a = fma(v, tc[q], a);
      b = fma(v, tr[q], b);
    }
    VTout[e] = a;
    VTtout[e] = b;
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Tout[e] = Ts[e / QB][e % QB];
}

// C <- C - X (V^T C) for the m x nc block C (leading dimension ldc) and the m x QB panels V, X
// (row-major, ld QB): the compact-WY application of one panel's block reflector (X = V T^T for
// the trailing update, X = V T for the accumulation of Q), fused into one kernel.  CTA = a strip
// of AR_W columns; phase 1 forms W = V^T C[:, strip] (QB x AR_W) with the rows split over the 8
// warps and reduced in shared memory, phase 2 updates the strip row by row.  Rows of V and X
// are warp-uniform (broadcast loads), C accesses are coalesced along the strip.
constexpr int AR_W = 4, AR_T = 256, AR_G = AR_T / AR_W, AR_U = 4;
__global__ void __launch_bounds__(AR_T) apply_reflector_k(int m, int nc, const double* __restrict__ V,
                                                          const double* __restrict__ X,
                                                          double* __restrict__ C, int64_t ldc) {
  __shared__ double red[AR_G][QB][AR_W];
  __shared__ double Ws[QB][AR_W];
  const int col = threadIdx.x % AR_W, rg = threadIdx.x / AR_W;
  const int gc = blockIdx.x * AR_W + col;
  const bool live = gc < nc;
  double acc[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) acc[q] = 0.0;
  // AR_U rows per iteration: their loads are independent (memory-level parallelism)
  for (int i0 = rg; i0 < m; i0 += AR_G * AR_U) {
    double c[AR_U];
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = i0 + u * AR_G;
      c[u] = (live && i < m) ? C[(int64_t)i * ldc + gc] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = min(i0 + u * AR_G, m - 1);
      const double2* vr = reinterpret_cast<const double2*>(V + (int64_t)i * QB);
#pragma unroll
      for (int q = 0; q < QB / 2; q++) {
        const double2 v = __ldg(vr + q);
        acc[2 * q] = fma(v.x, c[u], acc[2 * q]);
        acc[2 * q + 1] = fma(v.y, c[u], acc[2 * q + 1]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < QB; q++) red[rg][q][col] = acc[q];
  __syncthreads();
  for (int e = threadIdx.x; e < QB * AR_W; e += AR_T) {
    const int q = e / AR_W, cc = e % AR_W;
    double t = 0.0;
#pragma unroll
    for (int g = 0; g < AR_G; g++) t += red[g][q][cc];
    Ws[q][cc] = t;
  }
  __syncthreads();
  double w[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) w[q] = Ws[q][col];
  if (!live) return;
  for (int i0 = rg; i0 < m; i0 += AR_G * AR_U) {
    double d[AR_U];
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = min(i0 + u * AR_G, m - 1);
      const double2* xr = reinterpret_cast<const double2*>(X + (int64_t)i * QB);
      d[u] = 0.0;
#pragma unroll
      for (int q = 0; q < QB / 2; q++) {
        const double2 x = __ldg(xr + q);
        d[u] = fma(x.x, w[2 * q], d[u]);
        d[u] = fma(x.y, w[2 * q + 1], d[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = i0 + u * AR_G;
      if (i < m) C[(int64_t)i * ldc + gc] -= d[u];
    }
  }
}

}  // namespace

// Q (n x n, row-major) from the Householder QR of A (n x n, row-major; A is not modified).
int tk_householder_q(tk_ctx* ctx, int n, const double* A, double* Q) {
  if (n <= 0) return TK_OK;
  DevBuf Aw, Vb, Tb, VTb, VTtb;
  TK_TRY(Aw.get(ctx, (size_t)n * n));
  TK_CUDA_TRY(ctx, cudaMemcpyAsync(Aw.p, A, sizeof(double) * n * n, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
  const int np = (n + QB - 1) / QB;
  // panel p: V, V T, V T^T as (n - j0) x QB at offset p*n*QB;  T: QB x QB
  TK_TRY(Vb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTtb.get(ctx, (size_t)np * n * QB));
  TK_TRY(Tb.get(ctx, (size_t)np * QB * QB));
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
      const int rid = tk_prof_begin(ctx, "qr_reflector", 4.0 * m * (double)nt * QB, 0.0);
      apply_reflector_k<<<(nt + AR_W - 1) / AR_W, AR_T, 0, ctx->stream>>>(m, nt, Vp, VTtp, At, n);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, rid);
    }
  }
  // Q = H_1 ... H_np : backward accumulation from the identity, Qs <- Qs - (V T) (V^T Qs)
  TK_TRY(tk_eye(ctx, Q, n));
  for (int p = np - 1; p >= 0; p--) {
    const int j0 = p * QB, m = n - j0;
    double* Vp = Vb.p + (size_t)p * n * QB;
    double* VTp = VTb.p + (size_t)p * n * QB;
    double* Qs = Q + (int64_t)j0 * n + j0;
    const int rid = tk_prof_begin(ctx, "qr_reflector", 4.0 * m * (double)m * QB, 0.0);
    apply_reflector_k<<<(m + AR_W - 1) / AR_W, AR_T, 0, ctx->stream>>>(m, m, Vp, VTp, Qs, n);
    TK_LAUNCH_CHECK(ctx);
    tk_prof_end(ctx, rid);
  }
  return TK_OK;
}
