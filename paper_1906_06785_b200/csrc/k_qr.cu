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

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ttk_internal.h"

namespace {

constexpr int QB = 16;     // panel width
constexpr int kQrPoll = 8; // host polls of the early-stop flag every kQrPoll panels
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
                    double* __restrict__ VTout, double* __restrict__ VTtout,
                    const double* __restrict__ Vprev, const double* __restrict__ VTtprev,
                    unsigned long long* __restrict__ dbg) {
  // Vprev / VTtprev (nullable): the previous panel's reflector block, still to be applied to
  // this panel's columns (look-ahead without a separate launch).  Then Pg points QB rows higher
  // (the previous panel's diagonal row) and m + QB rows are loaded; H_prev = I - V T V^T acts
  // on all of them, and the factorisation proceeds on the lower m rows.
  extern __shared__ double psm_all[];
  __shared__ double s_tau[QB], s_z[QB][QB];
  __shared__ double Ts[QB][QB + 1];
  __shared__ double s_w[QB][QB + 1];
  auto stamp = [&](int k) {
    if (dbg && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[k] = t;
    }
  };
  stamp(0);
  constexpr int LD = QB + 1;
  constexpr int NT = 32 * QB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int off = Vprev ? QB : 0;  // extra leading rows (the previous panel's block rows)
  const int mt = m + off;
  // panel -> shared memory, 8 loads in flight per thread (thread's column j = tid % QB is fixed)
  {
    const int j = tid % QB;
    for (int i0 = tid / QB; i0 < mt; i0 += 8 * (NT / QB)) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        v[u] = (i < mt && j < jb) ? Pg[(int64_t)i * ldg + j] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        if (i < mt) psm_all[i * LD + j] = v[u];
      }
    }
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  if (Vprev) {
    // W = V_prev^T C (QB x QB): warp q forms row q (lanes over rows, 16 column sums each)
    {
      const int q = warp;
      double acc[QB];
#pragma unroll
      for (int j = 0; j < QB; j++) acc[j] = 0.0;
      for (int i = lane; i < mt; i += 32) {
        const double v = __ldg(Vprev + (int64_t)i * QB + q);
#pragma unroll
        for (int j = 0; j < QB; j++) acc[j] = fma(v, psm_all[i * LD + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < QB; j++) {
        const double t = warp_sum(acc[j]);
        if (lane == 0) s_w[q][j] = t;
      }
    }
    __syncthreads();
    // C -= (V T^T) W
    {
      const int j = tid % QB;
      double w[QB];
#pragma unroll
      for (int q = 0; q < QB; q++) w[q] = s_w[q][j];
      for (int i = tid / QB; i < mt; i += NT / QB) {
        const double2* xr = reinterpret_cast<const double2*>(VTtprev + (int64_t)i * QB);
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < QB / 2; q++) {
          const double2 x = __ldg(xr + q);
          d = fma(x.x, w[2 * q], d);
          d = fma(x.y, w[2 * q + 1], d);
        }
        psm_all[i * LD + j] -= d;
      }
    }
    __syncthreads();
  }
  double* psm = psm_all + off * LD;  // this panel's m rows
  stamp(1);
  if (warp == 0 && jb > 0) make_reflector(psm, 0, m, lane, s_tau);
  __syncthreads();
  stamp(2);
  for (int c = 0; c < jb; c++) {
    const double tau = s_tau[c];
    if (warp > c && warp < jb) {
      const int j = warp;
      const bool fs = dbg && c == 4 && j == 5 && lane == 0;
      auto fst = [&](int k) {
        if (fs) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          dbg[k] = t;
        }
      };
      fst(5);
      // row c counted once (v_c = 1)
      double w = col_dot<LD>(psm, c, j, c + 1, m, lane) + (lane == 0 ? psm[c * LD + j] : 0.0);
      fst(6);
      w = warp_sum(w) * tau;
      fst(7);
      if (lane == 0) psm[c * LD + j] -= w;
#pragma unroll 4
      for (int i = c + 1 + lane; i < m; i += 32) psm[i * LD + j] = fma(-w, psm[i * LD + c], psm[i * LD + j]);
      __syncwarp();
      fst(8);
      if (j == c + 1) make_reflector(psm, j, m, lane, s_tau);
      fst(9);
    } else if (warp < c) {
      const int j = warp;
      // z_j = V[:, j]^T v_c over rows >= c (v_c is zero above c; V[c, j] is stored below diag j)
      double z = col_dot<LD>(psm, j, c, c + 1, m, lane) + (lane == 0 ? psm[c * LD + j] : 0.0);
      z = warp_sum(z);
      if (lane == 0) s_z[c][j] = z;
    }
    __syncthreads();
    if (dbg && c == 4 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[10] = t;
    }
  }
  // T (dlarft, forward, columnwise) off the column loop's critical path:
  //   T[0:c, c] = -tau_c T[0:c, 0:c] z_c,  T[c, c] = tau_c
  if (warp == 0) {
    for (int c = 0; c < jb; c++) {
      if (lane < c) {
        double t = 0.0;
        for (int q = lane; q < c; q++) t = fma(Ts[lane][q], s_z[c][q], t);
        Ts[lane][c] = -s_tau[c] * t;
      }
      if (lane == 0) Ts[c][c] = s_tau[c];
      __syncwarp();
    }
  }
  __syncthreads();
  stamp(3);
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
  __syncthreads();
  stamp(4);
}

// Register-resident panel factorisation (m + off <= 32 * MAXR): warp j holds column j of the
// panel in registers (lane l, slot k <-> row i = l + 32 k, rows counted from the first loaded
// row), so the column loop touches shared memory only to publish each reflector v_c (double
// buffered) — the shared-memory version above was bandwidth-bound on the 15 warps re-reading
// v_c and their own columns every column (measured ~2.5 us per column at m ~ 450).
// Same contract as qr_panel_warp_k (including the fused look-ahead application of H_prev).
template <int MAXR>
__global__ void __launch_bounds__(32 * QB)
    qr_panel_reg_k(int m, int jb, const double* __restrict__ Pg, int64_t ldg,
                   double* __restrict__ Vout, double* __restrict__ Tout,
                   double* __restrict__ VTout, double* __restrict__ VTtout,
                   const double* __restrict__ Vprev, const double* __restrict__ VTtprev,
                   unsigned long long* __restrict__ dbg, int panel, int* __restrict__ stop_at,
                   const double* __restrict__ sqprev, int nsq, const double* __restrict__ thr2) {
  // early stop (rank revealed): the trailing block beyond this panel, as measured two panels
  // ago (H_prev is orthogonal: its norm can only be smaller now), is at the noise level
  __shared__ int s_stop;
  if (threadIdx.x == 0) {
    int stop = *(volatile int*)stop_at <= panel;
    if (!stop && sqprev) {
      double t = 0.0;
      for (int i = 0; i < nsq; i++) t += sqprev[i];
      if (t <= thr2[0]) {
        atomicMin(stop_at, panel);
        stop = 1;
      }
    }
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) return;
  auto stamp = [&](int k) {
    if (dbg && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[k] = t;
    }
  };
  stamp(0);
  constexpr int LD = QB + 1;
  constexpr int MR = 32 * MAXR;
  constexpr int NT = 32 * QB;
  __shared__ double vbuf[2][MR];
  __shared__ double s_tau[QB], s_z[QB][QB];
  __shared__ double Ts[QB][QB + 1];
  __shared__ double s_w[2][QB][QB + 1];
  // dynamic shared memory: the loaded panel (mt x LD) — staging for the look-ahead update and
  // the register columns, reused at the end for the export of V (m x LD)
  extern __shared__ double psm[];
  const int tid = threadIdx.x, lane = tid & 31, j = tid >> 5;
  const int off = Vprev ? QB : 0;
  const int mt = m + off;
  // panel -> shared memory (coalesced rows), 8 loads in flight per thread
  {
    const int jj = tid % QB;
    for (int i0 = tid / QB; i0 < mt; i0 += 8 * (NT / QB)) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        v[u] = (i < mt && jj < jb) ? Pg[(int64_t)i * ldg + jj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int i = i0 + u * (NT / QB);
        if (i < mt) psm[i * LD + jj] = v[u];
      }
    }
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  if (Vprev) {
    // W = V_prev^T C (QB x QB): thread -> (q, jj, half); V_prev rows streamed from global
    // (each warp reads two q's of a row: near-broadcast), C from shared memory
    {
      // warp w sums the rows i = w, w + 16, ...; lane l owns q = l / 2 and the 8 columns
      // jj = 8 (l & 1) + u: one broadcast load of V_prev[i][q] and 8 shared-memory reads of
      // row i of C per row, the rows' loads independent (the former thread-per-(q, jj) loop was
      // a dependent chain of ~mt/4 L2 loads: most of the 15 us "load" phase at m = 896).
      // Per-warp partials, then a fixed-order reduction (deterministic).
      double* part = psm + (size_t)mt * LD;  // 16 x QB x QB partials (extra dynamic smem)
      const int q = lane >> 1, j0 = 8 * (lane & 1);
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; u++) acc[u] = 0.0;
#pragma unroll 4
      for (int i = j; i < mt; i += QB) {
        const double v = __ldg(Vprev + (int64_t)i * QB + q);
#pragma unroll
        for (int u = 0; u < 8; u++) acc[u] = fma(v, psm[i * LD + j0 + u], acc[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; u++) part[(j * QB + q) * QB + j0 + u] = acc[u];
      __syncthreads();
      if (tid < QB * QB) {
        const int qq = tid / QB, jj = tid % QB;
        double t = 0.0;
        for (int w = 0; w < QB; w++) t += part[(w * QB + qq) * QB + jj];
        s_w[0][qq][jj] = t;
        s_w[1][qq][jj] = 0.0;
      }
    }
    __syncthreads();
    // C -= (V_prev T_prev^T) W
    {
      const int jj = tid % QB;
      double w[QB];
#pragma unroll
      for (int q = 0; q < QB; q++) w[q] = s_w[0][q][jj] + s_w[1][q][jj];
      for (int i = tid / QB; i < mt; i += NT / QB) {
        const double2* xr = reinterpret_cast<const double2*>(VTtprev + (int64_t)i * QB);
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < QB / 2; q++) {
          const double2 x = __ldg(xr + q);
          d = fma(x.x, w[2 * q], d);
          d = fma(x.y, w[2 * q + 1], d);
        }
        psm[i * LD + jj] -= d;
      }
    }
    __syncthreads();
  }
  double c[MAXR];
#pragma unroll
  for (int k = 0; k < MAXR; k++) {
    const int i = lane + 32 * k;
    c[k] = (i < mt) ? psm[i * LD + j] : 0.0;
  }
  __syncthreads();  // psm is reused for the export below
  stamp(1);
  stamp(2);
  // reflector of column j from its rows i >= r0 = j + off (register column), v -> vbuf[buf]
  auto reflect = [&](int buf) {
    const int r0 = j + off;
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; k++) {
      const int i = lane + 32 * k;
      if (i > r0 && i < mt) sq = fma(c[k], c[k], sq);
    }
    sq = warp_sum(sq);
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; k++)
      if (lane + 32 * k == r0) a = c[k];
    const double alpha = __shfl_sync(0xffffffffu, a, r0 & 31);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sq > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sq));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
#pragma unroll
    for (int k = 0; k < MAXR; k++) {
      const int i = lane + 32 * k;
      double v = 0.0;
      if (i > r0 && i < mt) {
        c[k] *= scale;
        v = c[k];
      } else if (i == r0) {
        c[k] = 1.0;  // v_j(r0) = 1 (the R entry beta is not needed)
        v = 1.0;
      } else if (i < r0) {
        c[k] = 0.0;
      }
      if (i < MR) vbuf[buf][i] = v;
    }
    if (lane == 0) s_tau[j] = tau;
  };
  if (j == 0 && jb > 0) reflect(0);
  __syncthreads();
  for (int cc = 0; cc < jb; cc++) {
    const int buf = cc & 1;
    const double tau = s_tau[cc];
    const int r0 = cc + off;
    if (j > cc && j < jb) {
      const bool fs = dbg && cc == 4 && j == 5 && lane == 0;
      auto fst = [&](int k) {
        if (fs) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          dbg[k] = t;
        }
      };
      fst(5);
      // v_cc read once into registers (shared-memory bandwidth is the limit: every active
      // warp needs all of v_cc each column), two partial sums
      double vr[MAXR];
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int k = 0; k < MAXR; k++) {
        const int i = lane + 32 * k;
        vr[k] = (i >= r0 && i < mt) ? vbuf[buf][i] : 0.0;
        if (k & 1)
          w1 = fma(vr[k], c[k], w1);
        else
          w0 = fma(vr[k], c[k], w0);
      }
      fst(6);
      const double w = warp_sum(w0 + w1) * tau;
      fst(7);
#pragma unroll
      for (int k = 0; k < MAXR; k++) c[k] = fma(-w, vr[k], c[k]);
      fst(8);
      if (j == cc + 1) reflect(buf ^ 1);
      fst(9);
    } else if (j < cc) {
      // z_j = V[:, j]^T v_cc (register column j is v_j: zeros above its diagonal)
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int k = 0; k < MAXR; k++) {
        const int i = lane + 32 * k;
        const double v = (i >= r0 && i < mt) ? vbuf[buf][i] : 0.0;
        if (k & 1)
          z1 = fma(v, c[k], z1);
        else
          z0 = fma(v, c[k], z0);
      }
      const double z = warp_sum(z0 + z1);
      if (lane == 0) s_z[cc][j] = z;
    }
    __syncthreads();
  }
  // T (dlarft, forward, columnwise): T[0:c, c] = -tau_c T[0:c, 0:c] z_c, T[c, c] = tau_c
  if (j == 0) {
    for (int cc = 0; cc < jb; cc++) {
      if (lane < cc) {
        double t = 0.0;
        for (int q = lane; q < cc; q++) t = fma(Ts[lane][q], s_z[cc][q], t);
        Ts[lane][cc] = -s_tau[cc] * t;
      }
      if (lane == 0) Ts[cc][cc] = s_tau[cc];
      __syncwarp();
    }
  }
  stamp(3);
  // V (rows off .. mt-1 of the register columns; zero columns beyond jb) to shared memory
#pragma unroll
  for (int k = 0; k < MAXR; k++) {
    const int i = lane + 32 * k;
    if (i >= off && i < mt) psm[(i - off) * LD + j] = (j < jb) ? c[k] : 0.0;
  }
  __syncthreads();
  const int jj = tid % QB;
  double tc[QB], tr[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) {
    tc[q] = Ts[q][jj];
    tr[q] = Ts[jj][q];
  }
  for (int e = tid; e < m * QB; e += blockDim.x) {
    const int i = e / QB;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int q = 0; q < QB; q++) {
      const double v = psm[i * LD + q];
      a = fma(v, tc[q], a);
      b = fma(v, tr[q], b);
    }
    Vout[e] = psm[i * LD + jj];
    VTout[e] = a;
    VTtout[e] = b;
  }
  for (int e = tid; e < QB * QB; e += blockDim.x) Tout[e] = Ts[e / QB][e % QB];
  __syncthreads();
  stamp(4);
}

// Tall-panel variant of qr_panel_reg_k for m > 32 * MAXR (the pass-1 QR of the c5 / c6 Grams,
// k ~ 1300-2800): warp j holds rows [0, 32 MAXR) of column j in registers, rows [32 MAXR, BIG_M)
// in a per-column shared-memory overflow region and — only when m > BIG_M — the rows beyond in
// a global-memory tail (gtail: QB columns of mt = m - BIG_M rows, column-major, then two
// reflector tails of mt rows; L2-resident, a fraction of the panel), so the panel is factored by
// one CTA (the former fallback, qr_panel_k<false> working entirely in global memory, took
// ~460 us per 16-column panel at m = 2240).  Same contract as qr_panel_k<false>: the panel
// (m x jb, ld ldg, already updated by the previous reflectors) in, V (m x QB, unit lower
// trapezoidal, zero padded) and T (QB x QB) out; VT / VT^T are formed by the caller.  Dynamic
// smem: QB x (BIG_M - 32 MAXR) doubles.
constexpr int BIG_M = 2256;
constexpr int kBigTail = 4096;  // rows beyond BIG_M the tall kernel keeps in global memory
template <int MAXR>
__global__ void __launch_bounds__(32 * QB)
    qr_panel_big_k(int m, int jb, const double* __restrict__ Pg, int64_t ldg,
                   double* __restrict__ Vout, double* __restrict__ Tout,
                   double* __restrict__ gtail) {
  constexpr int MR = 32 * MAXR;
  constexpr int OVL = BIG_M - MR;  // overflow rows per column
  __shared__ double vbuf[2][BIG_M];
  __shared__ double s_tau[QB], s_z[QB][QB];
  __shared__ double Ts[QB][QB + 1];
  extern __shared__ double ov_all[];
  const int tid = threadIdx.x, lane = tid & 31, j = tid >> 5;
  const int ms = min(m, BIG_M);        // rows held on chip
  const int mt = m - ms;               // rows in the global tail (0 unless m > BIG_M)
  double* ov = ov_all + (size_t)j * OVL;  // rows MR.. of column j
  double* gc = gtail + (size_t)j * mt;    // rows BIG_M.. of column j
  double* gv0 = gtail + (size_t)QB * mt;  // reflector tails, two buffers
  double c[MAXR];
#pragma unroll
  for (int k = 0; k < MAXR; k++) {
    const int i = lane + 32 * k;
    c[k] = (i < m && j < jb) ? Pg[(int64_t)i * ldg + j] : 0.0;
  }
  for (int i = MR + lane; i < ms; i += 32) ov[i - MR] = j < jb ? Pg[(int64_t)i * ldg + j] : 0.0;
  for (int i = lane; i < mt; i += 32) gc[i] = j < jb ? Pg[(int64_t)(BIG_M + i) * ldg + j] : 0.0;
  for (int e = tid; e < QB * QB; e += blockDim.x) Ts[e / QB][e % QB] = 0.0;
  __syncthreads();
  auto reflect = [&](int buf) {
    const int r0 = j;
    double* gv = gv0 + (size_t)buf * mt;
    double sq = 0.0, sq2 = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; k++) {
      const int i = lane + 32 * k;
      if (i > r0 && i < m) sq = fma(c[k], c[k], sq);
    }
    for (int i = MR + lane; i < ms; i += 32) sq = fma(ov[i - MR], ov[i - MR], sq);
    for (int i = lane; i < mt; i += 32) sq2 = fma(gc[i], gc[i], sq2);
    sq = warp_sum(sq + sq2);
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < MAXR; k++)
      if (lane + 32 * k == r0) a = c[k];
    const double alpha = __shfl_sync(0xffffffffu, a, r0 & 31);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sq > 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sq));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
#pragma unroll
    for (int k = 0; k < MAXR; k++) {
      const int i = lane + 32 * k;
      double v = 0.0;
      if (i > r0 && i < m) {
        c[k] *= scale;
        v = c[k];
      } else if (i == r0) {
        c[k] = 1.0;
        v = 1.0;
      } else if (i < r0) {
        c[k] = 0.0;
      }
      vbuf[buf][i] = v;
    }
    for (int i = MR + lane; i < ms; i += 32) {
      ov[i - MR] *= scale;
      vbuf[buf][i] = ov[i - MR];
    }
    for (int i = lane; i < mt; i += 32) {
      const double v = gc[i] * scale;
      gc[i] = v;
      gv[i] = v;
    }
    if (lane == 0) s_tau[j] = tau;
  };
  if (j == 0 && jb > 0) reflect(0);
  __syncthreads();
  for (int cc = 0; cc < jb; cc++) {
    const int buf = cc & 1;
    const double tau = s_tau[cc];
    const int r0 = cc;
    const double* gv = gv0 + (size_t)buf * mt;
    if (j > cc && j < jb) {
      double vr[MAXR];
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int k = 0; k < MAXR; k++) {
        const int i = lane + 32 * k;
        vr[k] = (i >= r0 && i < m) ? vbuf[buf][i] : 0.0;
        if (k & 1)
          w1 = fma(vr[k], c[k], w1);
        else
          w0 = fma(vr[k], c[k], w0);
      }
      for (int i = MR + lane; i < ms; i += 32) w0 = fma(vbuf[buf][i], ov[i - MR], w0);
      for (int i = lane; i < mt; i += 32) w1 = fma(gv[i], gc[i], w1);
      const double w = warp_sum(w0 + w1) * tau;
#pragma unroll
      for (int k = 0; k < MAXR; k++) c[k] = fma(-w, vr[k], c[k]);
      for (int i = MR + lane; i < ms; i += 32) ov[i - MR] = fma(-w, vbuf[buf][i], ov[i - MR]);
      for (int i = lane; i < mt; i += 32) gc[i] = fma(-w, gv[i], gc[i]);
      if (j == cc + 1) reflect(buf ^ 1);
    } else if (j < cc) {
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int k = 0; k < MAXR; k++) {
        const int i = lane + 32 * k;
        const double v = (i >= r0 && i < m) ? vbuf[buf][i] : 0.0;
        if (k & 1)
          z1 = fma(v, c[k], z1);
        else
          z0 = fma(v, c[k], z0);
      }
      for (int i = MR + lane; i < ms; i += 32) z0 = fma(vbuf[buf][i], ov[i - MR], z0);
      for (int i = lane; i < mt; i += 32) z1 = fma(gv[i], gc[i], z1);
      const double z = warp_sum(z0 + z1);
      if (lane == 0) s_z[cc][j] = z;
    }
    __syncthreads();
  }
  if (j == 0) {
    for (int cc = 0; cc < jb; cc++) {
      if (lane < cc) {
        double t = 0.0;
        for (int q = lane; q < cc; q++) t = fma(Ts[lane][q], s_z[cc][q], t);
        Ts[lane][cc] = -s_tau[cc] * t;
      }
      if (lane == 0) Ts[cc][cc] = s_tau[cc];
      __syncwarp();
    }
  }
  __syncthreads();
  // V out (warp j writes column j; zero columns beyond jb)
#pragma unroll
  for (int k = 0; k < MAXR; k++) {
    const int i = lane + 32 * k;
    if (i < m) Vout[(int64_t)i * QB + j] = (j < jb) ? c[k] : 0.0;
  }
  for (int i = MR + lane; i < ms; i += 32) Vout[(int64_t)i * QB + j] = (j < jb) ? ov[i - MR] : 0.0;
  for (int i = lane; i < mt; i += 32) Vout[(int64_t)(BIG_M + i) * QB + j] = (j < jb) ? gc[i] : 0.0;
  for (int e = tid; e < QB * QB; e += blockDim.x) Tout[e] = Ts[e / QB][e % QB];
}

// C <- C - X (V^T C) for the m x nc block C (leading dimension ldc) and the m x QB panels V, X
// (row-major, ld QB): the compact-WY application of one panel's block reflector (X = V T^T for
// the trailing update, X = V T for the accumulation of Q), fused into one kernel.  CTA = a strip
// of AR_W columns; phase 1 forms W = V^T C[:, strip] (QB x AR_W) with the rows split over the 8
// warps and reduced in shared memory, phase 2 updates the strip row by row.  Rows of V and X
// are warp-uniform (broadcast loads), C accesses are coalesced along the strip.
constexpr int AR_W = 4, AR_T = 256, AR_G = AR_T / AR_W, AR_U = 4;
// Optional early-stop bookkeeping (trailing updates of pass 1): the kernel is skipped when
// panel >= *stop_at, and writes to sqpart[blockIdx.x] the sum of squares of its updated values in
// rows >= rowskip (deterministic per-CTA partial; the panel two steps later sums them).
__global__ void __launch_bounds__(AR_T) apply_reflector_k(int m, int nc, const double* __restrict__ V,
                                                          const double* __restrict__ X,
                                                          double* __restrict__ C, int64_t ldc,
                                                          int panel = 0,
                                                          const int* __restrict__ stop_at = nullptr,
                                                          double* __restrict__ sqpart = nullptr,
                                                          int rowskip = 0) {
  if (stop_at && panel >= *(volatile const int*)stop_at) return;
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
  double sq = 0.0;
  for (int i0 = rg; live && i0 < m; i0 += AR_G * AR_U) {
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
    // all AR_U reads of C before the stores (the compiler cannot prove the rows distinct —
    // ldc is a runtime value — so a load after a store waited for it: one L2 round trip per row)
    double cv[AR_U];
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = i0 + u * AR_G;
      cv[u] = i < m ? C[(int64_t)i * ldc + gc] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < AR_U; u++) {
      const int i = i0 + u * AR_G;
      if (i < m) {
        const double v = cv[u] - d[u];
        C[(int64_t)i * ldc + gc] = v;
        if (i >= rowskip) sq = fma(v, v, sq);
      }
    }
  }
  if (sqpart) {
    __syncthreads();  // red is reused for the partial sums
    double* r = &red[0][0][0];
    r[threadIdx.x] = sq;
    __syncthreads();
    for (int st = AR_T / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) r[threadIdx.x] += r[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) sqpart[blockIdx.x] = r[0];
  }
}

// C <- C H = C - (C V) (V T^T)^T for the n x m block C (leading dimension ldc): the forward
// accumulation Q <- Q H_p of the orthogonal factor.  Rows are independent: one warp per row,
// lanes over the columns; w = C[i, :] V (16 sums, warp-reduced), then C[i, c] -= w . VTt[c, :].
__global__ void __launch_bounds__(256) apply_reflector_right_k(int n, int m,
                                                               const double* __restrict__ V,
                                                               const double* __restrict__ VTt,
                                                               double* __restrict__ C,
                                                               int64_t ldc, int panel,
                                                               const int* __restrict__ stop_at) {
  if (panel >= *(volatile const int*)stop_at) return;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= n) return;
  double* row = C + (int64_t)i * ldc;
  double w[QB];
#pragma unroll
  for (int q = 0; q < QB; q++) w[q] = 0.0;
  for (int c = lane; c < m; c += 32) {
    const double x = row[c];
    const double2* vr = reinterpret_cast<const double2*>(V + (int64_t)c * QB);
#pragma unroll
    for (int q = 0; q < QB / 2; q++) {
      const double2 v = __ldg(vr + q);
      w[2 * q] = fma(x, v.x, w[2 * q]);
      w[2 * q + 1] = fma(x, v.y, w[2 * q + 1]);
    }
  }
#pragma unroll
  for (int q = 0; q < QB; q++) w[q] = warp_sum(w[q]);
  for (int c = lane; c < m; c += 32) {
    const double2* yr = reinterpret_cast<const double2*>(VTt + (int64_t)c * QB);
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < QB / 2; q++) {
      const double2 y = __ldg(yr + q);
      d = fma(w[2 * q], y.x, d);
      d = fma(w[2 * q + 1], y.y, d);
    }
    row[c] -= d;
  }
}

// thr2[0] = (64 eps ||A||_F)^2 and stop_at[0] = INT_MAX, in two small launches: per-CTA partial
// sums of squares (fixed-order tree), then their sum in CTA order — deterministic, and ~5 us
// instead of the ~70 us a single CTA needed for n = 896 (a chain of ~200 L2 round trips per
// thread at the start of every pass-1 QR).
constexpr int SQ_T = 256, SQ_MAXG = 148;
__global__ void __launch_bounds__(SQ_T) qr_sq_partial_k(int64_t nn, const double* __restrict__ A,
                                                        double* __restrict__ part) {
  __shared__ double red[SQ_T];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * SQ_T;
  int64_t e = (int64_t)blockIdx.x * SQ_T + threadIdx.x;
  for (; e + 3 * stride < nn; e += 4 * stride) {
    const double a0 = A[e], a1 = A[e + stride], a2 = A[e + 2 * stride], a3 = A[e + 3 * stride];
    s0 = fma(a0, a0, s0);
    s1 = fma(a1, a1, s1);
    s2 = fma(a2, a2, s2);
    s3 = fma(a3, a3, s3);
  }
  for (; e < nn; e += stride) s0 = fma(A[e], A[e], s0);
  red[threadIdx.x] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  for (int st = SQ_T / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void qr_stop_fin_k(int g, const double* __restrict__ part, double* __restrict__ thr2,
                              int* __restrict__ stop_at) {
  double t = 0.0;
  for (int i = 0; i < g; i++) t += part[i];
  const double e64 = 64.0 * 2.220446049250313e-16;
  thr2[0] = e64 * e64 * t;
  stop_at[0] = 0x7fffffff;
}

}  // namespace

// Q (n x n, row-major) from the Householder QR of A (n x n, row-major; A is not modified).
int tk_householder_q(tk_ctx* ctx, int n, const double* A, double* Q) {
  if (n <= 0) return TK_OK;
  DevBuf Aw, Vb, Tb, VTb, VTtb;
  TK_TRY(Aw.get(ctx, (size_t)n * n));
  TK_TRY(tk_copy2d(ctx, 1, (int64_t)n * n, A, (int64_t)n * n, Aw.p, (int64_t)n * n));
  const int np = (n + QB - 1) / QB;
  // panel p: V, V T, V T^T as (n - j0) x QB at offset p*n*QB;  T: QB x QB
  TK_TRY(Vb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTb.get(ctx, (size_t)np * n * QB));
  TK_TRY(VTtb.get(ctx, (size_t)np * n * QB));
  TK_TRY(Tb.get(ctx, (size_t)np * QB * QB));
  TK_TRY(tk_eye(ctx, Q, n));
  // early stop once the trailing block is at the rounding-noise level (numerical rank reached):
  // the remaining reflectors would act on noise and the identity completion is as good a pass-1
  // basis; sqpart[p]: per-CTA squared norms written by the trailing update of panel p
  const int sq_stride = (n + AR_W - 1) / AR_W + 1;
  DevBuf qst, sqpart;
  TK_TRY(qst.get(ctx, 2 + SQ_MAXG));
  TK_TRY(sqpart.get(ctx, (size_t)np * sq_stride));
  double* thr2 = qst.p;
  int* stop_at = (int*)(qst.p + 1);
  const bool no_stop = false;
  {
    const int64_t nn = (int64_t)n * n;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>(SQ_MAXG, nn / (8 * SQ_T)));
    qr_sq_partial_k<<<g, SQ_T, 0, ctx->stream>>>(nn, A, qst.p + 2);
    TK_LAUNCH_CHECK(ctx);
    qr_stop_fin_k<<<1, 1, 0, ctx->stream>>>(g, qst.p + 2, thr2, stop_at);
    TK_LAUNCH_CHECK(ctx);
  }
  DevBuf dbgb;  // (per-panel clock stamps of the panel kernels: not allocated = off)
  // global tail of the tall panel kernel (rows beyond BIG_M: QB columns + two reflector tails)
  DevBuf gtail;
  if (n > BIG_M && n <= BIG_M + kBigTail)
    TK_TRY(gtail.get(ctx, (size_t)(QB + 2) * (n - BIG_M)));
  // Streams: s0 (ctx->stream) carries the critical path  F_0, U_0', F_1, U_1', ...  where F_p
  // factors panel p and U_p' applies H_p to panel p+1 only; s1 applies H_p to the columns
  // beyond panel p+1 (overlapping F_{p+1}); s2 accumulates Q <- Q H_p forward (overlapping
  // everything).  evF[p]: V_p ready; evR[p]: H_p applied beyond panel p+1.
  TK_TRY(tk_aux_streams(ctx, 2 * (size_t)np + 2));
  cudaStream_t s0 = ctx->stream, s1 = ctx->aux[0], s2 = ctx->aux[1];
  cudaEvent_t* evF = ctx->fork_ev.data();
  cudaEvent_t* evR = evF + np;
  cudaEvent_t evStart = evF[2 * np], evEnd = evF[2 * np + 1];
  TK_CUDA_TRY(ctx, cudaEventRecord(evStart, s0));
  TK_CUDA_TRY(ctx, cudaStreamWaitEvent(s1, evStart, 0));
  TK_CUDA_TRY(ctx, cudaStreamWaitEvent(s2, evStart, 0));
  // join on EVERY exit (also the error returns inside the panel loop): everything on s1 / s2
  // before s0 continues, and before the scratch buffers above are freed on s0 (declared after
  // them, so destroyed first)
  struct AuxJoin {
    cudaStream_t s0, s1, s2;
    cudaEvent_t ev;
    ~AuxJoin() {
      cudaEventRecord(ev, s1);
      cudaStreamWaitEvent(s0, ev, 0);
      cudaEventRecord(ev, s2);
      cudaStreamWaitEvent(s0, ev, 0);
    }
  } join{s0, s1, s2, evEnd};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qr_panel_warp_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  // factor(p): panel p; with look-ahead (p > 0) the kernel first applies H_{p-1} itself
  auto factor = [&](int p) -> int {
    const int j0 = p * QB, jb = std::min(QB, n - j0), m = n - j0;
    double* Vp = Vb.p + (size_t)p * n * QB;
    double* VTp = VTb.p + (size_t)p * n * QB;
    double* VTtp = VTtb.p + (size_t)p * n * QB;
    double* Tp = Tb.p + (size_t)p * QB * QB;
    const int pid = tk_prof_begin(ctx, "qr_panel", 2.0 * m * (double)jb * jb, 0.0);
    const int off = p > 0 ? QB : 0;
    const int mt = m + off;
    const double* Vq0 = p > 0 ? Vb.p + (size_t)(p - 1) * n * QB : nullptr;
    const double* VTtq0 = p > 0 ? VTtb.p + (size_t)(p - 1) * n * QB : nullptr;
    if (mt <= 32 * 28) {
      // register-resident columns
      // the loaded panel (mt x (QB+1)) + the look-ahead's per-warp partials (16 x QB x QB)
      const size_t rsmem = sizeof(double) * ((size_t)mt * (QB + 1) + (size_t)QB * QB * QB);
      const double* Pp = Aw.p + (int64_t)(j0 - off) * n + j0;
      // the trailing update of panel p-2 measured the block this panel would work on
      const double* sqp = nullptr;
      int nsq = 0;
      if (!no_stop && p >= 2) {
        const int c2q = (p - 2) * QB + 2 * QB;
        if (n - c2q > 0) {
          sqp = sqpart.p + (size_t)(p - 2) * sq_stride;
          nsq = (n - c2q + AR_W - 1) / AR_W;
        }
      }
#define TK_QR_REG(MR)                                                                        \
  {                                                                                          \
    static bool at = false;                                                                  \
    if (!at) {                                                                               \
      cudaFuncSetAttribute(qr_panel_reg_k<MR>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                           200 * 1024);                                                      \
      at = true;                                                                             \
    }                                                                                        \
    qr_panel_reg_k<MR><<<1, 32 * QB, rsmem, s0>>>(m, jb, Pp, n, Vp, Tp, VTp, VTtp, Vq0, VTtq0, \
        dbgb.p ? (unsigned long long*)dbgb.p + 12 * p : nullptr, p, stop_at,                   \
        sqp, nsq, thr2);                                                                       \
  }
      if (mt <= 32 * 8)
        TK_QR_REG(8)
      else if (mt <= 32 * 16)
        TK_QR_REG(16)
      else
        TK_QR_REG(28)
#undef TK_QR_REG
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      TK_CUDA_TRY(ctx, cudaEventRecord(evF[p], s0));
      return TK_OK;
    }
    const size_t psmem = (size_t)(m + off) * (QB + 1) * sizeof(double);
    if (psmem <= 200 * 1024 && m > BIG_M) {  // (never: the big kernel serves 896 < m <= BIG_M)
      const double* Vq = p > 0 ? Vb.p + (size_t)(p - 1) * n * QB : nullptr;
      const double* VTtq = p > 0 ? VTtb.p + (size_t)(p - 1) * n * QB : nullptr;
      qr_panel_warp_k<<<1, 32 * QB, psmem, s0>>>(
          m, jb, Aw.p + (int64_t)(j0 - off) * n + j0, n, Vp, Tp, VTp, VTtp, Vq, VTtq,
          dbgb.p ? (unsigned long long*)dbgb.p + 12 * p : nullptr);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
    } else {
      if (p > 0) {
        // no room for the fused look-ahead: apply H_{p-1} to this panel first
        const int mp = m + QB;
        apply_reflector_k<<<(jb + AR_W - 1) / AR_W, AR_T, 0, s0>>>(
            mp, jb, Vb.p + (size_t)(p - 1) * n * QB, VTtb.p + (size_t)(p - 1) * n * QB,
            Aw.p + (int64_t)(j0 - QB) * n + j0, n);
        TK_LAUNCH_CHECK(ctx);
      }
      if (m <= BIG_M + kBigTail) {
        constexpr int BMR = 26;  // 832 register rows; the rest in shared memory (and, beyond
                                 // BIG_M rows, in the global tail gtail)
        const size_t osmem = sizeof(double) * (size_t)QB * (BIG_M - 32 * BMR);
        static bool at = false;
        if (!at) {
          cudaFuncSetAttribute(qr_panel_big_k<BMR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)osmem);
          at = true;
        }
        qr_panel_big_k<BMR><<<1, 32 * QB, osmem, s0>>>(m, jb, Aw.p + (int64_t)j0 * n + j0, n, Vp,
                                                      Tp, gtail.p);
      } else {
        qr_panel_k<false><<<1, QT, 0, s0>>>(m, jb, Aw.p + (int64_t)j0 * n + j0, n, Vp, Tp);
      }
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      TK_TRY(tk_dgemm(ctx, false, false, m, QB, QB, 1.0, Vp, QB, Tp, QB, 0.0, VTp, QB));
      TK_TRY(tk_dgemm(ctx, false, true, m, QB, QB, 1.0, Vp, QB, Tp, QB, 0.0, VTtp, QB));
    }
    TK_CUDA_TRY(ctx, cudaEventRecord(evF[p], s0));
    return TK_OK;
  };
  TK_TRY(factor(0));
  for (int p = 0; p < np; p++) {
    const int j0 = p * QB, jb = std::min(QB, n - j0), m = n - j0;
    const double* Vp = Vb.p + (size_t)p * n * QB;
    const double* VTtp = VTtb.p + (size_t)p * n * QB;
    const int c1 = j0 + jb;                     // first column of panel p+1
    const int nnext = std::min(QB, n - c1);     // its width (<= 0 at the last panel)
    const int c2 = c1 + std::max(nnext, 0);     // first column beyond panel p+1
    // s1: H_p on the columns beyond panel p+1
    TK_CUDA_TRY(ctx, cudaStreamWaitEvent(s1, evF[p], 0));
    if (n - c2 > 0) {
      apply_reflector_k<<<(n - c2 + AR_W - 1) / AR_W, AR_T, 0, s1>>>(
          m, n - c2, Vp, VTtp, Aw.p + (int64_t)j0 * n + c2, n, p, stop_at,
          sqpart.p + (size_t)p * sq_stride, jb);
      TK_LAUNCH_CHECK(ctx);
    }
    TK_CUDA_TRY(ctx, cudaEventRecord(evR[p], s1));
    // s2: Q <- Q H_p (all n rows, columns j0..n)
    TK_CUDA_TRY(ctx, cudaStreamWaitEvent(s2, evF[p], 0));
    apply_reflector_right_k<<<(n + 7) / 8, 256, 0, s2>>>(n, m, Vp, VTtp, Q + j0, n, p, stop_at);
    TK_LAUNCH_CHECK(ctx);
    // s0: panel p+1 (its columns got H_{p-1} from s1; it applies H_p itself), then factor it
    if (nnext > 0) {
      if (p > 0) TK_CUDA_TRY(ctx, cudaStreamWaitEvent(s0, evR[p - 1], 0));
      TK_TRY(factor(p + 1));
    }
    // Every kQrPoll panels the host reads the early-stop flag (one s0 synchronisation): once
    // the numerical rank is reached the remaining panels and reflector updates would only
    // return early, but each still costs its launch and event latencies (c4: ~40 of the 56
    // panels of the rank-128 time-core Gram).
    if (!no_stop && (p + 1) % kQrPoll == 0 && p + 2 < np) {
      int st = 0;
      TK_TRY(tk_read_host(ctx, s0, &st, stop_at, sizeof(int)));
      if (st <= p + 1) break;
    }
  }
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_qr_k() {}
const void* tk_anchor_k_qr() { return (const void*)tk_anchor_k_qr_k; }
