// Pivoted Cholesky (diagonal pivoting, LAPACK dpstrf semantics) of a symmetric positive
// semi-definite fp64 matrix, and the small triangular helpers of the CholeskyQR2 basis used by
// orth_rows:
//
//   H = P R^T R P^T      R: k x n upper trapezoidal in pivot order, k = numerical rank
//
// R is returned in ORIGINAL column indexing, Ro[t, piv[c]] = R[t, c], so that the trailing
// update never moves data: Ro P = R, and H ~ Ro^T Ro.  The factorisation stops when the largest
// remaining Schur-complement diagonal is <= tol.
//
// Blocked right-looking: a panel of nb pivot steps runs in ONE CTA (the Schur diagonal and the
// panel's rows of Ro live in shared memory); a step is an argmax and one row
//     Ro[j, c] = (Hw[p, c] - sum_{t in panel, t < j} Ro[t, p] Ro[t, c]) / sqrt(d_p)
// ), then the whole working matrix takes the panel's rank-NB update Hw -= Ro_panel^T Ro_panel
// on the DMMA GEMM (symmetric mode).  Rows of the pivots already taken receive meaningless
// updates but are never read again (their d is retired).
#include <cuda_runtime.h>
#include <stdint.h>

#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "ttk_internal.h"

namespace {

constexpr int PT = 512;  // threads of the panel kernel

// Block-wide argmax of (v, idx) pairs (ties -> smaller index); result in (s_p, s_dmax) for all.
__device__ __forceinline__ void block_argmax(double bv, int bi, double* s_val, int* s_idx,
                                             int* s_p, double* s_dmax) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_val[warp] = bv;
    s_idx[warp] = bi;
  }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    bv = lane < nw ? s_val[lane] : -INFINITY;
    bi = lane < nw ? s_idx[lane] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      *s_p = bi;
      *s_dmax = bv;
    }
  }
  __syncthreads();
}

// Block-wide argmax with ONE barrier: every warp reduces the per-warp candidates itself, so the
// result lands in registers of all threads (no second barrier / shared broadcast).  The
// per-warp candidate arrays are double-buffered by call parity: a warp may still be reading
// buffer `par` of this call while faster warps write buffer `par ^ 1` of the next one.
template <int NW>
__device__ __forceinline__ void block_argmax_reg(double bv, int bi, double (*s_val)[NW],
                                                 int (*s_idx)[NW], int par, int& p_out,
                                                 double& dmax_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s_val[par][warp] = bv;
    s_idx[par][warp] = bi;
  }
  __syncthreads();
  bv = lane < NW ? s_val[par][lane] : -INFINITY;
  bi = lane < NW ? s_idx[par][lane] : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  p_out = bi;
  dmax_out = bv;
}

// Panel of nb pivot steps (one CTA).  Shared memory: the panel's rows of Ro for every column
// (sR[t * n + c], t < nb) and the live Schur diagonal sd[c] (-inf once retired).  A step: row
// j of Ro for the pivot p, the Schur diagonal update, and — fused into the same pass over the
// columns — each thread's candidate for the NEXT pivot, reduced block-wide (two barriers per
// step; without pivoting the next index is simply j + 1).
__global__ void __launch_bounds__(PT) pchol_panel_k(int n, int j0, int nb, int pivot,
                                                    const double* __restrict__ Hw,
                                                    double* __restrict__ Ro, int* __restrict__ piv,
                                                    int* __restrict__ state,
                                                    const double* __restrict__ tol_dev,
                                                    double* __restrict__ rem_out) {
  // state[0]: rank so far / final (k); state[1]: 1 once stopped; state[2 + c]: retired flags
  extern __shared__ double psm[];
  double* sR = psm;                    // nb x n
  double* sd = psm + (int64_t)nb * n;  // n
  __shared__ double s_val[PT / 32];
  __shared__ int s_idx[PT / 32];
  __shared__ int s_p;
  __shared__ double s_dmax;
  if (state[1]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double tol = tol_dev[0];
  int* retired = state + 2;
  // retired columns carry d = -inf, so they never win the argmax
  double bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int c = tid; c < n; c += blockDim.x) {
    const double v = retired[c] ? -INFINITY : Hw[(int64_t)c * n + c];
    sd[c] = v;
    if (v > bv) {  // ascending c per thread: strict > keeps the smaller index on ties
      bv = v;
      bi = c;
    }
  }
  if (pivot) {
    block_argmax(bv, bi, s_val, s_idx, &s_p, &s_dmax);
  } else {
    __syncthreads();
    if (tid == 0) {
      s_p = j0;
      s_dmax = j0 < n ? sd[j0] : -INFINITY;
    }
    __syncthreads();
  }
  for (int s = 0; s < nb; s++) {
    const int j = j0 + s;
    if (j >= n) break;
    const int p = s_p;
    const double dmax = s_dmax;
    if (!(dmax > tol) || p >= n) {  // uniform: rank reached (or nothing left / non-finite)
      if (tid == 0) {
        state[0] = j;
        state[1] = 1;
      }
      if (rem_out) {
        // trace of the dropped Schur complement (its eigenvalues' sum: part of the tail)
        double t = 0.0;
        for (int c = tid; c < n; c += blockDim.x)
          if (sd[c] != -INFINITY) t += fmax(sd[c], 0.0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        __syncthreads();
        if (lane == 0) s_val[warp] = t;
        __syncthreads();
        if (tid == 0) {
          double tt = 0.0;
          for (int w = 0; w < (int)(blockDim.x >> 5); w++) tt += s_val[w];
          rem_out[0] = tt;
        }
      }
      return;
    }
    const double rinv = rsqrt(dmax), r = dmax * rinv;  // one special function per step
    // row j of Ro:  Ro[j, c] = (Hw[p, c] - sum_{t < s} sR[t, p] sR[t, c]) / r, then the next
    // pivot candidate among the updated live columns
    const double* hrow = Hw + (int64_t)p * n;
    double* orow = Ro + (int64_t)j * n;
    bv = -INFINITY;
    bi = 0x7fffffff;
    for (int c = tid; c < n; c += blockDim.x) {
      double out;
      if (c == p) {
        out = r;
        sd[c] = -INFINITY;
        retired[c] = 1;
      } else if (sd[c] == -INFINITY) {
        out = 0.0;
      } else {
        // four independent partial sums (the shared-memory latency bounds a single chain)
        double v0 = hrow[c], v1 = 0.0, v2 = 0.0, v3 = 0.0;
        int t = 0;
        for (; t + 3 < s; t += 4) {
          v0 = fma(-sR[t * n + p], sR[t * n + c], v0);
          v1 = fma(-sR[(t + 1) * n + p], sR[(t + 1) * n + c], v1);
          v2 = fma(-sR[(t + 2) * n + p], sR[(t + 2) * n + c], v2);
          v3 = fma(-sR[(t + 3) * n + p], sR[(t + 3) * n + c], v3);
        }
        for (; t < s; t++) v0 = fma(-sR[t * n + p], sR[t * n + c], v0);
        out = ((v0 + v1) + (v2 + v3)) * rinv;
        const double nd = fma(-out, out, sd[c]);
        sd[c] = nd;
        if (nd > bv) {
          bv = nd;
          bi = c;
        }
      }
      orow[c] = out;
      sR[s * n + c] = out;
    }
    if (tid == 0) {
      piv[j] = p;
      state[0] = j + 1;
    }
    if (pivot) {
      block_argmax(bv, bi, s_val, s_idx, &s_p, &s_dmax);  // also orders this step's writes
    } else {
      __syncthreads();
      if (tid == 0) {
        s_p = j + 1;
        s_dmax = j + 1 < n ? sd[j + 1] : -INFINITY;
      }
      __syncthreads();
    }
  }
}

// Register variant for n <= PT: each thread keeps its own column's panel values in
// registers (Rp), so a step reads only the pivot column's values from shared memory (broadcast)
// — the shared-memory variant above streams both operands of every row dot product through
// shared memory.  The step loop is unrolled (NB compile-time) so Rp is statically indexed.
template <int MAXC, int NB, int NTH = PT>
__global__ void __launch_bounds__(NTH) pchol_panel_reg_k(int n, int j0, int pivot,
                                                        const double* __restrict__ Hw,
                                                        double* __restrict__ Ro,
                                                        int* __restrict__ piv,
                                                        int* __restrict__ state,
                                                        const double* __restrict__ tol_dev,
                                                        double* __restrict__ rem_out) {
  extern __shared__ double sR[];  // NB x n
  __shared__ double s_val[2][NTH / 32];
  __shared__ int s_idx[2][NTH / 32];
  __shared__ int s_p;
  __shared__ double s_dmax;
  int par = 0;           // parity of the argmax buffers
  int cur_p = 0;         // pivot of the next step (registers, every thread)
  double cur_dmax = 0.0;
  if (state[1]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double tol = tol_dev[0];
  int* retired = state + 2;
  double d[MAXC], Rp[MAXC][NB];
  bool live[MAXC];
  double bv = -INFINITY;
  int bi = 0x7fffffff;
#pragma unroll
  for (int m = 0; m < MAXC; m++) {
    const int c = tid + m * NTH;
    live[m] = c < n && !retired[c];
    d[m] = live[m] ? Hw[(int64_t)c * n + c] : -INFINITY;
    if (d[m] > bv) {
      bv = d[m];
      bi = c;
    }
#pragma unroll
    for (int t = 0; t < NB; t++) Rp[m][t] = 0.0;
  }
  if (pivot) {
    block_argmax_reg<NTH / 32>(bv, bi, s_val, s_idx, par, cur_p, cur_dmax);
    par ^= 1;
  } else {
#pragma unroll
    for (int m = 0; m < MAXC; m++)
      if (tid + m * NTH == j0) {
        s_p = j0;
        s_dmax = d[m];
      }
    __syncthreads();
    cur_p = s_p;
    cur_dmax = s_dmax;
  }
#pragma unroll
  for (int s = 0; s < NB; s++) {
    const int j = j0 + s;
    if (j >= n) break;
    const int p = cur_p;
    const double dmax = cur_dmax;
    if (!(dmax > tol) || p >= n) {  // uniform: rank reached (or nothing left / non-finite)
      if (tid == 0) {
        state[0] = j;
        state[1] = 1;
      }
      if (rem_out) {
        double t = 0.0;
#pragma unroll
        for (int m = 0; m < MAXC; m++)
          if (live[m]) t += fmax(d[m], 0.0);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        __syncthreads();
        if (lane == 0) s_val[par][warp] = t;
        __syncthreads();
        if (tid == 0) {
          double tt = 0.0;
          for (int w = 0; w < (int)(blockDim.x >> 5); w++) tt += s_val[par][w];
          rem_out[0] = tt;
        }
      }
      return;
    }
    const double rinv = rsqrt(dmax), r = dmax * rinv;  // one special function per step
    double pc[NB];
#pragma unroll
    for (int t = 0; t < NB; t++) pc[t] = t < s ? sR[t * n + p] : 0.0;
    const double* hrow = Hw + (int64_t)p * n;
    double* orow = Ro + (int64_t)j * n;
    bv = -INFINITY;
    bi = 0x7fffffff;
#pragma unroll
    for (int m = 0; m < MAXC; m++) {
      const int c = tid + m * NTH;
      if (c >= n) continue;
      double out = 0.0;
      if (c == p) {
        out = r;
        live[m] = false;
        d[m] = -INFINITY;
        retired[c] = 1;
      } else if (live[m]) {
        double v0 = hrow[c], v1 = 0.0;
#pragma unroll
        for (int t = 0; t < NB; t++) {
          if (t < s) {
            if (t & 1)
              v1 = fma(-pc[t], Rp[m][t], v1);
            else
              v0 = fma(-pc[t], Rp[m][t], v0);
          }
        }
        out = (v0 + v1) * rinv;
        d[m] = fma(-out, out, d[m]);
        if (d[m] > bv) {
          bv = d[m];
          bi = c;
        }
      }
      Rp[m][s] = out;
      orow[c] = out;
      sR[s * n + c] = out;
    }
    if (tid == 0) {
      piv[j] = p;
      state[0] = j + 1;
    }
    if (pivot) {
      block_argmax_reg<NTH / 32>(bv, bi, s_val, s_idx, par, cur_p, cur_dmax);  // (its barrier
      par ^= 1;                                     // also orders this step's writes)
    } else {
      __syncthreads();
#pragma unroll
      for (int m = 0; m < MAXC; m++)
        if (tid + m * NTH == j + 1) {
          s_p = j + 1;
          s_dmax = d[m];
        }
      if (j + 1 >= n && tid == 0) {
        s_p = n;
        s_dmax = -INFINITY;
      }
      __syncthreads();
      cur_p = s_p;
      cur_dmax = s_dmax;
    }
  }
}

__global__ void max_diag_tol_k(int n, const double* __restrict__ H, double rel,
                               const double* __restrict__ abs_dev, double* __restrict__ tol) {
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, H[(int64_t)i * n + i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double t = rel * red[0];
    if (abs_dev) t = fmax(t, abs_dev[0]);
    // strictly positive: a zero pivot never enters
    tol[0] = fmax(t, 1e-300);
  }
}

// Unpivoted blocked Cholesky, one 32-column panel per launch (the CholeskyQR passes: pivot ==
// false).  Every CTA factors the 32 x 32 diagonal block in warp 0 (lane c holds column c in
// registers; a step is one broadcast row through shared memory, no block-wide barriers),
// then each thread solves R11^T x = Hw[panel rows, c] for its own column c beyond the block
// (forward substitution against R11 in shared memory).  The trailing update is the DMMA GEMM.
// Stops (state[1] = 1, state[0] = rank) at the first column whose Schur diagonal is <= tol,
// the semantics of the pivoted kernels with pivot == false.
constexpr int UCT = 128;
__global__ void __launch_bounds__(UCT) chol_unpiv_panel_k(int n, int j0, const double* __restrict__ Hw,
                                                          double* __restrict__ Ro,
                                                          int* __restrict__ piv,
                                                          int* __restrict__ state,
                                                          const double* __restrict__ tol_dev) {
  __shared__ double R11[32][33];
  __shared__ double s_row[32];
  __shared__ double s_dinv[32];  // 1 / R11[i][i]
  __shared__ int s_kb;
  // Only a stop recorded by an EARLIER panel launch ends this one: that panel left
  // state[0] = its rank < j0.  CTA 0 of THIS launch may set state[1] while other CTAs are
  // still to be dispatched; they must still write their off-diagonal columns of Ro (state[0]
  // is then >= j0; before this launch it was j0 or, at j0 = 0, 0).
  if (state[1] && state[0] < j0) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const int jb = min(32, n - j0);
  if (tid < 32) {
    const double tol = tol_dev[0];
    double a[32];
#pragma unroll
    for (int i = 0; i < 32; i++)
      a[i] = (i < jb && lane < jb) ? Hw[(int64_t)(j0 + i) * n + j0 + lane] : 0.0;
    int kb = jb;
    for (int j = 0; j < jb; j++) {
      double aj = 0.0;
#pragma unroll
      for (int i = 0; i < 32; i++)
        if (i == j) aj = a[i];
      const double d = __shfl_sync(0xffffffffu, aj, j);
      if (!(d > tol)) {  // warp-uniform: rank reached
        kb = j;
        break;
      }
      const double rinv = rsqrt(d), r = d * rinv;  // one special function on the chain
      const double rowj = lane == j ? r : (lane > j && lane < jb ? aj * rinv : 0.0);
      s_row[lane] = rowj;
      R11[j][lane] = rowj;
      if (lane == j) s_dinv[j] = rinv;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; i++)
        if (i > j) a[i] = fma(-s_row[i], rowj, a[i]);
      __syncwarp();
    }
    for (int j = kb; j < 32; j++) R11[j][lane] = 0.0;
    if (lane == 0) s_kb = kb;
    if (blockIdx.x == 0) {
      for (int i = 0; i < kb; i++)
        if (lane < jb) Ro[(int64_t)(j0 + i) * n + j0 + lane] = R11[i][lane];
      if (lane < jb) piv[j0 + lane] = j0 + lane;
      if (lane == 0) {
        state[0] = j0 + kb;
        if (kb < jb) state[1] = 1;
      }
    }
  }
  __syncthreads();
  const int kb = s_kb;
  const int c = j0 + 32 + blockIdx.x * UCT + tid;
  if (c < n && kb > 0) {
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; i++) x[i] = i < kb ? Hw[(int64_t)(j0 + i) * n + c] : 0.0;
#pragma unroll
    for (int i = 0; i < 32; i++) {
      if (i < kb) {
        x[i] *= s_dinv[i];
#pragma unroll
        for (int t = i + 1; t < 32; t++) x[t] = fma(-R11[i][t], x[i], x[t]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; i++)
      if (i < kb) Ro[(int64_t)(j0 + i) * n + c] = x[i];
  }
}

constexpr int TS_H = 64;

// Inverse of every 64 x 64 (or smaller, last) diagonal block of the upper triangular R,
// written into the matching diagonal blocks of X: one CTA per block.  All DI_T threads load the
// block (unrolled: the former 64-thread loop was a chain of 64 dependent L2 loads per thread)
// and store the result; thread c < h computes column c of the block inverse by back
// substitution with reciprocal diagonals (no division on the chain) and four partial sums.
constexpr int DI_T = 256;
__global__ void __launch_bounds__(DI_T) diag_inv_k(int k, const double* __restrict__ R,
                                                   int64_t ldr, double* __restrict__ X,
                                                   int64_t ldx) {
  extern __shared__ double dsm[];
  double(*Rs)[TS_H + 1] = reinterpret_cast<double(*)[TS_H + 1]>(dsm);
  double(*xs)[TS_H + 1] = reinterpret_cast<double(*)[TS_H + 1]>(dsm + TS_H * (TS_H + 1));
  __shared__ double rdiag[TS_H];
  const int i0 = blockIdx.x * TS_H, h = min(TS_H, k - i0), c = threadIdx.x;
#pragma unroll 4
  for (int e = c; e < TS_H * TS_H; e += DI_T) {
    const int i = e / TS_H, l = e % TS_H;
    Rs[i][l] = (i < h && l < h && l >= i) ? R[(int64_t)(i0 + i) * ldr + i0 + l] : 0.0;
  }
  __syncthreads();
  if (c < h) rdiag[c] = 1.0 / Rs[c][c];
  __syncthreads();
  if (c < h) {
    for (int i = h - 1; i >= 0; i--) {
      double s = (i == c) ? 1.0 : 0.0;
      if (i < c) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int l = i + 1;
        for (; l + 3 <= c; l += 4) {
          s0 = fma(Rs[i][l], xs[l][c], s0);
          s1 = fma(Rs[i][l + 1], xs[l + 1][c], s1);
          s2 = fma(Rs[i][l + 2], xs[l + 2][c], s2);
          s3 = fma(Rs[i][l + 3], xs[l + 3][c], s3);
        }
        for (; l <= c; l++) s0 = fma(Rs[i][l], xs[l][c], s0);
        s -= (s0 + s1) + (s2 + s3);
      }
      xs[i][c] = (i <= c) ? s * rdiag[i] : 0.0;
    }
  }
  __syncthreads();
  for (int e = c; e < h * h; e += DI_T) {
    const int i = e / h, l = e % h;
    X[(int64_t)(i0 + i) * ldx + i0 + l] = xs[i][l];
  }
}

// gather columns: out[t, c] = Ro[t, piv[c]]   (rows x k)
__global__ void gather_cols_k(int64_t rows, int k, const double* __restrict__ Ro, int64_t ldr,
                              const int* __restrict__ piv, double* __restrict__ out) {
  const int64_t total = rows * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / k;
    const int c = (int)(e % k);
    out[e] = Ro[t * ldr + piv[c]];
  }
}

// scatter rows: S[piv[i], :] = X[i, :] for i < k, other rows of S zero  (S: n x cols)
__global__ void scatter_rows_k(int64_t n, int k, int64_t cols, const double* __restrict__ X,
                               const int* __restrict__ piv, double* __restrict__ S) {
  const int64_t total = (int64_t)k * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / cols);
    const int64_t c = e % cols;
    S[(int64_t)piv[i] * cols + c] = X[e];
  }
}

int grid_for(tk_ctx* ctx, int64_t total) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8LL * ctx->num_sms));
}

}  // namespace

// Host poll of the stop flag (state[1]) every kCholPoll panels: once the factorisation has
// stopped the remaining panel launches and (skipped) updates only cost launch latency.
constexpr int kCholPoll = 2;
static int chol_stopped(tk_ctx* ctx, const int* state, bool* stopped) {
  int st = 0;
  TK_TRY(tk_read_host(ctx, ctx->stream, &st, state + 1, sizeof(int)));
  *stopped = st != 0;
  return TK_OK;
}

int tk_pchol_max_n() { return 4096; }

int tk_pchol(tk_ctx* ctx, int n, const double* H, double tol_rel, const double* tol_abs_dev,
             double* Ro, int* piv, int* state, bool pivot, double* rem_out) {
  if (n <= 0) return TK_OK;
  if (n > tk_pchol_max_n()) {
    ctx->err = "tk_pchol: n too large";
    return TK_EARG;
  }
  TagScope tag(ctx, "pchol");
  DevBuf Hw, tol;
  TK_TRY(Hw.get(ctx, (size_t)n * n));
  TK_TRY(tol.get(ctx, 1));
  TK_TRY(tk_copy2d(ctx, 1, (int64_t)n * n, H, (int64_t)n * n, Hw.p, (int64_t)n * n));
  TK_TRY(tk_zero(ctx, Ro, 1, sizeof(double) * n * n, sizeof(double) * n * n));
  TK_TRY(tk_zero(ctx, state, 1, (2 + (int64_t)n) * sizeof(int), (2 + (int64_t)n) * sizeof(int)));
  if (rem_out) TK_TRY(tk_zero(ctx, rem_out, 1, sizeof(double), sizeof(double)));
  max_diag_tol_k<<<1, 256, 0, ctx->stream>>>(n, H, tol_rel, tol_abs_dev, tol.p);
  TK_LAUNCH_CHECK(ctx);
  if (!pivot && !rem_out) {
    // unpivoted: blocked right-looking with a warp-level diagonal factorisation (no pivot search)
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int pid = tk_prof_begin(ctx, "pchol_panel", 0.0, 0.0);
      const int rest = n - j0 - 32;
      const int grid = std::max(1, (rest + UCT - 1) / UCT);
      chol_unpiv_panel_k<<<grid, UCT, 0, ctx->stream>>>(n, j0, Hw.p, Ro, piv, state, tol.p);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      if (rest > 0) {
        const int c1 = j0 + 32;
        // Hw[c1:, c1:] -= R12^T R12  (R12 = Ro[j0:j0+32, c1:]; no-op once stopped)
        TK_TRY(tk_dgemm(ctx, true, false, rest, rest, 32, -1.0, Ro + (int64_t)j0 * n + c1, n,
                        Ro + (int64_t)j0 * n + c1, n, 1.0, Hw.p + (int64_t)c1 * n + c1, n, true,
                        false, state + 1));
      }
      if (ctx->pinned && (j0 / 32 + 1) % kCholPoll == 0 && rest > 32) {
        bool stopped = false;
        TK_TRY(chol_stopped(ctx, state, &stopped));
        if (stopped) break;
      }
    }
    return TK_OK;
  }
  // register variant (n <= 2 PT): nb = 16 panel rows in registers, broadcast reads of the pivot
  // column from shared memory
  // 512 < n <= 1024: the register variant with 1024 threads (16 panel rows in registers)
  if (n > PT && n <= 2 * PT) {
    constexpr int NBR = 16;
    const size_t rsmem = (size_t)NBR * n * sizeof(double);
    static size_t rattr = 0;
    if (rattr < rsmem) {  // (also at <= 48 KB: the kernel has static shared memory too)
      cudaFuncSetAttribute(pchol_panel_reg_k<1, NBR, 2 * PT>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
      rattr = rsmem;
    }
    for (int j0 = 0; j0 < n; j0 += NBR) {
      const int pid = tk_prof_begin(ctx, "pchol_panel", 0.0, 0.0);
      pchol_panel_reg_k<1, NBR, 2 * PT><<<1, 2 * PT, rsmem, ctx->stream>>>(
          n, j0, pivot ? 1 : 0, Hw.p, Ro, piv, state, tol.p, rem_out);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      const int jb = std::min(NBR, n - j0);
      if (j0 + jb < n)
        TK_TRY(tk_dgemm(ctx, true, false, n, n, jb, -1.0, Ro + (int64_t)j0 * n, n,
                        Ro + (int64_t)j0 * n, n, 1.0, Hw.p, n, true, false, state + 1));
      if (ctx->pinned && (j0 / NBR + 1) % (2 * kCholPoll) == 0 && j0 + 2 * NBR < n) {
        bool stopped = false;
        TK_TRY(chol_stopped(ctx, state, &stopped));
        if (stopped) break;
      }
    }
    return TK_OK;
  }
  if (n <= PT) {
    // one column per thread: 32 panel rows fit in registers (for two columns per thread only
    // 16 do, and the doubled number of rank-nb updates then costs more than it saves)
    constexpr int NBR = 32;
    const size_t rsmem = (size_t)NBR * n * sizeof(double);
    static size_t rattr = 0;
    if (rattr < rsmem) {  // (also at <= 48 KB: the kernel has static shared memory too)
      cudaFuncSetAttribute(pchol_panel_reg_k<1, NBR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)rsmem);
      rattr = rsmem;
    }
    for (int j0 = 0; j0 < n; j0 += NBR) {
      const int pid = tk_prof_begin(ctx, "pchol_panel", 0.0, 0.0);
      pchol_panel_reg_k<1, NBR><<<1, PT, rsmem, ctx->stream>>>(n, j0, pivot ? 1 : 0, Hw.p, Ro, piv,
                                                              state, tol.p, rem_out);
      TK_LAUNCH_CHECK(ctx);
      tk_prof_end(ctx, pid);
      const int jb = std::min(NBR, n - j0);
      if (j0 + jb < n)
        TK_TRY(tk_dgemm(ctx, true, false, n, n, jb, -1.0, Ro + (int64_t)j0 * n, n,
                        Ro + (int64_t)j0 * n, n, 1.0, Hw.p, n, true, false, state + 1));
      if (ctx->pinned && (j0 / NBR + 1) % kCholPoll == 0 && j0 + 2 * NBR < n) {
        bool stopped = false;
        TK_TRY(chol_stopped(ctx, state, &stopped));
        if (stopped) break;
      }
    }
    return TK_OK;
  }
  // panel width: the panel rows of Ro (nb x n) and the diagonal stay in shared memory
  const int nb = (int)std::max<int64_t>(4, std::min<int64_t>(32, (200 * 1024 / 8) / n - 1));
  const size_t smem = ((size_t)nb + 1) * n * sizeof(double);
  static size_t attr = 0;
  if (attr < smem) {  // (also at <= 48 KB: static shared memory counts too)
    cudaFuncSetAttribute(pchol_panel_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  // balanced column ownership: every thread handles the same number of columns
  const int per = (n + PT - 1) / PT;
  const int threads = std::min(PT, 32 * (((n + per - 1) / per + 31) / 32));
  for (int j0 = 0; j0 < n; j0 += nb) {
    const int pid = tk_prof_begin(ctx, "pchol_panel", 0.0, 0.0);
    pchol_panel_k<<<1, threads, smem, ctx->stream>>>(n, j0, nb, pivot ? 1 : 0, Hw.p, Ro, piv,
                                                  state, tol.p, rem_out);
    TK_LAUNCH_CHECK(ctx);
    tk_prof_end(ctx, pid);
    const int jb = std::min(nb, n - j0);
    if (j0 + jb < n) {
      // Hw -= Ro[j0:j0+jb, :]^T Ro[j0:j0+jb, :]   (rows of a stopped panel are zero: no-op)
      TK_TRY(tk_dgemm(ctx, true, false, n, n, jb, -1.0, Ro + (int64_t)j0 * n, n,
                      Ro + (int64_t)j0 * n, n, 1.0, Hw.p, n, true, false, state + 1));
    }
    if (ctx->pinned && (j0 / nb + 1) % kCholPoll == 0 && j0 + 2 * nb < n) {
      bool stopped = false;
      TK_TRY(chol_stopped(ctx, state, &stopped));
      if (stopped) break;
    }
  }
  return TK_OK;
}

// X = R^{-1} (k x k upper triangular), blocked back substitution from the bottom block row:
//   X[I, J>I] = -R[I, I]^{-1} R[I, >I] X[>I, J],   X[I, I] = R[I, I]^{-1}
// (one DMMA GEMM and one diagonal-block solve per 64-row block).
// X = R^{-1} (k x k upper triangular), blocked from the bottom block row:
//   X[I, I] = D_I = R[I, I]^{-1}  (all 64 x 64 diagonal blocks at once, diag_inv_k)
//   X[I, >I] = -D_I (R[I, >I] X[>I, >I])   (two DMMA GEMMs per block row)
int tk_tri_inv(tk_ctx* ctx, int k, const double* R, int64_t ldr, double* X, int64_t ldx) {
  if (k <= 0) return TK_OK;
  TagScope tag(ctx, "tri_inv");
  TK_TRY(tk_zero(ctx, X, k, sizeof(double) * k, sizeof(double) * ldx));
  const int nbk = (k + TS_H - 1) / TS_H;
  {
    const int pid = tk_prof_begin(ctx, "tri_inv_diag", 0.0, 0.0);
    const size_t dsm = sizeof(double) * 2 * TS_H * (TS_H + 1);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(diag_inv_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
      attr = true;
    }
    diag_inv_k<<<nbk, DI_T, dsm, ctx->stream>>>(k, R, ldr, X, ldx);
    TK_LAUNCH_CHECK(ctx);
    tk_prof_end(ctx, pid);
  }
  DevBuf T;
  if (nbk > 1) TK_TRY(T.get(ctx, (size_t)TS_H * k));
  for (int b = nbk - 2; b >= 0; b--) {
    const int i0 = b * TS_H, i1 = i0 + TS_H, h = TS_H, w = k - i1;
    // T = R[i0:i1, i1:k] X[i1:k, i1:k]   (X block upper triangular)
    TK_TRY(tk_dgemm(ctx, false, false, h, w, w, 1.0, R + (int64_t)i0 * ldr + i1, ldr,
                    X + (int64_t)i1 * ldx + i1, ldx, 0.0, T.p, w, false, true));
    // X[i0:i1, i1:k] = -D_b T
    TK_TRY(tk_dgemm(ctx, false, false, h, w, h, -1.0, X + (int64_t)i0 * ldx + i0, ldx, T.p, w,
                    0.0, X + (int64_t)i0 * ldx + i1, ldx));
  }
  return TK_OK;
}

int tk_gather_cols(tk_ctx* ctx, int64_t rows, int k, const double* Ro, int64_t ldr, const int* piv,
                   double* out) {
  if (rows <= 0 || k <= 0) return TK_OK;
  gather_cols_k<<<grid_for(ctx, rows * k), 256, 0, ctx->stream>>>(rows, k, Ro, ldr, piv, out);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

int tk_scatter_rows(tk_ctx* ctx, int64_t n, int k, int64_t cols, const double* X, const int* piv,
                    double* S) {
  if (n <= 0 || cols <= 0) return TK_OK;
  TK_TRY(tk_zero(ctx, S, 1, sizeof(double) * n * cols, sizeof(double) * n * cols));
  if (k <= 0) return TK_OK;
  scatter_rows_k<<<grid_for(ctx, (int64_t)k * cols), 256, 0, ctx->stream>>>(n, k, cols, X, piv, S);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_chol_k() {}
const void* tk_anchor_k_chol() { return (const void*)tk_anchor_k_chol_k; }
