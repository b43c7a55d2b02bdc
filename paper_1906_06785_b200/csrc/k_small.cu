// Small fp64 helper kernels of the rounding / dot / axpby path (sm_100a).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>

#include "ttk_internal.h"

namespace {

inline int grid_for(tk_ctx* ctx, int64_t n, int threads = 256) {
  int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 16LL * ctx->num_sms));
}

// mode 0: dst = src * f[col]; 1: dst = src / f[col] (0 where f == 0)
__global__ void col_scale_k(int64_t rows, int64_t cols, const double* __restrict__ src,
                            int64_t lds, double* __restrict__ dst, int64_t ldd,
                            const double* __restrict__ f, int mode) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    double s = src[r * lds + c], g = f[c];
    dst[r * ldd + c] = mode == 0 ? s * g : (g != 0.0 ? s / g : 0.0);
  }
}

__global__ void row_scale_k(int64_t rows, int64_t cols, const double* __restrict__ src,
                            int64_t lds, double* __restrict__ dst, int64_t ldd,
                            const double* __restrict__ f, int mode) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    double s = src[r * lds + c], g = f[r];
    dst[r * ldd + c] = mode == 0 ? s * g : (g != 0.0 ? s / g : 0.0);
  }
}

__global__ void copy2d_k(int64_t rows, int64_t cols, const double* __restrict__ src, int64_t lds,
                         double* __restrict__ dst, int64_t ldd) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

// zero a rows x cols block (leading dimension ld, in 4-byte words: serves doubles and ints)
__global__ void zero2d_k(int64_t rows, int64_t cols, uint32_t* __restrict__ dst, int64_t ld) {
  int64_t n = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / cols, c = e % cols;
    dst[r * ld + c] = 0u;
  }
}

__global__ void fill_k(double* dst, int64_t n, double v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = v;
}

__global__ void eye_k(double* dst, int64_t n) {
  int64_t nn = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// Rank rule of PAPER.md:247-249 / SPEC.md:105,109 on sigma = sqrt(max(lam,0)), lam descending.
// One warp: tail sums accumulated from the smallest value upward, sequentially (n <= a few
// thousand), so the result does not depend on the launch shape.
__global__ void rank_select_k(int n, const double* __restrict__ lam, double* __restrict__ sig,
                              double tol, const double* __restrict__ delta_in, int64_t rmax,
                              double kthr, int* __restrict__ info, double* __restrict__ dinfo,
                              int rcap) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) sig[i] = sqrt(fmax(lam[i], 0.0));
  __syncwarp();
  if (threadIdx.x != 0) return;
  info[2] = rcap;
  double nrm2 = 0.0;
  for (int i = n - 1; i >= 0; i--) nrm2 += sig[i] * sig[i];
  double nrm = sqrt(nrm2);
  double delta = delta_in ? delta_in[0] : tol * nrm / sqrt(2.0);
  // smallest r >= 1 with ||sig[r:]|| <= delta
  double tail2 = 0.0;
  int r = n;
  // walk from the end: tail2 after adding sig[j] is ||sig[j:]||^2
  // r = smallest cand with ||sig[cand:]|| <= delta; iterate cand from n down to 1
  for (int cand = n; cand >= 1; cand--) {
    double t = (cand < n) ? sqrt(tail2) : 0.0;
    if (t <= delta)
      r = cand;
    else
      break;
    if (cand - 1 >= 0) tail2 += sig[cand - 1] * sig[cand - 1];
  }
  while (r < n && sig[r] == sig[r - 1]) r++;
  if (rmax > 0 && r > rmax) r = (int)rmax;
  // only the first rcap eigenpairs are resolved (pass2_chol: entries >= kc hold the Schur
  // remainder, which counts in the discarded tail but has no singular vector)
  if (r > rcap) r = rcap;
  if (r < 1) r = 1;
  int k = 0;
  for (int i = 0; i < n; i++)
    if (sig[i] > kthr * sig[0]) k = i + 1;
  if (k < 1) k = 1;
  double disc2 = 0.0;
  for (int i = n - 1; i >= r; i--) disc2 += sig[i] * sig[i];
  info[0] = r;
  info[1] = k;
  dinfo[0] = nrm;
  dinfo[1] = delta;
  dinfo[2] = sqrt(disc2);
}

// z = a x + b y cores (concatenation)
// z1 = [x1 | y1] (n_x x (rx + ry)): a pure copy stream.  One thread per element (or per
// 16-byte pair when rx, ry are even and the bases aligned); 32-bit index arithmetic when the
// element count fits (the 64-bit division per element made the copy ALU-bound).
template <typename I, bool V2>
__global__ void axpby_u1_k(I n_x, I rx, I ry, const double* __restrict__ x1,
                           const double* __restrict__ y1, double* __restrict__ z1) {
  constexpr int W = V2 ? 2 : 1;
  const I ux = rx / W, uy = ry / W, U = ux + uy, n = n_x * U;
  for (I e = blockIdx.x * (I)blockDim.x + threadIdx.x; e < n; e += (I)gridDim.x * blockDim.x) {
    const I i = e / U, c = e - i * U;
    if (V2) {
      const double2 v = c < ux ? __ldcs((const double2*)x1 + i * ux + c)
                               : __ldcs((const double2*)y1 + i * uy + (c - ux));
      __stcs((double2*)z1 + e, v);
    } else {
      z1[e] = c < ux ? __ldcs(x1 + i * ux + c) : __ldcs(y1 + i * uy + (c - ux));
    }
  }
}
__global__ void axpby_u2_k(int64_t rx1, int64_t ry1, int64_t n_xi, int64_t rx2, int64_t ry2,
                           const double* __restrict__ x2, const double* __restrict__ y2,
                           double* __restrict__ z2) {
  int64_t R1 = rx1 + ry1, R2 = rx2 + ry2, n = R1 * n_xi * R2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e % R2, t = e / R2, i = t % n_xi, a = t / n_xi;
    double v = 0.0;
    if (a < rx1 && b < rx2)
      v = x2[(a * n_xi + i) * rx2 + b];
    else if (a >= rx1 && b >= rx2)
      v = y2[((a - rx1) * n_xi + i) * ry2 + (b - rx2)];
    z2[e] = v;
  }
}
__global__ void axpby_u3_k(int64_t rx2, int64_t ry2, int64_t n_t, const double* __restrict__ a,
                           const double* __restrict__ x3, const double* __restrict__ b,
                           const double* __restrict__ y3, double* __restrict__ z3) {
  int64_t n = (rx2 + ry2) * n_t;
  double av = a[0], bv = b[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / n_t;
    z3[e] = r < rx2 ? av * x3[e] : bv * y3[e - rx2 * n_t];
  }
}

__global__ void scale_k(double* U, int64_t n, const double* s, int invert) {
  double f = invert ? 1.0 / s[0] : s[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    U[e] *= f;
}

// out = sum(a .* b) (single block, deterministic order); optional sqrt
__global__ void dot_final_k(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                            double* out, int take_sqrt) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) s += a[e] * b[e];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = take_sqrt ? sqrt(fmax(red[0], 0.0)) : red[0];
}

__global__ void set_scalar_k(double* dst, double v) { dst[0] = v; }

// per-CTA partial sums of squares of P (fixed-order tree; summed in CTA order by noise_floor_k:
// deterministic).  One CTA took ~160 us for the 896 x 640 P of c4's bond 1, right before form_W.
constexpr int NF_T = 256, NF_MAXG = 148;
__global__ void __launch_bounds__(NF_T) sumsq_partial_k(int64_t nP, const double* __restrict__ P,
                                                        double* __restrict__ part) {
  __shared__ double red[NF_T];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  const int64_t stride = (int64_t)gridDim.x * NF_T;
  int64_t e = (int64_t)blockIdx.x * NF_T + threadIdx.x;
  for (; e + 3 * stride < nP; e += 4 * stride) {
    const double a0 = P[e], a1 = P[e + stride], a2 = P[e + 2 * stride], a3 = P[e + 3 * stride];
    s0 = fma(a0, a0, s0);
    s1 = fma(a1, a1, s1);
    s2 = fma(a2, a2, s2);
    s3 = fma(a3, a3, s3);
  }
  for (; e < nP; e += stride) s0 = fma(P[e], P[e], s0);
  red[threadIdx.x] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  for (int st = NF_T / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// trace of an n x n matrix (row-major) and ||P||_F^2 (npart partial sums), then the noise floor
__global__ void noise_floor_k(const double* __restrict__ G, int64_t n, double gscale,
                              const double* __restrict__ part, int npart, int64_t K, int64_t k,
                              double* out) {
  __shared__ double r1[256];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += G[i * n + i];
  r1[threadIdx.x] = a;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) r1[threadIdx.x] += r1[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double eps = 2.220446049250313e-16;
    double pf2 = (double)k;
    if (part) {
      pf2 = 0.0;
      for (int i = 0; i < npart; i++) pf2 += part[i];
    }
    out[0] = 16.0 * eps * eps * (double)K * (gscale * r1[0]) * pf2 / (double)k;
  }
}
__global__ void neg_scalar_k(const double* src, double* dst) { dst[0] = -src[0]; }

__global__ void transpose_k(int64_t rows, int64_t cols, const double* __restrict__ src,
                            int64_t lds, double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  for (int64_t r0 = (int64_t)blockIdx.y * 32; r0 < rows; r0 += (int64_t)gridDim.y * 32)
    for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < cols; c0 += (int64_t)gridDim.x * 32) {
      for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        int64_t r = r0 + dy, c = c0 + threadIdx.x;
        tile[dy][threadIdx.x] = (r < rows && c < cols) ? src[r * lds + c] : 0.0;
      }
      __syncthreads();
      for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
        int64_t c = c0 + dy, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][dy];
      }
      __syncthreads();
    }
}

__global__ void symmetrize_k(int64_t n, double* A) {
  int64_t nn = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / n, j = e % n;
    if (j > i) {
      double v = 0.5 * (A[i * n + j] + A[j * n + i]);
      A[i * n + j] = v;
      A[j * n + i] = v;
    }
  }
}

}  // namespace

int tk_noise_floor(tk_ctx* ctx, const double* trG_src, int64_t n_trG, double trG_scale,
                   const double* P, int64_t nP, int64_t K, int64_t k, double* out) {
  DevBuf part;
  int g = 0;
  if (P) {
    g = (int)std::max<int64_t>(1, std::min<int64_t>(NF_MAXG, nP / (8 * NF_T)));
    TK_TRY(part.get(ctx, (size_t)g));
    sumsq_partial_k<<<g, NF_T, 0, ctx->stream>>>(nP, P, part.p);
    TK_LAUNCH_CHECK(ctx);
  }
  noise_floor_k<<<1, 256, 0, ctx->stream>>>(trG_src, n_trG, trG_scale, P ? part.p : nullptr, g, K, k,
                                            out);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_neg_scalar(tk_ctx* ctx, const double* src, double* dst) {
  neg_scalar_k<<<1, 1, 0, ctx->stream>>>(src, dst);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_transpose(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd) {
  if (rows <= 0 || cols <= 0) return TK_OK;
  dim3 grid((unsigned)std::min<int64_t>((cols + 31) / 32, 1024),
            (unsigned)std::min<int64_t>((rows + 31) / 32, 1024));
  transpose_k<<<grid, dim3(32, 8), 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_symmetrize(tk_ctx* ctx, int64_t n, double* A) {
  if (n <= 1) return TK_OK;
  symmetrize_k<<<grid_for(ctx, n * n), 256, 0, ctx->stream>>>(n, A);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

int tk_col_scale(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd, const double* f, int mode) {
  if (rows <= 0 || cols <= 0) return TK_OK;
  col_scale_k<<<grid_for(ctx, rows * cols), 256, 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd,
                                                                   f, mode);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_row_scale(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd, const double* f, int mode) {
  if (rows <= 0 || cols <= 0) return TK_OK;
  row_scale_k<<<grid_for(ctx, rows * cols), 256, 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd,
                                                                   f, mode);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_copy2d(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
              double* dst, int64_t ldd) {
  if (rows <= 0 || cols <= 0) return TK_OK;
  copy2d_k<<<grid_for(ctx, rows * cols), 256, 0, ctx->stream>>>(rows, cols, src, lds, dst, ldd);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
// Kernel zero-fill / copy (not cudaMemsetAsync / cudaMemcpyAsync): the rounding's critical path
// must not share the copy engines with a user's concurrent bulk H2D / D2H transfers (measured:
// a 408 MB H2D beside a c4 op slowed it by ~6 ms).
int tk_zero(tk_ctx* ctx, void* dst, int64_t rows, int64_t cols_bytes, int64_t ld_bytes) {
  if (rows <= 0 || cols_bytes <= 0) return TK_OK;
  const int64_t cw = (cols_bytes + 3) / 4, lw = ld_bytes / 4;
  zero2d_k<<<grid_for(ctx, rows * cw), 256, 0, ctx->stream>>>(rows, cw, (uint32_t*)dst, lw);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_fill(tk_ctx* ctx, double* dst, int64_t n, double v) {
  if (n <= 0) return TK_OK;
  fill_k<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(dst, n, v);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_eye(tk_ctx* ctx, double* dst, int64_t n) {
  if (n <= 0) return TK_OK;
  eye_k<<<grid_for(ctx, n * n), 256, 0, ctx->stream>>>(dst, n);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_rank_select(tk_ctx* ctx, int n, const double* lam, double* sig, double tol,
                   const double* delta_dev_in, int64_t rmax, double kthr, int* info,
                   double* dinfo, int rcap) {
  rank_select_k<<<1, 32, 0, ctx->stream>>>(n, lam, sig, tol, delta_dev_in, rmax, kthr, info,
                                           dinfo, rcap > 0 ? std::min(rcap, n) : n);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_axpby_cores(tk_ctx* ctx, const double* a_dev, const tk_tt* x, const double* b_dev,
                   const tk_tt* y, tk_tt* z) {
  int64_t R1 = x->r1 + y->r1, R2 = x->r2 + y->r2;
  {
    const bool v2 = x->r1 % 2 == 0 && y->r1 % 2 == 0 && ((uintptr_t)x->U1 & 15) == 0 &&
                    ((uintptr_t)y->U1 & 15) == 0 && ((uintptr_t)z->U1 & 15) == 0;
    const int64_t n = x->n_x * R1 / (v2 ? 2 : 1);
    const int g = grid_for(ctx, n);
    if (n < (int64_t)INT32_MAX - 256LL * g) {
      if (v2)
        axpby_u1_k<uint32_t, true><<<g, 256, 0, ctx->stream>>>(
            (uint32_t)x->n_x, (uint32_t)x->r1, (uint32_t)y->r1, x->U1, y->U1, z->U1);
      else
        axpby_u1_k<uint32_t, false><<<g, 256, 0, ctx->stream>>>(
            (uint32_t)x->n_x, (uint32_t)x->r1, (uint32_t)y->r1, x->U1, y->U1, z->U1);
    } else if (v2) {
      axpby_u1_k<int64_t, true><<<g, 256, 0, ctx->stream>>>(x->n_x, x->r1, y->r1, x->U1, y->U1,
                                                             z->U1);
    } else {
      axpby_u1_k<int64_t, false><<<g, 256, 0, ctx->stream>>>(x->n_x, x->r1, y->r1, x->U1, y->U1,
                                                              z->U1);
    }
  }
  TK_LAUNCH_CHECK(ctx);
  axpby_u2_k<<<grid_for(ctx, R1 * x->n_xi * R2), 256, 0, ctx->stream>>>(
      x->r1, y->r1, x->n_xi, x->r2, y->r2, x->U2, y->U2, z->U2);
  TK_LAUNCH_CHECK(ctx);
  axpby_u3_k<<<grid_for(ctx, R2 * x->n_t), 256, 0, ctx->stream>>>(x->r2, y->r2, x->n_t, a_dev,
                                                                  x->U3, b_dev, y->U3, z->U3);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_scale_rows(tk_ctx* ctx, double* U3, int64_t n, const double* s_dev, int invert) {
  scale_k<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(U3, n, s_dev, invert);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_dot_final(tk_ctx* ctx, int64_t n, const double* a, const double* b, double* out,
                 int take_sqrt) {
  dot_final_k<<<1, 256, 0, ctx->stream>>>(n, a, b, out, take_sqrt);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}
int tk_set_scalar(tk_ctx* ctx, double* dst, double v) {
  set_scalar_k<<<1, 1, 0, ctx->stream>>>(dst, v);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

namespace {
__global__ void col_norms_k(int64_t rows, int64_t cols, const double* __restrict__ A, int64_t lda,
                            double* __restrict__ out) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < cols;
       c += (int64_t)gridDim.x * blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    int64_t r = 0;
    for (; r + 1 < rows; r += 2) {
      const double a = A[r * lda + c], b = A[(r + 1) * lda + c];
      s0 = fma(a, a, s0);
      s1 = fma(b, b, s1);
    }
    if (r < rows) s0 = fma(A[r * lda + c], A[r * lda + c], s0);
    out[c] = sqrt(s0 + s1);
  }
}
}  // namespace

int tk_col_norms(tk_ctx* ctx, int64_t rows, int64_t cols, const double* A, int64_t lda,
                 double* out) {
  if (cols <= 0) return TK_OK;
  col_norms_k<<<(int)((cols + 127) / 128), 128, 0, ctx->stream>>>(rows, cols, A, lda, out);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

namespace {
// out[b][q][p][w] = in[b][p][q][w]  (w contiguous)
__global__ void swap_mid_k(int64_t nb, int64_t np, int64_t nq, int64_t nw,
                           const double* __restrict__ in, double* __restrict__ out) {
  const int64_t total = nb * np * nq * nw;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = e % nw;
    int64_t t = e / nw;
    const int64_t q = t % nq;
    t /= nq;
    const int64_t p = t % np;
    const int64_t b = t / np;
    out[((b * nq + q) * np + p) * nw + w] = in[e];
  }
}
}  // namespace

int tk_swap_mid(tk_ctx* ctx, int64_t nb, int64_t np, int64_t nq, int64_t nw, const double* in,
                double* out) {
  const int64_t total = nb * np * nq * nw;
  if (total <= 0) return TK_OK;
  swap_mid_k<<<grid_for(ctx, total), 256, 0, ctx->stream>>>(nb, np, nq, nw, in, out);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

namespace {
__global__ void group_rows_k(int T, int G, int64_t r, int64_t c, const int* __restrict__ group,
                             const double* __restrict__ coef, const double* __restrict__ L,
                             double* __restrict__ Lg) {
  const int64_t n = (int64_t)G * r * c;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % c, ga = e / c, a = ga % r;
    const int g = (int)(ga / r);
    double s = 0.0;
    for (int k = 0; k < T; k++)
      if (group[k] == g) s = fma(coef[k], L[((int64_t)k * r + a) * c + j], s);
    Lg[e] = s;
  }
}
}  // namespace

int tk_group_rows(tk_ctx* ctx, int T, int G, int64_t r, int64_t c, const int* group,
                  const double* coef, const double* L, double* Lg) {
  const int64_t n = (int64_t)G * r * c;
  if (n <= 0) return TK_OK;
  group_rows_k<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(T, G, r, c, group, coef, L, Lg);
  TK_LAUNCH_CHECK(ctx);
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_small_k() {}
const void* tk_anchor_k_small() { return (const void*)tk_anchor_k_small_k; }
