// NEXT-3: the mean-based preconditioner of PAPER.md section 5 on the device.
//
//   * tk_bt: block-tridiagonal direct solves of the spatial factors (the "solve with" of
//     eq:mean_lsc and eq:11_prec): block LU (block Thomas) over the grid
//     lines of the lexicographic FD ordering (R10), dense N x N blocks on DMMA.
//   * tk_prec: P^{-1} of eq:prec with S_LSC,0 (eq:mean_lsc) and the inner
//     (F0 + C) GMRES (eq:11_sys) preconditioned by M (eq:11_prec) — the steps of DESIGN.md R20.
// See include/ttk.h for the contracts.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <memory>
#include <vector>

#include "ttk_internal.h"

// ============================================================================ kernels
namespace {

int grid1(int64_t n, int threads = 256) {
  return (int)std::min<int64_t>((n + threads - 1) / threads, 148 * 32);
}

// Dense blocks of K = A + shift I from the CSR A: D_i = K[i, i], Lo_i = K[i, i-1],
// Up_i = K[i, i+1] (N x N row-major each, pre-zeroed).  One thread per row (sums in CSR order).
__global__ void bt_blocks_csr_k(int64_t n, int64_t N, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ cl, const double* __restrict__ v,
                                double shift, double* __restrict__ D, double* __restrict__ Lo,
                                double* __restrict__ Up, int* __restrict__ bad) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = row / N, a = row % N;
    const int64_t base = i * N * N + a * N;
    for (int32_t e = rp[row]; e < rp[row + 1]; e++) {
      const int64_t c = cl[e], j = c / N, b = c % N;
      if (j == i)
        D[base + b] += v[e];
      else if (j == i - 1)
        Lo[base + b] += v[e];
      else if (j == i + 1)
        Up[base + b] += v[e];
      else
        atomicExch(bad, 1);
    }
    D[base + a] += shift;
  }
}

// Dense blocks of K = B B^T (B: n x ncols CSR): entry (a, b) for b in the block rows
// i-1 .. i+1 of a = sum over the shared columns c of B[a, c] B[b, c] (row a's CSR order).
__global__ void bt_blocks_gram_k(int64_t n, int64_t N, int64_t nb,
                                 const int32_t* __restrict__ rp, const int32_t* __restrict__ cl,
                                 const double* __restrict__ v, double* __restrict__ D,
                                 double* __restrict__ Lo, double* __restrict__ Up) {
  const int64_t total = n * 3 * N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = g / (3 * N), t = g % (3 * N);
    const int64_t i = a / N, j = i - 1 + t / N;
    if (j < 0 || j >= nb) continue;
    const int64_t b = j * N + t % N;
    double s = 0.0;
    for (int32_t e = rp[a]; e < rp[a + 1]; e++) {
      const int32_t c = cl[e];
      for (int32_t f = rp[b]; f < rp[b + 1]; f++)
        if (cl[f] == c) s = fma(v[e], v[f], s);
    }
    double* dst = (j == i ? D : (j == i - 1 ? Lo : Up)) + i * N * N + (a % N) * N + (b % N);
    *dst = s;
  }
}

// (I - C)^{-1} on the time core: each row of U3 (r2 x n_t) replaced by its cumulative sum
// (C = the unit sub-diagonal shift).  One thread per row, sequential in t.
__global__ void time_cumsum_k(int64_t rows, int64_t n_t, const double* __restrict__ x,
                              double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t t = 0; t < n_t; t++) {
      s += x[r * n_t + t];
      y[r * n_t + t] = s;
    }
  }
}

}  // namespace

// X = A^{-1} (n x n, row-major) via the Householder QR A = Q R: X = R^{-1} Q^T.
static int dense_inv(tk_ctx* ctx, int n, const double* A, double* X) {
  DevBuf Q, R, Ri;
  TK_TRY(Q.get(ctx, (size_t)n * n));
  TK_TRY(R.get(ctx, (size_t)n * n));
  TK_TRY(Ri.get(ctx, (size_t)n * n));
  TK_TRY(tk_householder_q(ctx, n, A, Q.p));
  TK_TRY(tk_dgemm(ctx, true, false, n, n, n, 1.0, Q.p, n, A, n, 0.0, R.p, n));  // R = Q^T A
  TK_TRY(tk_tri_inv(ctx, n, R.p, n, Ri.p, n));
  TK_TRY(tk_dgemm(ctx, false, true, n, n, n, 1.0, Ri.p, n, Q.p, n, 0.0, X, n));  // R^-1 Q^T
  return TK_OK;
}

// ============================================================================ tk_bt
struct tk_bt {
  tk_ctx* ctx = nullptr;
  int64_t nb = 0, N = 0;
  double* E = nullptr;  // nb blocks S_i^{-1}
  double* F = nullptr;  // nb blocks E_i U_i (i < nb - 1)
  double* G = nullptr;  // nb blocks E_i L_i (i > 0)
};

extern "C" int tk_bt_destroy(tk_bt* bt) {
  { tk_ctx* _gc = bt ? bt->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  if (!bt) return TK_OK;
  cudaFree(bt->E);
  cudaFree(bt->F);
  cudaFree(bt->G);
  delete bt;
  return TK_OK;
}

// Block LU of the block-tridiagonal K from its dense blocks D, Lo, Up (device, nb N^2 each).
static int bt_factor(tk_ctx* ctx, tk_bt* bt, const double* D, const double* Lo,
                     const double* Up) {
  const int64_t nb = bt->nb, N = bt->N, NN = N * N;
  DevBuf S;
  TK_TRY(S.get(ctx, NN));
  TagScope tag(ctx, "bt_factor");
  for (int64_t i = 0; i < nb; i++) {
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(S.p, D + i * NN, sizeof(double) * NN,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
    if (i > 0)  // S_i = D_i - L_i F_{i-1}
      TK_TRY(tk_dgemm(ctx, false, false, N, N, N, -1.0, Lo + i * NN, N, bt->F + (i - 1) * NN, N,
                      1.0, S.p, N));
    TK_TRY(dense_inv(ctx, (int)N, S.p, bt->E + i * NN));
    if (i + 1 < nb)
      TK_TRY(tk_dgemm(ctx, false, false, N, N, N, 1.0, bt->E + i * NN, N, Up + i * NN, N, 0.0,
                      bt->F + i * NN, N));
    if (i > 0)
      TK_TRY(tk_dgemm(ctx, false, false, N, N, N, 1.0, bt->E + i * NN, N, Lo + i * NN, N, 0.0,
                      bt->G + i * NN, N));
  }
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TK_OK;
}

static int bt_alloc(tk_ctx* ctx, int64_t nb, int64_t N, std::unique_ptr<tk_bt>& bt) {
  bt.reset(new tk_bt());
  bt->ctx = ctx;
  bt->nb = nb;
  bt->N = N;
  const size_t bytes = sizeof(double) * nb * N * N;
  TK_CUDA_TRY(ctx, cudaMalloc(&bt->E, bytes));
  TK_CUDA_TRY(ctx, cudaMalloc(&bt->F, bytes));
  TK_CUDA_TRY(ctx, cudaMalloc(&bt->G, bytes));
  return TK_OK;
}

struct DevInts {
  int32_t* p = nullptr;
  ~DevInts() { cudaFree(p); }
};

static int upload_csr(tk_ctx* ctx, int64_t n, const int32_t* rowptr, const int32_t* col,
                      const double* val, DevInts& drp, DevInts& dcl, DevBuf& dv) {
  const int64_t nnz = rowptr[n];
  TK_CUDA_TRY(ctx, cudaMalloc(&drp.p, sizeof(int32_t) * (n + 1)));
  TK_CUDA_TRY(ctx, cudaMalloc(&dcl.p, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  TK_TRY(dv.get(ctx, std::max<int64_t>(nnz, 1)));
  TK_CUDA_TRY(ctx, cudaMemcpy(drp.p, rowptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice));
  if (nnz > 0) {
    TK_CUDA_TRY(ctx, cudaMemcpy(dcl.p, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(dv.p, val, sizeof(double) * nnz, cudaMemcpyHostToDevice,
                                     ctx->stream));
  }
  return TK_OK;
}

static bool csr_ok(int64_t n, int64_t ncols, const int32_t* rp, const int32_t* cl) {
  if (!rp || rp[0] != 0) return false;
  for (int64_t i = 0; i < n; i++)
    if (rp[i + 1] < rp[i]) return false;
  for (int64_t e = 0; e < rp[n]; e++)
    if (cl[e] < 0 || cl[e] >= ncols) return false;
  return true;
}

static int bt_create_impl(tk_ctx* ctx, tk_bt** out, int64_t nb, int64_t N, int64_t ncols,
                          const int32_t* rowptr, const int32_t* col, const double* val,
                          double shift, bool gram) {
  if (!ctx || !out || nb < 1 || N < 1 || !rowptr || (rowptr[nb * N] > 0 && (!col || !val)))
    return TK_EARG;
  const int64_t n = nb * N;
  if (!csr_ok(n, gram ? ncols : n, rowptr, col)) {
    ctx->err = "tk_bt_create: malformed CSR";
    return TK_EARG;
  }
  if (gram) {  // every column of B must couple rows of adjacent block rows only
    std::vector<int64_t> lo(ncols, INT64_MAX), hi(ncols, -1);
    for (int64_t r = 0; r < n; r++)
      for (int32_t e = rowptr[r]; e < rowptr[r + 1]; e++) {
        lo[col[e]] = std::min(lo[col[e]], r / N);
        hi[col[e]] = std::max(hi[col[e]], r / N);
      }
    for (int64_t c = 0; c < ncols; c++)
      if (hi[c] >= 0 && hi[c] - lo[c] > 1) {
        ctx->err = "tk_bt_create_gram: B B^T is not block tridiagonal in blocks of N rows";
        return TK_EARG;
      }
  }
  std::unique_ptr<tk_bt> bt;
  TK_TRY(bt_alloc(ctx, nb, N, bt));
  {
    DevInts drp, dcl;
    DevBuf dv, D, Lo, Up, bad;
    TK_TRY(upload_csr(ctx, n, rowptr, col, val, drp, dcl, dv));
    TK_TRY(D.get(ctx, nb * N * N));
    TK_TRY(Lo.get(ctx, nb * N * N));
    TK_TRY(Up.get(ctx, nb * N * N));
    TK_TRY(bad.get(ctx, 1));
    TK_CUDA_TRY(ctx, cudaMemsetAsync(D.p, 0, sizeof(double) * nb * N * N, ctx->stream));
    TK_CUDA_TRY(ctx, cudaMemsetAsync(Lo.p, 0, sizeof(double) * nb * N * N, ctx->stream));
    TK_CUDA_TRY(ctx, cudaMemsetAsync(Up.p, 0, sizeof(double) * nb * N * N, ctx->stream));
    TK_CUDA_TRY(ctx, cudaMemsetAsync(bad.p, 0, sizeof(double), ctx->stream));
    if (gram) {
      bt_blocks_gram_k<<<grid1(n * 3 * N), 256, 0, ctx->stream>>>(n, N, nb, drp.p, dcl.p, dv.p,
                                                                  D.p, Lo.p, Up.p);
    } else {
      bt_blocks_csr_k<<<grid1(n), 256, 0, ctx->stream>>>(n, N, drp.p, dcl.p, dv.p, shift, D.p,
                                                         Lo.p, Up.p, (int*)bad.p);
    }
    TK_LAUNCH_CHECK(ctx);
    int hbad = 0;
    TK_TRY(tk_sync_read(ctx, &hbad, bad.p, sizeof(int)));
    if (hbad) {
      ctx->err = "tk_bt_create: an entry lies outside the block-tridiagonal band";
      return TK_EARG;
    }
    TK_TRY(bt_factor(ctx, bt.get(), D.p, Lo.p, Up.p));
  }
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  *out = bt.release();
  return TK_OK;
}

extern "C" int tk_bt_create(tk_ctx* ctx, tk_bt** bt, int64_t nb, int64_t N, const int32_t* rowptr,
                            const int32_t* col, const double* val, double shift) {
  TK_ASYNC_GUARD(ctx);
  return bt_create_impl(ctx, bt, nb, N, nb * N, rowptr, col, val, shift, false);
}

extern "C" int tk_bt_create_gram(tk_ctx* ctx, tk_bt** bt, int64_t nb, int64_t N, int64_t ncols,
                                 const int32_t* rowptr, const int32_t* col, const double* val) {
  TK_ASYNC_GUARD(ctx);
  if (ncols < 1) return TK_EARG;
  return bt_create_impl(ctx, bt, nb, N, ncols, rowptr, col, val, 0.0, true);
}

// y = K^{-1} applied to rows [row0, row0 + reps n) of x's space core (zero elsewhere).
static int bt_solve_impl(tk_ctx* ctx, const tk_bt* bt, const tk_tt* x, int64_t row0, int reps,
                         tk_tt* y) {
  const int64_t nb = bt->nb, N = bt->N, NN = N * N, n = nb * N, r = x->r1;
  if (row0 < 0 || reps < 1 || row0 + reps * n > x->n_x) {
    ctx->err = "tk_bt_solve: row range outside the space mode";
    return TK_EARG;
  }
  if (y->n_x != x->n_x || y->n_xi != x->n_xi || y->n_t != x->n_t) {
    ctx->err = "tk_bt_solve: mode sizes differ";
    return TK_ESHAPE;
  }
  if (y->cap1 < x->r1 || y->cap2 < x->r2) {
    ctx->err = "tk_bt_solve: output capacity";
    return TK_ECAP;
  }
  TagScope tag(ctx, "bt_solve");
  y->r1 = x->r1;
  y->r2 = x->r2;
  TK_TRY(tk_zero(ctx, y->U1, 1, sizeof(double) * x->n_x * r, sizeof(double) * x->n_x * r));
  {
    const int64_t n2 = x->r1 * x->n_xi * x->r2, n3 = x->r2 * x->n_t;
    TK_TRY(tk_copy2d(ctx, 1, n2, x->U2, n2, y->U2, n2));
    TK_TRY(tk_copy2d(ctx, 1, n3, x->U3, n3, y->U3, n3));
  }
  for (int s = 0; s < reps; s++) {
    const double* B = x->U1 + (row0 + s * n) * r;
    double* Y = y->U1 + (row0 + s * n) * r;
    for (int64_t i = 0; i < nb; i++) {  // forward: y_i = E_i b_i - G_i y_{i-1}
      TK_TRY(tk_dgemm(ctx, false, false, N, r, N, 1.0, bt->E + i * NN, N, B + i * N * r, r, 0.0,
                      Y + i * N * r, r));
      if (i > 0)
        TK_TRY(tk_dgemm(ctx, false, false, N, r, N, -1.0, bt->G + i * NN, N, Y + (i - 1) * N * r,
                        r, 1.0, Y + i * N * r, r));
    }
    for (int64_t i = nb - 2; i >= 0; i--)  // back: x_i = y_i - F_i x_{i+1}
      TK_TRY(tk_dgemm(ctx, false, false, N, r, N, -1.0, bt->F + i * NN, N, Y + (i + 1) * N * r,
                      r, 1.0, Y + i * N * r, r));
  }
  return TK_OK;
}

static int check_tt_basic(tk_ctx* ctx, const tk_tt* x) {
  if (!x || !x->U1 || !x->U2 || !x->U3 || x->r1 < 1 || x->r2 < 1 || x->n_x < 1 || x->n_xi < 1 ||
      x->n_t < 1) {
    ctx->err = "invalid TT";
    return TK_EARG;
  }
  return TK_OK;
}

extern "C" int tk_bt_solve(tk_ctx* ctx, const tk_bt* bt, const tk_tt* x, int64_t row0, int reps,
                           tk_tt* y) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !bt) return TK_EARG;
  TK_TRY(check_tt_basic(ctx, x));
  TK_TRY(check_tt_basic(ctx, y));
  return bt_solve_impl(ctx, bt, x, row0, reps, y);
}

// ============================================================================ tk_prec
struct tk_prec {
  tk_ctx* ctx = nullptr;
  int64_t n_v = 0, n_p = 0, n_x = 0, n_xi = 0, n_t = 0;
  double tau = 0.0, tol = 0.0, tol_in = 0.1;
  int restart_in = 10, max_cycles_in = 3;
  tk_bt* bt_v = nullptr;  // K_s = tau^-1 I + F0s (eq:11_prec)
  tk_bt* bt_p = nullptr;  // B B^T (eq:mean_lsc, M* = I)
  tk_op* op_F0C = nullptr, *op_Bt = nullptr, *op_B = nullptr;
  ~tk_prec() {
    tk_bt_destroy(bt_v);
    tk_bt_destroy(bt_p);
    tk_op_destroy(op_F0C);
    tk_op_destroy(op_Bt);
    tk_op_destroy(op_B);
  }
};

extern "C" int tk_prec_destroy(tk_prec* P) {
  { tk_ctx* _gc = P ? P->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  delete P;
  return TK_OK;
}

extern "C" const tk_op* tk_prec_operator(const tk_prec* P, int which) {
  if (!P) return nullptr;
  return which == 0 ? P->op_F0C : which == 1 ? P->op_Bt : which == 2 ? P->op_B : nullptr;
}

namespace {
// Host CSR (int32) for assembling the preconditioner's embedded spatial factors.
struct Csr {
  int64_t n = 0;
  std::vector<int32_t> rp{0}, cl;
  std::vector<double> v;
  void end_row() { rp.push_back((int32_t)cl.size()); n++; }
};

// rows [r0, r1) of A (CSR) appended with column offset coff
void append_rows(Csr& out, const int32_t* rp, const int32_t* cl, const double* v, int64_t r0,
                 int64_t r1, int64_t coff) {
  for (int64_t r = r0; r < r1; r++) {
    for (int32_t e = rp[r]; e < rp[r + 1]; e++) {
      out.cl.push_back((int32_t)(cl[e] + coff));
      out.v.push_back(v[e]);
    }
    out.end_row();
  }
}
void empty_rows(Csr& out, int64_t k) {
  for (int64_t i = 0; i < k; i++) out.end_row();
}
}  // namespace

extern "C" int tk_prec_create_lsc(tk_ctx* ctx, tk_prec** out, int64_t n_xi, int64_t n_t,
                                  int64_t grid, const int32_t* F_rowptr, const int32_t* F_col,
                                  const double* F_val, const int32_t* B_rowptr,
                                  const int32_t* B_col, const double* B_val, double tau, double tol,
                                  double tol_in, int restart_in, int max_cycles_in) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out || n_xi < 1 || n_t < 1 || grid < 1 || !F_rowptr || !B_rowptr ||
      !(tau > 0.0) || !(tol >= 0.0) || !(tol_in >= 0.0) || restart_in < 1 || max_cycles_in < 0)
    return TK_EARG;
  const int64_t nv = grid * grid, np = grid * grid, nx = 2 * nv + np;
  if (!csr_ok(nv, nv, F_rowptr, F_col) || !csr_ok(np, 2 * nv, B_rowptr, B_col)) {
    ctx->err = "tk_prec_create_lsc: malformed CSR";
    return TK_EARG;
  }
  std::unique_ptr<tk_prec> P(new tk_prec());
  P->ctx = ctx;
  P->n_v = nv;
  P->n_p = np;
  P->n_x = nx;
  P->n_xi = n_xi;
  P->n_t = n_t;
  P->tau = tau;
  P->tol = tol;
  P->tol_in = tol_in;
  P->restart_in = restart_in;
  P->max_cycles_in = max_cycles_in;
  TK_TRY(tk_bt_create(ctx, &P->bt_v, grid, grid, F_rowptr, F_col, F_val, 1.0 / tau));
  TK_TRY(tk_bt_create_gram(ctx, &P->bt_p, grid, grid, 2 * nv, B_rowptr, B_col, B_val));
  // embedded spatial factors on the stacked mode [u1; u2; p]
  Csr Iv, F0e, Bte, Be;
  for (int64_t i = 0; i < 2 * nv; i++) {
    Iv.cl.push_back((int32_t)i);
    Iv.v.push_back(1.0);
    Iv.end_row();
  }
  empty_rows(Iv, np);
  append_rows(F0e, F_rowptr, F_col, F_val, 0, nv, 0);
  append_rows(F0e, F_rowptr, F_col, F_val, 0, nv, nv);
  empty_rows(F0e, np);
  {  // B^T (2 nv x np) into the velocity rows, pressure columns (counting sort of B)
    std::vector<int32_t> cnt(2 * nv + 1, 0);
    for (int64_t e = 0; e < B_rowptr[np]; e++) cnt[B_col[e] + 1]++;
    for (int64_t c = 0; c < 2 * nv; c++) cnt[c + 1] += cnt[c];
    std::vector<int32_t> tcl(B_rowptr[np]);
    std::vector<double> tv(B_rowptr[np]);
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t r = 0; r < np; r++)
      for (int32_t e = B_rowptr[r]; e < B_rowptr[r + 1]; e++) {
        const int32_t p = pos[B_col[e]]++;
        tcl[p] = (int32_t)r;
        tv[p] = B_val[e];
      }
    append_rows(Bte, cnt.data(), tcl.data(), tv.data(), 0, 2 * nv, 2 * nv);
    empty_rows(Bte, np);
  }
  empty_rows(Be, 2 * nv);
  append_rows(Be, B_rowptr, B_col, B_val, 0, np, 0);
  // time factors: (I - C)/tau (lower bidiagonal, LAPACK band kl = 1, ku = 0) and I
  std::vector<double> band_imc(2 * n_t), band_i(n_t, 1.0);
  for (int64_t j = 0; j < n_t; j++) {
    band_imc[2 * j] = 1.0 / tau;
    band_imc[2 * j + 1] = j + 1 < n_t ? -1.0 / tau : 0.0;
  }
  std::vector<double> Ixi(n_xi * n_xi, 0.0);
  for (int64_t i = 0; i < n_xi; i++) Ixi[i * n_xi + i] = 1.0;
  auto mk = [&](int T, const Csr* const* K, const double* const* bands, const int* kl,
                tk_op** op) {
    const int32_t* rps[2];
    const int32_t* cls[2];
    const double* vs[2];
    const double* Gs[2];
    int ku[2] = {0, 0};
    for (int k = 0; k < T; k++) {
      rps[k] = K[k]->rp.data();
      cls[k] = K[k]->cl.data();
      vs[k] = K[k]->v.data();
      Gs[k] = Ixi.data();
    }
    return tk_op_create(ctx, op, T, nx, n_xi, n_t, rps, cls, vs, Gs, kl, ku, bands);
  };
  {
    const Csr* K[2] = {&Iv, &F0e};
    const double* bands[2] = {band_imc.data(), band_i.data()};
    const int kl[2] = {1, 0};
    TK_TRY(mk(2, K, bands, kl, &P->op_F0C));
  }
  {
    const Csr* K[1] = {&Bte};
    const double* bands[1] = {band_i.data()};
    const int kl[1] = {0};
    TK_TRY(mk(1, K, bands, kl, &P->op_Bt));
  }
  {
    const Csr* K[1] = {&Be};
    const double* bands[1] = {band_i.data()};
    const int kl[1] = {0};
    TK_TRY(mk(1, K, bands, kl, &P->op_B));
  }
  *out = P.release();
  return TK_OK;
}

namespace {

int make_like(tk_ctx* ctx, const tk_tt* x, OwnedPtr& y) {
  y = std::make_unique<OwnedTT>();
  return y->make(ctx, x->n_x, x->n_xi, x->n_t, x->r1, x->r2);
}

// x with its space core zeroed outside rows [lo, hi) (ranks unchanged)
int restrict_rows(tk_ctx* ctx, const tk_tt* x, int64_t lo, int64_t hi, OwnedPtr& y) {
  TK_TRY(make_like(ctx, x, y));
  const int64_t r = x->r1;
  TK_TRY(tk_zero(ctx, y->t.U1, 1, sizeof(double) * x->n_x * r, sizeof(double) * x->n_x * r));
  TK_TRY(tk_copy2d(ctx, 1, (hi - lo) * r, x->U1 + lo * r, (hi - lo) * r, y->t.U1 + lo * r,
                   (hi - lo) * r));
  const int64_t n2 = x->r1 * x->n_xi * x->r2, n3 = x->r2 * x->n_t;
  TK_TRY(tk_copy2d(ctx, 1, n2, x->U2, n2, y->t.U2, n2));
  TK_TRY(tk_copy2d(ctx, 1, n3, x->U3, n3, y->t.U3, n3));
  return TK_OK;
}

int apply_owned(tk_ctx* ctx, const tk_op* op, const tk_tt* x, OwnedPtr& y) {
  y = std::make_unique<OwnedTT>();
  TK_TRY(y->make(ctx, x->n_x, x->n_xi, x->n_t, op->T * x->r1, op->T * x->r2));
  return tk_apply_op(ctx, op, x, &y->t);
}

int axpby_round(tk_ctx* ctx, double a, const tk_tt* x, double b, const tk_tt* y, double tol,
                OwnedPtr& z) {
  z = std::make_unique<OwnedTT>();
  TK_TRY(z->make(ctx, x->n_x, x->n_xi, x->n_t, x->r1 + y->r1, x->r2 + y->r2));
  TK_TRY(tk_axpby_host(ctx, a, x, b, y, &z->t));
  return tk_round_now(ctx, &z->t, tol, 0, nullptr, nullptr, nullptr, nullptr);
}

// M^{-1} x (eq:11_prec): (I - C)^{-1} on the time core, K_s^{-1} on both velocity blocks.
int m_inv(tk_ctx* ctx, const tk_prec* P, const tk_tt* x, OwnedPtr& out) {
  OwnedPtr tc;
  TK_TRY(make_like(ctx, x, tc));
  {
    const int64_t n1 = x->n_x * x->r1, n2 = x->r1 * x->n_xi * x->r2;
    TK_TRY(tk_copy2d(ctx, 1, n1, x->U1, n1, tc->t.U1, n1));
    TK_TRY(tk_copy2d(ctx, 1, n2, x->U2, n2, tc->t.U2, n2));
  }
  time_cumsum_k<<<grid1(x->r2), 256, 0, ctx->stream>>>(x->r2, x->n_t, x->U3, tc->t.U3);
  TK_LAUNCH_CHECK(ctx);
  TK_TRY(make_like(ctx, x, out));
  return bt_solve_impl(ctx, P->bt_v, &tc->t, 0, 2, &out->t);
}

// S_LSC,0^{-1} v_p (eq:mean_lsc; steps 2-4 of R20 without the sign): vp must be zero outside
// the pressure rows.  B (F0 + C) B^T is applied as B, then F0 + C, then B^T (the same operator
// as the assembled product, up to rounding order).
int schur_inv(tk_ctx* ctx, const tk_prec* P, const tk_tt* vp, OwnedPtr& out) {
  const int64_t p0 = 2 * P->n_v;
  OwnedPtr q1, a, b, q2;
  TK_TRY(make_like(ctx, vp, q1));
  TK_TRY(bt_solve_impl(ctx, P->bt_p, vp, p0, 1, &q1->t));    // (B B^T)^{-1}
  TK_TRY(apply_owned(ctx, P->op_Bt, &q1->t, a));             // B^T
  TK_TRY(apply_owned(ctx, P->op_F0C, &a->t, b));             // F0 + C
  TK_TRY(tk_apply_round_owned(ctx, P->op_B, &b->t, q2, P->tol));  // T(B ...)
  TK_TRY(make_like(ctx, &q2->t, out));
  return bt_solve_impl(ctx, P->bt_p, &q2->t, p0, 1, &out->t);  // (B B^T)^{-1}
}

// P^{-1} v: steps 1-7 of DESIGN.md R20 (eq:prec block back substitution).
int lsc_apply(tk_ctx* ctx, const tk_prec* P, const tk_tt* v, OwnedPtr& out) {
  const int64_t nv2 = 2 * P->n_v;
  OwnedPtr vp, ph, vu, btp, w, uh;
  TK_TRY(restrict_rows(ctx, v, nv2, P->n_x, vp));            // 1
  TK_TRY(schur_inv(ctx, P, &vp->t, ph));                      // 2-4
  {
    DevBuf m1;
    TK_TRY(m1.get(ctx, 1));
    TK_TRY(tk_set_scalar(ctx, m1.p, -1.0));
    TK_TRY(tk_scale(ctx, &ph->t, m1.p, 0));                   // p^ = -S^{-1} v_p
  }
  TK_TRY(restrict_rows(ctx, v, 0, nv2, vu));
  TK_TRY(apply_owned(ctx, P->op_Bt, &ph->t, btp));
  TK_TRY(axpby_round(ctx, 1.0, &vu->t, -1.0, &btp->t, P->tol, w));  // 5
  {                                                           // 6: inner (F0 + C) solve
    TkPrecFn mfn = [ctx, P](const tk_tt* x, OwnedPtr& o) { return m_inv(ctx, P, x, o); };
    std::vector<double> expl;
    TK_TRY(tk_gmres_solve_core(ctx, P->op_F0C, &w->t, P->restart_in, P->max_cycles_in, P->tol,
                               P->tol_in, P->tol, &mfn, uh, expl, nullptr, nullptr));
    if (!uh) {
      uh = std::make_unique<OwnedTT>();
      TK_TRY(uh->make(ctx, P->n_x, P->n_xi, P->n_t, 1, 1));
      TK_TRY(set_zero_tt(ctx, &uh->t));
    }
  }
  return axpby_round(ctx, 1.0, &uh->t, 1.0, &ph->t, P->tol, out);  // 7
}

int prec_part(tk_ctx* ctx, const tk_prec* P, int part, const tk_tt* v, OwnedPtr& out) {
  if (v->n_x != P->n_x || v->n_xi != P->n_xi || v->n_t != P->n_t) {
    ctx->err = "tk_prec_apply: mode sizes differ from the preconditioner's";
    return TK_ESHAPE;
  }
  TagScope tag(ctx, "prec");
  if (part == 0) return lsc_apply(ctx, P, v, out);
  if (part == 1) return m_inv(ctx, P, v, out);
  if (part == 2) {
    OwnedPtr vp;
    TK_TRY(restrict_rows(ctx, v, 2 * P->n_v, P->n_x, vp));
    return schur_inv(ctx, P, &vp->t, out);
  }
  ctx->err = "tk_prec_apply: part must be 0, 1 or 2";
  return TK_EARG;
}

}  // namespace

TkPrecFn tk_prec_fn(tk_ctx* ctx, const tk_prec* P, int part) {
  return [ctx, P, part](const tk_tt* v, OwnedPtr& out) { return prec_part(ctx, P, part, v, out); };
}

extern "C" int tk_prec_apply(tk_ctx* ctx, const tk_prec* P, int part, const tk_tt* v,
                             tk_tt* out) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !P) return TK_EARG;
  TK_TRY(check_tt_basic(ctx, v));
  TK_TRY(check_tt_basic(ctx, out));
  OwnedPtr o;
  TK_TRY(prec_part(ctx, P, part, v, o));
  if (out->n_x != o->t.n_x || out->n_xi != o->t.n_xi || out->n_t != o->t.n_t) {
    ctx->err = "tk_prec_apply: output mode sizes";
    return TK_ESHAPE;
  }
  if (o->t.r1 > out->cap1 || o->t.r2 > out->cap2) {
    ctx->err = "tk_prec_apply: result ranks exceed the output capacity";
    return TK_ECAP;
  }
  out->r1 = o->t.r1;
  out->r2 = o->t.r2;
  TK_TRY(tk_copy2d(ctx, out->n_x, out->r1, o->t.U1, out->r1, out->U1, out->r1));
  TK_TRY(tk_copy2d(ctx, out->r1 * out->n_xi, out->r2, o->t.U2, out->r2, out->U2, out->r2));
  TK_TRY(tk_copy2d(ctx, out->r2, out->n_t, o->t.U3, out->n_t, out->U3, out->n_t));
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_prec_k() {}
const void* tk_anchor_prec() { return (const void*)tk_anchor_prec_k; }
