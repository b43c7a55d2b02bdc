// NEXT-1: the TT-format convection operator N(u) of eq:N_kron, built ON THE
// DEVICE from a device-resident velocity TT, and the concatenation of
// operators (the Picard matrix F(u) = fixed terms + N(u)).
//
//   N(u) = sum_{a < r1, b < r2} diag(U3[b, :]) (x) (sum_l U2[a, l, b] H_l) (x) N(U1[:, a])
//
// in this repo's core order (R18; the paper's u^(1)(k, alpha_1) = U3[alpha_1, k],
// u^(2)(alpha_1, l, alpha_2) = U2[alpha_2, l, alpha_1], u^(3)(alpha_2, j) = U1[j, alpha_2]).
// The spatial factor of the a-th space-bond basis vector w = U1[:, a] is
//   N(w) = blkdiag over the d velocity components of  sum_c diag(w_c) D_c,
// w_c = U1[c n_v : (c+1) n_v, a] (the velocity parts; rows >= d n_v — the pressure — do not
// convect), D_c the n_v x n_v difference operators of the discretisation (tk_conv_create).
//
// Device layout of the built operator (T = r1 r2 terms, term k = a r2 + b):
//   * spatial GROUPS a < r1 (all b share N(U1[:, a])): merged-SpMM chunks of <= 16 groups whose
//     records are a host-built skeleton (pattern, masks) with the values filled by conv_fill_k;
//     no per-term CSR (the merged kernel computes each N(w_a) U1 product once and writes it to
//     the r2 output blocks of its terms);
//   * G_k = sum_l U2[a, l, b] H_l            (conv_g_k: one thread per output entry);
//   * T_k = diag(U3[b, :]) as a width-0 band  (conv_band_k).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <memory>
#include <vector>

#include "ttk_internal.h"

struct tk_conv {
  tk_ctx* ctx = nullptr;
  int64_t n_x = 0, n_xi = 0, n_t = 0, n_v = 0;
  int d = 0;
  // union pattern of the d difference operators (n_v rows, sorted columns) and, per operator,
  // its coefficient at every union entry (0 where it has none): host + device copies
  std::vector<int32_t> h_pp, h_pc;
  int32_t* pp = nullptr;
  int32_t* pc = nullptr;
  double* coef = nullptr;  // d x nnz
  double* H = nullptr;     // n_xi^3: H[l][r][s]
  int64_t nnz = 0;
  // record skeletons per chunk width ng (device recptr, rec, and the rec length)
  struct Skel {
    int64_t* recptr = nullptr;
    int64_t* rec = nullptr;
    int64_t len = 0;
  };
  std::map<int, Skel> skel;
};

namespace {

// values of the chunk's records: slot (j, g) of row i (i < d n_v, component s = i / n_v, node
// p = i % n_v) = sum_c U1[(c n_v + p) r1 + g0 + g] coef[c][pp[p] + j]
__global__ void conv_fill_k(int64_t n_rows, int64_t n_v, int d, int ng, int g0, int r1,
                            const int64_t* __restrict__ recptr, int64_t* __restrict__ rec,
                            const int32_t* __restrict__ pp, const double* __restrict__ coef,
                            int64_t nnz, const double* __restrict__ U1) {
  for (int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pos < n_rows;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = recptr[pos];
    const int64_t h = rec[base];
    const int64_t i = h & 0xffffffffLL;
    const int gn = (int)(h >> 32);
    if (gn == 0 || i >= d * n_v) continue;
    const int64_t p = i % n_v;
    const int64_t e0 = pp[p];
    double* vals = reinterpret_cast<double*>(rec + base + 1 + gn);
    for (int g = 0; g < ng; g++) {
      double w[8];
      for (int c = 0; c < d; c++) w[c] = U1[(c * n_v + p) * r1 + g0 + g];
      for (int j = 0; j < gn; j++) {
        double v = 0.0;
        for (int c = 0; c < d; c++) v = fma(w[c], coef[c * nnz + e0 + j], v);
        vals[j * ng + g] = v;
      }
    }
  }
}

// G[(a r2 + b), r, s] = sum_l U2[a, l, b] H[l, r, s]
__global__ void conv_g_k(int r1, int r2, int n_xi, const double* __restrict__ U2,
                         const double* __restrict__ H, double* __restrict__ G) {
  const int64_t nn = (int64_t)n_xi * n_xi;
  const int64_t total = (int64_t)r1 * r2 * nn;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / nn, rs = e % nn;
    const int a = (int)(k / r2), b = (int)(k % r2);
    double v = 0.0;
    for (int l = 0; l < n_xi; l++)
      v = fma(U2[((int64_t)a * n_xi + l) * r2 + b], H[(int64_t)l * nn + rs], v);
    G[e] = v;
  }
}

// band[(a r2 + b) n_t + t] = U3[b n_t + t]; band_off[k] = k n_t
__global__ void conv_band_k(int r1, int r2, int64_t n_t, const double* __restrict__ U3,
                            double* __restrict__ band, int64_t* __restrict__ band_off,
                            int* __restrict__ kl, int* __restrict__ ku, int* __restrict__ group,
                            double* __restrict__ gcoef) {
  const int64_t T = (int64_t)r1 * r2;
  const int64_t total = T * n_t;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / n_t, t = e % n_t;
    band[e] = U3[(k % r2) * n_t + t];
    if (t == 0) {
      kl[k] = 0;
      ku[k] = 0;
      group[k] = (int)(k / r2);
      gcoef[k] = 1.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t k = 0; k <= T; k++) band_off[k] = k * n_t;
}

int grid_of(tk_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms));
}

// The record skeleton of a chunk of ng groups: natural row order; row i < d n_v holds the
// union-pattern columns of node p = i % n_v shifted into its component block, every column
// with the full mask (all ng groups share the pattern), and gn * ng zero value slots.
int conv_skeleton(tk_conv* cv, int ng, tk_conv::Skel** out) {
  tk_ctx* ctx = cv->ctx;
  auto it = cv->skel.find(ng);
  if (it != cv->skel.end()) {
    *out = &it->second;
    return TK_OK;
  }
  const int64_t n_x = cv->n_x, n_v = cv->n_v;
  std::vector<int64_t> recptr(n_x + 1, 0), rec;
  rec.reserve(n_x + (size_t)cv->d * cv->nnz * (1 + ng));
  const int64_t mask = (int64_t)((ng >= 32) ? 0xffffffffu : ((1u << ng) - 1u));
  for (int64_t i = 0; i < n_x; i++) {
    if (i < cv->d * n_v) {
      const int64_t s = i / n_v, p = i % n_v;
      const int64_t e0 = cv->h_pp[p], gn = cv->h_pp[p + 1] - e0;
      rec.push_back(i | (gn << 32));
      for (int64_t j = 0; j < gn; j++)
        rec.push_back((int64_t)(uint32_t)(s * n_v + cv->h_pc[e0 + j]) | (mask << 32));
      rec.insert(rec.end(), (size_t)(gn * ng), 0LL);
    } else {
      rec.push_back(i);  // gn = 0: a zero row (pressure)
    }
    recptr[i + 1] = (int64_t)rec.size();
  }
  tk_conv::Skel sk;
  sk.len = (int64_t)rec.size();
  TK_CUDA_TRY(ctx, cudaMalloc((void**)&sk.recptr, sizeof(int64_t) * recptr.size()));
  TK_CUDA_TRY(ctx, cudaMalloc((void**)&sk.rec, sizeof(int64_t) * rec.size()));
  TK_CUDA_TRY(ctx, cudaMemcpy(sk.recptr, recptr.data(), sizeof(int64_t) * recptr.size(),
                              cudaMemcpyHostToDevice));
  TK_CUDA_TRY(ctx, cudaMemcpy(sk.rec, rec.data(), sizeof(int64_t) * rec.size(),
                              cudaMemcpyHostToDevice));
  *out = &(cv->skel[ng] = sk);
  return TK_OK;
}

}  // namespace

extern "C" int tk_conv_create(tk_ctx* ctx, tk_conv** out, int64_t n_x, int64_t n_xi,
                              int64_t n_t, int d, int64_t n_v, const int32_t* const* D_rowptr,
                              const int32_t* const* D_col, const double* const* D_val,
                              const double* H) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out || !D_rowptr || !D_col || !D_val || !H) return TK_EARG;
  if (d < 1 || d > 8 || n_v < 1 || n_xi < 1 || n_t < 1 || n_x < d * n_v || n_x >= INT32_MAX) {
    ctx->err = "tk_conv_create: need 1 <= d <= 8, n_v >= 1 and d n_v <= n_x < 2^31";
    return TK_EARG;
  }
  struct Del {
    void operator()(tk_conv* c) const { tk_conv_destroy(c); }
  };
  std::unique_ptr<tk_conv, Del> cv(new tk_conv());
  cv->ctx = ctx;
  cv->n_x = n_x;
  cv->n_xi = n_xi;
  cv->n_t = n_t;
  cv->n_v = n_v;
  cv->d = d;
  // union pattern and per-operator coefficients
  std::vector<std::vector<double>> cf(d);
  cv->h_pp.assign(n_v + 1, 0);
  std::vector<std::pair<int32_t, int>> ents;
  for (int c = 0; c < d; c++) {
    if (!D_rowptr[c] || D_rowptr[c][0] != 0) {
      ctx->err = "tk_conv_create: D rowptr must start at 0";
      return TK_EARG;
    }
    const int32_t nz = D_rowptr[c][n_v];
    for (int64_t i = 0; i < n_v; i++)
      if (D_rowptr[c][i + 1] < D_rowptr[c][i] || D_rowptr[c][i + 1] > nz) {
        ctx->err = "tk_conv_create: D rowptr must be non-decreasing and <= nnz";
        return TK_EARG;
      }
    for (int32_t e = 0; e < nz; e++)
      if (D_col[c][e] < 0 || D_col[c][e] >= n_v) {
        ctx->err = "tk_conv_create: D column index out of range";
        return TK_EARG;
      }
  }
  for (int64_t i = 0; i < n_v; i++) {
    ents.clear();
    for (int c = 0; c < d; c++)
      for (int32_t e = D_rowptr[c][i]; e < D_rowptr[c][i + 1]; e++) ents.push_back({D_col[c][e], c});
    std::vector<int32_t> cols;
    for (auto& e : ents) cols.push_back(e.first);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    if (cols.size() > 32) {
      ctx->err = "tk_conv_create: more than 32 distinct columns in a stencil row";
      return TK_EARG;
    }
    const size_t e0 = cv->h_pc.size();
    cv->h_pc.insert(cv->h_pc.end(), cols.begin(), cols.end());
    for (int c = 0; c < d; c++) {
      cf[c].resize(cv->h_pc.size(), 0.0);
      for (int32_t e = D_rowptr[c][i]; e < D_rowptr[c][i + 1]; e++) {
        const size_t j = std::lower_bound(cols.begin(), cols.end(), D_col[c][e]) - cols.begin();
        cf[c][e0 + j] += D_val[c][e];  // duplicates summed
      }
    }
    cv->h_pp[i + 1] = (int32_t)cv->h_pc.size();
  }
  cv->nnz = (int64_t)cv->h_pc.size();
  std::vector<double> coef((size_t)d * cv->nnz);
  for (int c = 0; c < d; c++) std::copy(cf[c].begin(), cf[c].end(), coef.begin() + c * cv->nnz);
  auto up = [&](void** p, const void* h, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(p, b ? b : 8));
    if (b) TK_CUDA_TRY(ctx, cudaMemcpy(*p, h, b, cudaMemcpyHostToDevice));
    return TK_OK;
  };
  TK_TRY(up((void**)&cv->pp, cv->h_pp.data(), sizeof(int32_t) * cv->h_pp.size()));
  TK_TRY(up((void**)&cv->pc, cv->h_pc.data(), sizeof(int32_t) * cv->h_pc.size()));
  TK_TRY(up((void**)&cv->coef, coef.data(), sizeof(double) * coef.size()));
  TK_TRY(up((void**)&cv->H, H, sizeof(double) * n_xi * n_xi * n_xi));
  *out = cv.release();
  return TK_OK;
}

extern "C" int tk_conv_destroy(tk_conv* cv) {
  { tk_ctx* _gc = cv ? cv->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  if (!cv) return TK_OK;
  cudaFree(cv->pp);
  cudaFree(cv->pc);
  cudaFree(cv->coef);
  cudaFree(cv->H);
  for (auto& kv : cv->skel) {
    cudaFree(kv.second.recptr);
    cudaFree(kv.second.rec);
  }
  delete cv;
  return TK_OK;
}

extern "C" int tk_op_convection(tk_ctx* ctx, const tk_conv* cvc, const tk_tt* u, tk_op** out) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !cvc || !u || !out || !u->U1 || !u->U2 || !u->U3) return TK_EARG;
  tk_conv* cv = const_cast<tk_conv*>(cvc);  // (the skeleton cache is mutable state)
  if (u->n_x != cv->n_x || u->n_xi != cv->n_xi || u->n_t != cv->n_t) {
    ctx->err = "tk_op_convection: velocity mode sizes differ from the convection setup's";
    return TK_ESHAPE;
  }
  if (u->r1 < 1 || u->r2 < 1 || u->r1 > u->cap1 || u->r2 > u->cap2) {
    ctx->err = "tk_op_convection: bad velocity ranks";
    return TK_EARG;
  }
  const int r1 = (int)u->r1, r2 = (int)u->r2;
  const int64_t T64 = (int64_t)r1 * r2;
  if (T64 > (1 << 20)) {
    ctx->err = "tk_op_convection: too many terms";
    return TK_EARG;
  }
  const int T = (int)T64;
  const int64_t n_x = cv->n_x, n_xi = cv->n_xi, n_t = cv->n_t;
  struct OpDel {
    void operator()(tk_op* o) const { tk_op_destroy(o); }
  };
  std::unique_ptr<tk_op, OpDel> op(new tk_op());
  op->ctx = ctx;
  op->T = T;
  op->n_x = n_x;
  op->n_xi = n_xi;
  op->n_t = n_t;
  op->n_groups = r1;
  op->h_nnz.assign(T, cv->d * cv->nnz);
  auto dmal = [&](void** p, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(p, b ? b : 8));
    return TK_OK;
  };
  TK_TRY(dmal((void**)&op->G, sizeof(double) * T * n_xi * n_xi));
  TK_TRY(dmal((void**)&op->band, sizeof(double) * T * n_t));
  TK_TRY(dmal((void**)&op->band_off, sizeof(int64_t) * (T + 1)));
  TK_TRY(dmal((void**)&op->band_kl, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->band_ku, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->d_group, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->d_coef, sizeof(double) * T));
  cudaStream_t st = ctx->stream;
  conv_g_k<<<grid_of(ctx, T64 * n_xi * n_xi), 256, 0, st>>>(r1, r2, (int)n_xi, u->U2, cv->H,
                                                            op->G);
  TK_LAUNCH_CHECK(ctx);
  conv_band_k<<<grid_of(ctx, T64 * n_t), 256, 0, st>>>(r1, r2, n_t, u->U3, op->band,
                                                       op->band_off, op->band_kl, op->band_ku,
                                                       op->d_group, op->d_coef);
  TK_LAUNCH_CHECK(ctx);
  // spatial chunks of <= 16 groups: skeleton copy + value fill
  for (int g0 = 0; g0 < r1; g0 += 16) {
    const int ng = std::min(16, r1 - g0);
    tk_conv::Skel* sk = nullptr;
    TK_TRY(conv_skeleton(cv, ng, &sk));
    SpmmChunk c;
    c.g0 = g0;
    c.ng = ng;
    c.ident = r2 == 1;  // then the chunk's groups are terms g0 .. g0+ng-1
    c.k0 = g0;
    std::vector<int> tk, tg;
    std::vector<double> tc;
    for (int a = g0; a < g0 + ng; a++)
      for (int b = 0; b < r2; b++) {
        tk.push_back(a * r2 + b);
        tg.push_back(a - g0);
        tc.push_back(1.0);
      }
    op->chunks.push_back(c);
    SpmmChunk& cc = op->chunks.back();
    TK_TRY(dmal((void**)&cc.recptr, sizeof(int64_t) * (n_x + 1)));
    TK_TRY(dmal((void**)&cc.rec, sizeof(int64_t) * sk->len));
    TK_TRY(tk_upload_terms(ctx, cc, tk, tg, tc));
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(cc.recptr, sk->recptr, sizeof(int64_t) * (n_x + 1),
                                     cudaMemcpyDeviceToDevice, st));
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(cc.rec, sk->rec, sizeof(int64_t) * sk->len,
                                     cudaMemcpyDeviceToDevice, st));
    conv_fill_k<<<grid_of(ctx, n_x), 256, 0, st>>>(n_x, cv->n_v, cv->d, ng, g0, r1, cc.recptr,
                                                   cc.rec, cv->pp, cv->coef, cv->nnz, u->U1);
    TK_LAUNCH_CHECK(ctx);
  }
  // group-space output: the same records, identity over the groups (aliases, not owned)
  for (const SpmmChunk& c : op->chunks) {
    SpmmChunk g = c;
    g.owns = false;
    g.ident = true;
    g.k0 = c.g0;
    op->gchunks.push_back(g);
  }
  *out = op.release();
  return TK_OK;
}

// Concatenation of operators with equal mode sizes: the terms of ops[0], then ops[1], ...
// (A = sum_i A_i).  Device arrays are copied; the inputs may be destroyed afterwards.
extern "C" int tk_op_concat(tk_ctx* ctx, int n, const tk_op* const* ops, tk_op** out) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out || n < 1 || !ops) return TK_EARG;
  for (int i = 0; i < n; i++)
    if (!ops[i] || ops[i]->n_x != ops[0]->n_x || ops[i]->n_xi != ops[0]->n_xi ||
        ops[i]->n_t != ops[0]->n_t) {
      ctx->err = "tk_op_concat: null operator or mode sizes differ";
      return ops[i] ? TK_ESHAPE : TK_EARG;
    }
  struct OpDel {
    void operator()(tk_op* o) const { tk_op_destroy(o); }
  };
  std::unique_ptr<tk_op, OpDel> op(new tk_op());
  op->ctx = ctx;
  op->n_x = ops[0]->n_x;
  op->n_xi = ops[0]->n_xi;
  op->n_t = ops[0]->n_t;
  int64_t band_tot = 0, nnz_tot = 0;
  bool all_csr = true, all_chunks = true;
  for (int i = 0; i < n; i++) {
    op->T += ops[i]->T;
    op->n_groups += ops[i]->n_groups;
    op->max_kl = std::max(op->max_kl, ops[i]->max_kl);
    op->max_ku = std::max(op->max_ku, ops[i]->max_ku);
    op->h_nnz.insert(op->h_nnz.end(), ops[i]->h_nnz.begin(), ops[i]->h_nnz.end());
    all_csr = all_csr && ops[i]->rowptr;
    all_chunks = all_chunks && !ops[i]->chunks.empty();
    std::vector<int64_t> bo(ops[i]->T + 1);
    TK_CUDA_TRY(ctx, cudaMemcpy(bo.data(), ops[i]->band_off, sizeof(int64_t) * bo.size(),
                                cudaMemcpyDeviceToHost));
    band_tot += bo.back();
    for (auto v : ops[i]->h_nnz) nnz_tot += v;
  }
  if (!all_chunks && !all_csr) {
    ctx->err = "tk_op_concat: the operators share no SpMM kernel (merged vs per-term only)";
    return TK_EARG;
  }
  const int T = op->T;
  const int64_t n_x = op->n_x, nn = op->n_xi * op->n_xi;
  auto dmal = [&](void** p, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(p, b ? b : 8));
    return TK_OK;
  };
  auto d2d = [&](void* dst, const void* src, size_t b) -> int {
    if (b) TK_CUDA_TRY(ctx, cudaMemcpy(dst, src, b, cudaMemcpyDeviceToDevice));
    return TK_OK;
  };
  TK_TRY(dmal((void**)&op->G, sizeof(double) * T * nn));
  TK_TRY(dmal((void**)&op->band, sizeof(double) * band_tot));
  TK_TRY(dmal((void**)&op->band_off, sizeof(int64_t) * (T + 1)));
  TK_TRY(dmal((void**)&op->band_kl, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->band_ku, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->d_group, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->d_coef, sizeof(double) * T));
  if (all_csr) {
    TK_TRY(dmal((void**)&op->rowptr, sizeof(int32_t) * T * (n_x + 1)));
    TK_TRY(dmal((void**)&op->col, sizeof(int32_t) * nnz_tot));
    TK_TRY(dmal((void**)&op->val, sizeof(double) * nnz_tot));
    TK_TRY(dmal((void**)&op->nnz_off, sizeof(int64_t) * (T + 1)));
  }
  std::vector<int64_t> band_off(T + 1, 0), nnz_off(T + 1, 0);
  std::vector<int> group(T);
  int k0 = 0, gofs = 0;
  int64_t boff = 0, noff = 0;
  for (int i = 0; i < n; i++) {
    const tk_op* s = ops[i];
    const int Ti = s->T;
    TK_TRY(d2d(op->G + (int64_t)k0 * nn, s->G, sizeof(double) * Ti * nn));
    TK_TRY(d2d(op->band_kl + k0, s->band_kl, sizeof(int) * Ti));
    TK_TRY(d2d(op->band_ku + k0, s->band_ku, sizeof(int) * Ti));
    TK_TRY(d2d(op->d_coef + k0, s->d_coef, sizeof(double) * Ti));
    std::vector<int64_t> bo(Ti + 1);
    TK_CUDA_TRY(ctx, cudaMemcpy(bo.data(), s->band_off, sizeof(int64_t) * bo.size(),
                                cudaMemcpyDeviceToHost));
    TK_TRY(d2d(op->band + boff, s->band, sizeof(double) * bo.back()));
    for (int k = 0; k < Ti; k++) band_off[k0 + k] = boff + bo[k];
    std::vector<int> gi(Ti);
    TK_CUDA_TRY(ctx, cudaMemcpy(gi.data(), s->d_group, sizeof(int) * Ti, cudaMemcpyDeviceToHost));
    for (int k = 0; k < Ti; k++) group[k0 + k] = gi[k] + gofs;
    if (all_csr) {
      std::vector<int64_t> no(Ti + 1);
      TK_CUDA_TRY(ctx, cudaMemcpy(no.data(), s->nnz_off, sizeof(int64_t) * no.size(),
                                  cudaMemcpyDeviceToHost));
      TK_TRY(d2d(op->rowptr + (int64_t)k0 * (n_x + 1), s->rowptr,
                 sizeof(int32_t) * Ti * (n_x + 1)));
      TK_TRY(d2d(op->col + noff, s->col, sizeof(int32_t) * no.back()));
      TK_TRY(d2d(op->val + noff, s->val, sizeof(double) * no.back()));
      for (int k = 0; k < Ti; k++) nnz_off[k0 + k] = noff + no[k];
      noff += no.back();
    }
    if (all_chunks) {
      // full output: the source's term list shifted by k0; group-space output: the source's
      // group chunks shifted by gofs (copies of the records)
      for (int pass = 0; pass < 2; pass++) {
        const std::vector<SpmmChunk>& src = pass == 0 ? s->chunks : s->gchunks;
        for (const SpmmChunk& sc : src) {
          std::vector<int> tk = sc.h_tk, tg(sc.nterm);
          std::vector<double> tc = sc.h_tc;
          for (int g = 0; g < sc.ng; g++)
            for (int t = sc.h_goff[g]; t < sc.h_goff[g + 1]; t++) tg[t] = g;
          for (auto& v : tk) v += k0;
          std::vector<int64_t> recptr(n_x + 1);
          TK_CUDA_TRY(ctx, cudaMemcpy(recptr.data(), sc.recptr, sizeof(int64_t) * (n_x + 1),
                                      cudaMemcpyDeviceToHost));
          std::vector<int64_t> rec(recptr.back());
          TK_CUDA_TRY(ctx, cudaMemcpy(rec.data(), sc.rec, sizeof(int64_t) * rec.size(),
                                      cudaMemcpyDeviceToHost));
          SpmmChunk c;
          c.g0 = sc.g0 + gofs;
          c.ng = sc.ng;
          c.ident = sc.ident;
          c.k0 = pass == 0 ? sc.k0 + k0 : c.g0;
          std::vector<SpmmChunk>& dst = pass == 0 ? op->chunks : op->gchunks;
          dst.push_back(c);
          TK_TRY(tk_upload_chunk(ctx, dst.back(), recptr, rec, tk, tg, tc));
        }
      }
    }
    k0 += Ti;
    gofs += s->n_groups;
    boff += bo.back();
  }
  band_off[T] = boff;
  nnz_off[T] = noff;
  TK_CUDA_TRY(ctx, cudaMemcpy(op->band_off, band_off.data(), sizeof(int64_t) * (T + 1),
                              cudaMemcpyHostToDevice));
  TK_CUDA_TRY(ctx, cudaMemcpy(op->d_group, group.data(), sizeof(int) * T, cudaMemcpyHostToDevice));
  if (all_csr)
    TK_CUDA_TRY(ctx, cudaMemcpy(op->nnz_off, nnz_off.data(), sizeof(int64_t) * (T + 1),
                                cudaMemcpyHostToDevice));
  op->spmm_perterm = !all_chunks;
  // group-space output only if every part has one (else groups == terms: no grouping)
  bool all_g = true;
  for (int i = 0; i < n; i++) all_g = all_g && (!ops[i]->gchunks.empty() || ops[i]->n_groups == ops[i]->T);
  if (!all_g || !all_chunks) {
    tk_free_chunks(op->gchunks);
    op->n_groups = T;
  }
  *out = op.release();
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_conv_k() {}
const void* tk_anchor_k_conv() { return (const void*)tk_anchor_k_conv_k; }
