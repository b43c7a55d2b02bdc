// NEXT-4: the inexact Picard iteration of PAPER.md Alg. 1 (:199-213) on the
// all-at-once stochastic Galerkin Navier-Stokes system, driven over the library's own calls:
// N(u) of eq:N_kron built on the device from the iterate (tk_op_convection), the system
// operator as a concatenation (tk_op_concat), the linear solves by the restarted (optionally
// preconditioned) low-rank GMRES with the inexact stopping rule eq:inexact_solve (:536-538).
// Readings: DESIGN.md R21.  Contract: include/ttk.h.
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "ttk_internal.h"

namespace {

struct OpDel {
  void operator()(tk_op* o) const { tk_op_destroy(o); }
};
using OpPtr = std::unique_ptr<tk_op, OpDel>;

// L(u) = stokes + N(T_eps_conv(z))  (stokes terms first)
int system_operator(tk_ctx* ctx, const tk_op* stokes, const tk_conv* conv, const tk_tt* z,
                    double eps_conv, OpPtr& L) {
  OwnedTT u;
  TK_TRY(clone_tt(ctx, z, u));
  TK_TRY(tk_round_now(ctx, &u.t, eps_conv, 0, nullptr, nullptr, nullptr, nullptr));
  tk_op* N = nullptr;
  TK_TRY(tk_op_convection(ctx, conv, &u.t, &N));
  OpPtr Np(N);
  const tk_op* parts[2] = {stokes, N};
  tk_op* out = nullptr;
  TK_TRY(tk_op_concat(ctx, 2, parts, &out));
  L.reset(out);
  return TK_OK;
}

// r = T_eps(f - L z), ||r|| on the host
int residual(tk_ctx* ctx, const tk_op* L, const tk_tt* f, const tk_tt* z, double eps,
             OwnedPtr& r, double* nrm) {
  OwnedTT lz;
  TK_TRY(lz.make(ctx, z->n_x, z->n_xi, z->n_t, L->T * z->r1, L->T * z->r2));
  TK_TRY(tk_apply_op(ctx, L, z, &lz.t));
  r = std::make_unique<OwnedTT>();
  TK_TRY(r->make(ctx, z->n_x, z->n_xi, z->n_t, f->r1 + lz.t.r1, f->r2 + lz.t.r2));
  TK_TRY(tk_axpby_host(ctx, 1.0, f, -1.0, &lz.t, &r->t));
  TK_TRY(tk_round_now(ctx, &r->t, eps, 0, nullptr, nullptr, nullptr, nullptr));
  DevBuf d;
  TK_TRY(d.get(ctx, 1));
  TK_TRY(tk_norm(ctx, &r->t, d.p));
  return tk_sync_read(ctx, nrm, d.p, sizeof(double));
}

int zero_owned(tk_ctx* ctx, int64_t n_x, int64_t n_xi, int64_t n_t, OwnedPtr& z) {
  z = std::make_unique<OwnedTT>();
  TK_TRY(z->make(ctx, n_x, n_xi, n_t, 1, 1));
  return set_zero_tt(ctx, &z->t);
}

}  // namespace

extern "C" int tk_picard(tk_ctx* ctx, const tk_op* stokes, const tk_conv* conv, const tk_prec* P,
                         const tk_tt* f, double tol_picard, int maxit, double tol_gmres,
                         double eps_gmres, double eps_conv, int restart, int max_cycles,
                         tk_tt* z_out, double* residuals_out, int* iterations,
                         int64_t* ranks_out) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !stokes || !conv || !f || !z_out || !residuals_out || !iterations || maxit < 0 ||
      restart < 1 || max_cycles < 1 || !(tol_picard >= 0.0) || !(tol_gmres >= 0.0) ||
      !(eps_gmres >= 0.0))
    return TK_EARG;
  if (!f->U1 || !f->U2 || !f->U3 || f->r1 < 1 || f->r2 < 1 || f->n_x != stokes->n_x ||
      f->n_xi != stokes->n_xi || f->n_t != stokes->n_t || z_out->n_x != stokes->n_x ||
      z_out->n_xi != stokes->n_xi || z_out->n_t != stokes->n_t) {
    ctx->err = "tk_picard: f / z mode sizes differ from the operator's";
    return TK_ESHAPE;
  }
  if (eps_conv < 0.0) eps_conv = eps_gmres;
  const int64_t n_x = f->n_x, n_xi = f->n_xi, n_t = f->n_t;
  TagScope tag(ctx, "picard");
  TkPrecFn fn;
  if (P) fn = tk_prec_fn(ctx, P, 0);
  const TkPrecFn* pf = P ? &fn : nullptr;
  double fnorm;
  {
    DevBuf d;
    TK_TRY(d.get(ctx, 1));
    TK_TRY(tk_norm(ctx, f, d.p));
    TK_TRY(tk_sync_read(ctx, &fnorm, d.p, sizeof(double)));
  }
  // line 1: the Stokes solve (N = 0), ||s|| <= tol_gmres ||f||
  OwnedPtr z;
  {
    std::vector<double> expl;
    TK_TRY(tk_gmres_solve_core(ctx, stokes, f, restart, max_cycles, eps_gmres, tol_gmres,
                               eps_gmres, pf, z, expl, nullptr, nullptr));
    if (!z) TK_TRY(zero_owned(ctx, n_x, n_xi, n_t, z));
  }
  OpPtr L;
  TK_TRY(system_operator(ctx, stokes, conv, &z->t, eps_conv, L));
  OwnedPtr r;
  double rn;
  TK_TRY(residual(ctx, L.get(), f, &z->t, eps_gmres, r, &rn));
  residuals_out[0] = rn;
  if (ranks_out) {
    ranks_out[0] = z->t.r1;
    ranks_out[1] = z->t.r2;
  }
  int i = 0;
  while (rn > tol_picard * fnorm && i < maxit) {  // line 2
    i++;
    OwnedPtr dz;
    std::vector<double> expl;
    TK_TRY(tk_gmres_solve_core(ctx, L.get(), &r->t, restart, max_cycles, eps_gmres, tol_gmres,
                               eps_gmres, pf, dz, expl, nullptr, nullptr));  // line 4
    if (dz) {  // line 5: z <- T(z + dz)
      auto z2 = std::make_unique<OwnedTT>();
      TK_TRY(z2->make(ctx, n_x, n_xi, n_t, z->t.r1 + dz->t.r1, z->t.r2 + dz->t.r2));
      TK_TRY(tk_axpby_host(ctx, 1.0, &z->t, 1.0, &dz->t, &z2->t));
      TK_TRY(tk_round_now(ctx, &z2->t, eps_gmres, 0, nullptr, nullptr, nullptr, nullptr));
      z = std::move(z2);
    }
    TK_TRY(system_operator(ctx, stokes, conv, &z->t, eps_conv, L));  // line 6
    TK_TRY(residual(ctx, L.get(), f, &z->t, eps_gmres, r, &rn));      // line 7
    residuals_out[i] = rn;
    if (ranks_out) {
      ranks_out[2 * i] = z->t.r1;
      ranks_out[2 * i + 1] = z->t.r2;
    }
  }
  *iterations = i;
  if (z->t.r1 > z_out->cap1 || z->t.r2 > z_out->cap2) {
    ctx->err = "tk_picard: solution ranks exceed z's capacity";
    return TK_ECAP;
  }
  z_out->r1 = z->t.r1;
  z_out->r2 = z->t.r2;
  TK_TRY(tk_copy2d(ctx, n_x, z_out->r1, z->t.U1, z_out->r1, z_out->U1, z_out->r1));
  TK_TRY(tk_copy2d(ctx, z_out->r1 * n_xi, z_out->r2, z->t.U2, z_out->r2, z_out->U2, z_out->r2));
  TK_TRY(tk_copy2d(ctx, z_out->r2, n_t, z->t.U3, n_t, z_out->U3, n_t));
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TK_OK;
}
