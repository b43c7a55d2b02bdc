// Internal declarations of libttk (B200 / sm_100a, fp64).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ttk.h"

// One profiled kernel (or kernel group): CUDA events on the context stream around it, with
// the algorithmic flop / byte counts of that launch.
struct ProfRec {
  const char* cat;
  double flops, bytes;
  cudaEvent_t a, b;
};

struct tk_async;

struct tk_ctx {
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  int num_sms = 148;
  int device = 0;
  // pinned host scratch for the few device->host reads (ranks, scalars)
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* pinned_dev = nullptr;  // device alias of `pinned` (mapped): small reads are kernel stores

  // profiling (tk_ctx_profile): per-launch event pairs, tagged by the current phase
  bool prof = false;
  bool prof_timeline = false;  // tk_ctx_profile(ctx, 3): dump start offsets too
  int prof_level = 2;  // 1: only launches with >= 1e8 algorithmic flops or bytes; 2: all
  const char* tag = "misc";
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // scratch accounting (tk_alloc / tk_free) and the pool reservation made from it
  std::unordered_map<void*, size_t> live;
  size_t live_bytes = 0, high_bytes = 0, reserved_for = 0;
  // side streams for work that overlaps the latency-bound critical path (Householder pass 1),
  // forked from / joined to `stream` with events; created on first use
  cudaStream_t aux[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> fork_ev;
  // one more side stream for independent big work (the apply's SpMM while the small cores are
  // swept, the bond-1 reconstruction while bond 2 runs): side_ev[0] forks, side_ev[1] joins
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
  // the rounding's latency-bound critical path runs on an internal highest-priority stream
  // (forked from / joined back to the caller's stream per call), so the block scheduler hands
  // SMs to it before the side stream's big kernels (which cannot be preempted)
  cudaStream_t crit = nullptr;
  cudaEvent_t crit_ev[2] = {nullptr, nullptr};
  // async mode (tk_ctx_set_async, async.cu): the worker that runs queued roundings
  tk_async* async = nullptr;
  // operand feed of the big DMMA GEMMs: 1 = TMA tensor tiles (k_gemm_tma.cu, default),
  // 0 = cp.async (k_gemm.cu); tk_ctx_set_gemm_feed
  int gemm_tma = 1;
  // schedule of the block-Jacobi eigensolver: 1 = dataflow (pair CTAs and tile CTAs one round
  // apart, no grid barriers; default), 0 = grid barriers (k_jacobi.cu); tk_ctx_set_jacobi_schedule
  int jacobi_flow = 1;
  // copy-window gate (tk_ctx_gate_stream, async.cu): every public rounding gets a sequence
  // number (round_seq, caller thread) and publishes it to gate_flag (device) when it reaches its
  // DMMA-bound phase, at its end at the latest; a gated user stream waits for the number of the
  // most recently SUBMITTED rounding.  gate_job: the number the running rounding still has to
  // publish (0: none).
  uint32_t* gate_flag = nullptr;
  uint32_t round_seq = 0, gate_job = 0;
};
// Copy-window gate: claim (caller thread, when a rounding is submitted), open (on the stream the
// rounding runs on; idempotent), destroy.
uint32_t tk_gate_claim(tk_ctx* ctx);
void tk_gate_open(tk_ctx* ctx);
void tk_gate_destroy(tk_ctx* ctx);
struct GateGuard {  // opens the gate on every exit path of a rounding
  tk_ctx* c;
  GateGuard(tk_ctx* ctx, uint32_t job) : c(ctx) { c->gate_job = job; }
  ~GateGuard() { tk_gate_open(c); }
};
// Async mode (async.cu).  drain: wait until the queued jobs ran (returns their first error);
// submit: queue body() for the worker, ordered after (and gating) the caller's stream.
int tk_async_drain(tk_ctx* ctx);
int tk_async_submit(tk_ctx* ctx, std::function<int()> body);
bool tk_async_on_worker(const tk_ctx* ctx);
void tk_async_destroy(tk_ctx* ctx);
// First statement of every entry point that reads ranks or enqueues work: wait for the queued
// asynchronous roundings (a no-op on the worker thread and in synchronous mode).
#define TK_ASYNC_GUARD(c)                         \
  do {                                             \
    if ((c) && (c)->async) {                       \
      int _g = tk_async_drain(c);                  \
      if (_g != TK_OK) return _g;                  \
    }                                              \
  } while (0)
// The synchronous rounding entry points (what tk_round / tk_apply_round run, on the calling
// thread or on the async worker).  Library-internal callers use these.
int tk_round_now(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
                 double* sigma2_out, double* discarded_out, double* norm_out);
int tk_apply_round_now(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y, double tol,
                       int64_t rmax, double* sigma1_out, double* sigma2_out,
                       double* discarded_out, double* norm_out);
// Scoped move of a whole library call onto ctx->crit (fork from the caller's stream on entry,
// join back on exit).
struct CritScope {
  tk_ctx* c;
  cudaStream_t user = nullptr;
  bool on = false;
  explicit CritScope(tk_ctx* ctx);
  ~CritScope();
};
// Fork: work issued on ctx->side after this call runs after everything issued so far on
// ctx->stream.  Join: work issued on ctx->stream after this call runs after everything issued
// so far on ctx->side.
int tk_side_fork(tk_ctx* ctx);
int tk_side_join(tk_ctx* ctx);
// Joins the side stream on scope exit (also on early error returns) when armed.
struct SideJoin {
  tk_ctx* c;
  bool armed;
  SideJoin(tk_ctx* ctx, bool a) : c(ctx), armed(a) {}
  ~SideJoin() {
    if (armed) tk_side_join(c);
  }
};
// Scoped redirection of the context's launches to the side stream.
struct OnSide {
  tk_ctx* c;
  cudaStream_t old;
  explicit OnSide(tk_ctx* ctx) : c(ctx), old(ctx->stream) { ctx->stream = ctx->side; }
  ~OnSide() { c->stream = old; }
};
// Lazily created side streams and a pool of at least n sync events (timing disabled).
int tk_aux_streams(tk_ctx* ctx, size_t n_events);

// Scoped phase tag for profiling records.
struct TagScope {
  tk_ctx* c;
  const char* old;
  TagScope(tk_ctx* ctx, const char* t) : c(ctx), old(ctx->tag) { ctx->tag = t; }
  ~TagScope() { c->tag = old; }
};

// Open / close a profiling record on the context stream (no-ops unless ctx->prof).
int tk_prof_begin(tk_ctx* ctx, const char* cat, double flops, double bytes);
void tk_prof_end(tk_ctx* ctx, int id);

// One launch of the column-merged SpMM: merged records over groups [g0, g0 + ng) of the op and
// the terms those groups produce.
struct SpmmChunk {
  int g0 = 0, ng = 0;          // groups of this chunk
  int nterm = 0;               // terms written (full output)
  bool ident = false;          // the chunk's groups are terms k0 .. k0+ng-1 with coefficient 1
  int k0 = 0;                  // (ident) first term
  bool owns = true;            // false: the device arrays belong to another chunk
  int64_t* recptr = nullptr;   // n_x + 1 (device): record i at rec + recptr[i]
  int64_t* rec = nullptr;      // [row | gn << 32][gn words col | mask << 32][values]
  int* tk = nullptr;           // nterm (device): term index, sorted by group
  int* tg = nullptr;           // ng + 1 (device): group g's terms are tk[tg[g] .. tg[g+1])
  double* tc = nullptr;        // nterm (device): coefficient
  std::vector<int> h_tk, h_goff;  // host copies (tk_op_concat)
  std::vector<double> h_tc;
};

struct tk_op {
  tk_ctx* ctx = nullptr;
  int T = 0;
  int64_t n_x = 0, n_xi = 0, n_t = 0;
  // device copies
  int32_t* rowptr = nullptr;   // T * (n_x + 1), each term's rowptr offset into the global col/val
  int32_t* col = nullptr;      // sum nnz
  double* val = nullptr;       // sum nnz
  int64_t* nnz_off = nullptr;  // T+1 (device), prefix offsets of each term's nnz
  double* G = nullptr;         // T * n_xi * n_xi
  int* band_kl = nullptr;      // T
  int* band_ku = nullptr;      // T
  int64_t* band_off = nullptr; // T+1 prefix offsets into band
  double* band = nullptr;      // concatenated LAPACK band arrays
  // column-merged copy of the spatial factors (k_apply.cu spmm_merged_k), in chunks of <= 16
  // spatial GROUPS (terms whose K_k is bitwise proportional to a representative share a
  // group; K_k = coef[k] K_group(k)).  Empty when a merged row would exceed 32 distinct columns
  // (then only the per-term kernel runs).
  std::vector<SpmmChunk> chunks;
  // the same over the group REPRESENTATIVES only, for the group-space output Y1' = [K_g U1]_g
  // of tk_op_group_space (identity over groups); empty when nothing groups
  std::vector<SpmmChunk> gchunks;
  bool spmm_perterm = false;   // tk_op_set_spmm_kernel(op, 1): use the per-term kernel
  int n_groups = 0;            // number of groups (== T when nothing groups)
  bool group_space = false;    // opt-in: the fused apply+round stores Y1 as Y1' = [K_g U1]_g
  int* d_group = nullptr;      // T (device): group of term k
  double* d_coef = nullptr;    // T (device)
  std::vector<int64_t> h_nnz;  // host copy of per-term nnz
  int max_kl = 0, max_ku = 0;
};

void tk_free_chunks(std::vector<SpmmChunk>& cs);
int tk_upload_terms(tk_ctx* ctx, SpmmChunk& c, const std::vector<int>& tk,
                    const std::vector<int>& tg, const std::vector<double>& tc);
int tk_upload_chunk(tk_ctx* ctx, SpmmChunk& c, const std::vector<int64_t>& recptr,
                    const std::vector<int64_t>& rec, const std::vector<int>& tk,
                    const std::vector<int>& tg, const std::vector<double>& tc);

// ----------------------------------------------------------------------------- errors
#define TK_CUDA_TRY(ctx, call)                                                      \
  do {                                                                              \
    cudaError_t _e = (call);                                                        \
    if (_e != cudaSuccess) {                                                        \
      (ctx)->err = std::string(#call) + ": " + cudaGetErrorString(_e);              \
      return TK_ECUDA;                                                              \
    }                                                                               \
  } while (0)

#define TK_LAUNCH_CHECK(ctx)                                                        \
  do {                                                                              \
    (ctx)->launches++;                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess) {                                                        \
      (ctx)->err = std::string("kernel launch: ") + cudaGetErrorString(_e);         \
      return TK_ECUDA;                                                              \
    }                                                                               \
  } while (0)

#define TK_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != TK_OK) return _s;   \
  } while (0)

// ----------------------------------------------------------------------------- memory
int tk_alloc(tk_ctx* ctx, void** p, size_t bytes);  // stream-ordered (cudaMallocAsync)
void tk_free(tk_ctx* ctx, void* p);                 // stream-ordered (cudaFreeAsync)

// RAII scratch buffer on the context stream.
struct DevBuf {
  tk_ctx* ctx = nullptr;
  double* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  int get(tk_ctx* c, size_t n_doubles) {
    release();
    ctx = c;
    return tk_alloc(c, (void**)&p, (n_doubles ? n_doubles : 1) * sizeof(double));
  }
  void release() {
    if (p) tk_free(ctx, p);
    p = nullptr;
  }
};


// A TT whose buffers are owned by the library (stream-ordered pool).
struct OwnedTT {
  tk_tt t{};
  DevBuf b1, b2, b3;
  int make(tk_ctx* ctx, int64_t n_x, int64_t n_xi, int64_t n_t, int64_t c1, int64_t c2) {
    t.n_x = n_x;
    t.n_xi = n_xi;
    t.n_t = n_t;
    t.cap1 = c1;
    t.cap2 = c2;
    t.r1 = c1;
    t.r2 = c2;
    TK_TRY(b1.get(ctx, n_x * c1));
    TK_TRY(b2.get(ctx, c1 * n_xi * c2));
    TK_TRY(b3.get(ctx, c2 * n_t));
    t.U1 = b1.p;
    t.U2 = b2.p;
    t.U3 = b3.p;
    return TK_OK;
  }
};
using OwnedPtr = std::unique_ptr<OwnedTT>;

int tk_copy2d(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
              double* dst, int64_t ldd);
inline int clone_tt(tk_ctx* ctx, const tk_tt* src, OwnedTT& dst) {
  TK_TRY(dst.make(ctx, src->n_x, src->n_xi, src->n_t, src->r1, src->r2));
  const int64_t n1 = src->n_x * src->r1, n2 = src->r1 * src->n_xi * src->r2,
                n3 = src->r2 * src->n_t;
  TK_TRY(tk_copy2d(ctx, 1, n1, src->U1, n1, dst.t.U1, n1));  // kernels, not the copy engines
  TK_TRY(tk_copy2d(ctx, 1, n2, src->U2, n2, dst.t.U2, n2));
  return tk_copy2d(ctx, 1, n3, src->U3, n3, dst.t.U3, n3);
}

// A right preconditioner v -> P^{-1} v (Alg. 3 line 4) as the GMRES drivers see it: writes a
// new library-owned TT.
using TkPrecFn = std::function<int(const tk_tt* v, OwnedPtr& out)>;
// The restarted low-rank GMRES core (tk_gmres_solve / tk_gmres_solve_p and the inner solve of
// the LSC preconditioner): flexible when prec != nullptr.  z_out is null when b rounds to zero
// or max_cycles == 0.  explicit_out gets ||s_0||, then ||s|| per cycle; ls_out (nullable) per
// cycle the least-squares history (restart + 1 entries, zero padded); steps_out per cycle.
int tk_gmres_solve_core(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int restart,
                        int max_cycles, double tol, double tol_gmres, double eps_soln,
                        const TkPrecFn* prec, OwnedPtr& z_out, std::vector<double>& explicit_out,
                        std::vector<double>* ls_out, std::vector<int>* steps_out);
TkPrecFn tk_prec_fn(tk_ctx* ctx, const tk_prec* P, int part);
int tk_apply_round_owned(tk_ctx* ctx, const tk_op* op, const tk_tt* x, OwnedPtr& y, double tol);
int set_zero_tt(tk_ctx* ctx, tk_tt* x);
int tk_sync_read(tk_ctx* ctx, void* host, const void* dev, size_t bytes);
// Small device -> host read on `stream` (synchronises it): a one-CTA kernel stores the bytes into
// the context's mapped pinned buffer, so the read never queues behind bulk DMA copies that share
// the device-to-host copy engine (a concurrent 1 GB D2H delayed every rank decision).
int tk_read_host(tk_ctx* ctx, cudaStream_t stream, void* host, const void* dev, size_t bytes);

// ----------------------------------------------------------------------------- kernels (host wrappers)
// Row-major fp64 GEMM on DMMA (mma.sync m8n8k4 f64):
//   C[M x N] (ldc) = alpha * op(A) * op(B) + beta * C
//   transA: A is stored K x M (lda) and op(A) = A^T; else A is M x K.
//   transB: B is stored N x K (ldb) and op(B) = B^T; else B is K x N.
//   sym: M == N and the product is symmetric (a Gram); only the upper triangle of tiles is
//        computed and mirrored.  Split-K with a deterministic reduction is chosen internally.
//   triu_b: op(B) is upper triangular (K x N, zero below the diagonal): each tile column skips
//        the zero K range.
//   skip (nullable, device int): the launch is a no-op when *skip != 0 (read by every CTA).
int tk_dgemm(tk_ctx* ctx, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
             double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
             double beta, double* C, int64_t ldc, bool sym = false, bool triu_b = false,
             const int* skip = nullptr);

// TMA-fed variant of the 64 x 64 DMMA kernel (k_gemm_tma.cu); tk_dgemm picks it for eligible
// heavy products (beta == 0, no triangular-B mode) when ctx->gemm_tma is set.
bool tk_dgemm_tma_eligible(bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                           const double* A, int64_t lda, const double* B, int64_t ldb);
int tk_dgemm_tma_launch(tk_ctx* ctx, bool transA, bool transB, int64_t M, int64_t N, int64_t K,
                        double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                        double* C, int64_t ldc, int64_t kchunk, int splits, int sym,
                        double* partial, const int* skip, int bn = 64);

// Symmetric eigen-decomposition by parallel cyclic two-sided Jacobi.
//   A: n x n symmetric (device, row-major, ld = n), destroyed.
//   lam: n eigenvalues sorted DESCENDING; V: n x n eigenvectors (columns), row-major.
//   A rotation on (p,q) is skipped when |a_pq| <= max(abs_tol, rel_tol*sqrt(|a_pp a_qq|)).
//   lskip_dev (nullable device double[2]): rotations between two indices whose diagonal
//   entries are both <= the skip threshold are skipped (cluster skip of the bond SVDs, see
//   k_jacobi.cu).  In: [0] static threshold.  With rs_tol > 0 the threshold is also raised
//   each sweep to the (r + 32)-th largest diagonal (r = rank rule with rs_tol, rs_rmax).
//   Out: [0] effective threshold, [1] bound on the unresolved block's largest eigenvalue.
//   V0 (nullable, mv x n row-major): the rotations are accumulated onto V0 instead of the
//   identity, and V (mv x n) returns V0 J with columns permuted like lam.
//   stop_rel (> 0): stop after a sweep whose largest rotated relative coupling is <= stop_rel
//   (default 1e-10).
int tk_jacobi_eig(tk_ctx* ctx, int n, double* A, double* lam, double* V, double abs_tol_scale,
                  double rel_tol, int max_sweeps, int* sweeps_out, double* lskip_dev = nullptr,
                  double rs_tol = 0.0, int64_t rs_rmax = 0,
                  const double* abs_floor_dev = nullptr, const double* V0 = nullptr,
                  int mv = 0,
                  double stop_rel = 0.0);
// Rounding-noise floor of a pass-2 Gram W^T W with W = fl(Y P) (K = inner dimension, k = its
// columns): tau = (4 eps)^2 K (trG_scale * trG[0]) ||P||_F^2 / k, written to out[0] (device).
// P == nullptr means an orthogonal P (||P||_F^2 = k).
int tk_noise_floor(tk_ctx* ctx, const double* trG_src, int64_t n_trG, double trG_scale,
                   const double* P, int64_t nP, int64_t K, int64_t k, double* out);
// lskip for the cluster skip: the diagonal mass of A below it is <= delta^2/4,
// delta^2 = tol^2 trace(A)/2.


// Q (n x n, row-major, exactly orthogonal) of the blocked Householder QR of A (n x n).
int tk_householder_q(tk_ctx* ctx, int n, const double* A, double* Q);
// Pivoted Cholesky H = P R^T R P^T of the n x n PSD H (k_chol.cu).  Ro (n x n, zeroed rows
// >= k): R in ORIGINAL column indexing, Ro[t, piv[c]] = R[t, c], so H ~ Ro^T Ro.  Stops when the
// largest remaining Schur diagonal <= max(tol_rel * max diag(H), *tol_abs_dev).  piv (n ints):
// pivot order (identity when !pivot).  state (2 + n ints, device): state[0] = k on completion.
// rem_out (nullable, device): trace of the Schur complement left when it stopped (0 if full rank).
int tk_pchol(tk_ctx* ctx, int n, const double* H, double tol_rel, const double* tol_abs_dev,
             double* Ro, int* piv, int* state, bool pivot = true, double* rem_out = nullptr);
int tk_pchol_max_n();
// X = R^{-1} for the k x k upper triangular R.
int tk_tri_inv(tk_ctx* ctx, int k, const double* R, int64_t ldr, double* X, int64_t ldx);
// out[t, c] = Ro[t, piv[c]]  (rows x k, ld k)
int tk_gather_cols(tk_ctx* ctx, int64_t rows, int k, const double* Ro, int64_t ldr, const int* piv,
                   double* out);
// S (n x cols) = 0 except S[piv[i], :] = X[i, :] for i < k
int tk_scatter_rows(tk_ctx* ctx, int64_t n, int k, int64_t cols, const double* X, const int* piv,
                    double* S);

// Apply kernels
int tk_launch_spmm_multi(tk_ctx* ctx, const tk_op* op, int r, const double* U1, double* Y1,
                         bool grouped = false);
// Lg[g r + a, j] = sum_{k : group[k] == g} coef[k] L[k r + a, j]   (L: T r x c, Lg: G r x c)
int tk_group_rows(tk_ctx* ctx, int T, int G, int64_t r, int64_t c, const int* group,
                  const double* coef, const double* L, double* Lg);
int tk_launch_stoch_apply(tk_ctx* ctx, const tk_op* op, int r1, int r2, const double* U2,
                          double* Y2, bool compact = false);
int tk_launch_time_apply(tk_ctx* ctx, const tk_op* op, int r2, const double* U3, double* Y3);

// small helpers (k_small.cu)
int tk_col_scale(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd, const double* f, int mode);  // mode 0: *f, 1: /f
int tk_row_scale(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd, const double* f, int mode);
int tk_copy2d(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
              double* dst, int64_t ldd);
int tk_fill(tk_ctx* ctx, double* dst, int64_t n, double v);
// zero rows x cols_bytes bytes at dst with row stride ld_bytes (multiples of 4 bytes), by a kernel
int tk_zero(tk_ctx* ctx, void* dst, int64_t rows, int64_t cols_bytes, int64_t ld_bytes);
int tk_eye(tk_ctx* ctx, double* dst, int64_t n);
// Rank decision on device from eigenvalues lam (descending, n of them):
//   sigma = sqrt(max(lam,0)) written to sig; info[0] = r (rule), info[1] = k (numerical dim
//   sigma > kthr*sigma_0), dinfo[0] = ||sigma||, dinfo[1] = delta used, dinfo[2] = discarded.
//   If delta_in < 0, delta = tol * ||sigma|| / sqrt(2) else delta = delta_in (device).
//   info[2] = number of lam > *lskip_dev (n if lskip_dev is null).
int tk_rank_select(tk_ctx* ctx, int n, const double* lam, double* sig, double tol,
                   const double* delta_dev_in, int64_t rmax, double kthr, int* info,
                   double* dinfo, int rcap = 0);
int tk_axpby_cores(tk_ctx* ctx, const double* a_dev, const tk_tt* x, const double* b_dev,
                   const tk_tt* y, tk_tt* z);
int tk_scale_rows(tk_ctx* ctx, double* U3, int64_t n, const double* s_dev, int invert);
int tk_dot_final(tk_ctx* ctx, int64_t n, const double* a, const double* b, double* out,
                 int take_sqrt);
int tk_set_scalar(tk_ctx* ctx, double* dst, double v);
int tk_neg_scalar(tk_ctx* ctx, const double* src, double* dst);
int tk_transpose(tk_ctx* ctx, int64_t rows, int64_t cols, const double* src, int64_t lds,
                 double* dst, int64_t ldd);
int tk_symmetrize(tk_ctx* ctx, int64_t n, double* A);
// out[b][q][p][w] = in[b][p][q][w] (swap of the two middle indices, w contiguous).
int tk_swap_mid(tk_ctx* ctx, int64_t nb, int64_t np, int64_t nq, int64_t nw, const double* in,
                double* out);
// Euclidean norms of the columns of the rows x cols matrix A (ld lda) into out (device).
int tk_col_norms(tk_ctx* ctx, int64_t rows, int64_t cols, const double* A, int64_t lda,
                 double* out);
