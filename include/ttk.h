/*
 * ttk.h — C ABI of the B200 (sm_100a) tensor-train hot path of arXiv:1906.06785
 * ("Low-rank solvers for unsteady Navier–Stokes with stochastic viscosity").
 *
 * The path: apply the Kronecker-sum operator  A = sum_k T_k (x) G_k (x) K_k
 * (time (x) stochastic (x) space; PAPER.md:157 eq:F, :239-244 eq:Xz) to a 3-core tensor
 * train, TT-round the result back to low rank (Alg. 2 :259-273), and the
 * TT dot / axpby used by low-rank GMRES (Alg. 3).  One GPU, fp64.
 *
 * Conventions (R1):
 *   A TT is X(i_x,i_xi,i_t) = sum_{a,b} U1[i_x,a] U2[a,i_xi,b] U3[b,i_t].  vec(X) runs space
 *   fastest.  Paper cores z^(1), z^(2), z^(3) (time, stoch, space) map to
 *   U3^T, U2 with swapped bonds, U1^T.
 *   All core buffers are DEVICE pointers, float64, compact row-major with the CURRENT ranks:
 *     U1: n_x  x r1            element (i, a)    at U1[i*r1 + a]
 *     U2: r1 x n_xi x r2       element (a, i, b) at U2[(a*n_xi + i)*r2 + b]
 *     U3: r2 x n_t             element (b, t)    at U3[b*n_t + t]
 *   cap1/cap2 give the rank capacity the buffers were allocated for: U1 holds >= n_x*cap1
 *   doubles, U2 >= cap1*n_xi*cap2, U3 >= cap2*n_t.
 *
 * Ownership: the caller owns every tk_tt buffer (allocated with PyTorch in the binding).
 * The library owns the context (stream, stream-ordered memory pool for temporaries) and the
 * device copy of the operator descriptor.  Inputs are never modified except by tk_round,
 * which rounds in place (ranks never grow).
 *
 * Errors: every call returns TK_OK (0) or a negative code; tk_last_error(ctx) returns a
 * message.  No call falls back to the CPU.  Work is enqueued on the context stream.  By
 * default tk_round / tk_apply_round block the host until the ranks they choose are known (the
 * launches after a rank decision are sized on the host).  In async mode (tk_ctx_set_async)
 * they return at once: the rounding runs on a library worker thread, the context stream waits
 * for it in stream order, and the ranks are published into the caller's tk_tt by
 * tk_sync_ranks.  The GMRES / preconditioner / Picard drivers and the tk_*_host variants block.
 */
#ifndef TTK_H
#define TTK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TK_OK = 0,
  TK_ESHAPE = -1,    /* mode sizes disagree                        */
  TK_ECAP = -2,      /* output rank exceeds the capacity of the caller's buffers           */
  TK_EARG = -3,      /* invalid argument: tol < 0, T < 1, null pointer, rank < 1, ...      */
  TK_ENUMERIC = -4,  /* non-finite singular values / norms                                 */
  TK_ECUDA = -5      /* a CUDA runtime error (message in tk_last_error)                    */
};

typedef struct tk_ctx tk_ctx;
typedef struct tk_op tk_op;
typedef struct tk_conv tk_conv;

typedef struct {
  int64_t n_x, n_xi, n_t; /* mode sizes (space, stochastic, time)                          */
  int64_t r1, r2;         /* current TT ranks (space bond, time bond), >= 1                */
  int64_t cap1, cap2;     /* rank capacity of the buffers                                  */
  double *U1, *U2, *U3;   /* device pointers, layouts above                                */
} tk_tt;

/* Library version string. */
const char* tk_version(void);

/* Create a context bound to `cuda_stream` (a cudaStream_t; NULL = legacy default stream).
 * All work of the context is enqueued on that stream. */
int tk_ctx_create(tk_ctx** ctx, void* cuda_stream);
int tk_ctx_destroy(tk_ctx* ctx);
const char* tk_last_error(const tk_ctx* ctx);
/* Number of kernels this context has launched since creation (for the bench's
 * "gpu_launches"). */
int64_t tk_ctx_launch_count(const tk_ctx* ctx);
/* Profiling: enable != 0 clears the record list and starts recording CUDA events around
 * every kernel (tagged with its phase and its algorithmic flop and byte counts); 0 stops.
 * enable == 2 records only the heavy launches (>= 1e8 algorithmic flops or bytes): the event
 * pairs around the many small kernels of the latency-bound chain cost ~2 ms per c4 step.
 * enable == 3 records every launch and the dump adds a fifth field, the start offset (ms)
 * from the first record (timeline).
 * tk_ctx_profile_dump synchronises the stream and writes one line per record,
 * "<phase> <ms> <flops> <bytes>\n", into buf (truncated to len); returns the number of
 * records. */
int tk_ctx_profile(tk_ctx* ctx, int enable);
int tk_ctx_profile_dump(tk_ctx* ctx, char* buf, size_t len);

/* Asynchronous rounding.  on != 0: from now on tk_round and tk_apply_round
 * only validate their handles and return TK_OK at once; the rounding is queued to a worker
 * thread of the context that runs the queued roundings in order on a private stream, ordered
 * after everything enqueued so far on the context stream, and the context stream waits for it
 * (a device-side wait: later work on that stream runs after the rounding, without a host
 * synchronisation).  The caller's tk_tt structs (and the optional host outputs) are read and
 * written by the worker: they must stay valid, and their rank fields are undefined, until
 * tk_sync_ranks returns.  Every other entry point first waits for the queued roundings.  Errors
 * of a queued rounding are returned by tk_sync_ranks (or the next call).  Returns 1 if async
 * mode is on, 0 if the driver has no stream memory operations (the context stays synchronous
 * and correct), or a negative error.  on == 0 drains the queue and returns to synchronous mode.
 * tk_sync_ranks: block until every queued rounding has finished and published its ranks (x may
 * be NULL; all TTs are published).  A no-op in synchronous mode. */
int tk_ctx_set_async(tk_ctx* ctx, int on);
/* Copy-window gate for pipelined host <-> device transfers.  The latency-bound phases of a
 * rounding (thousands of short kernels) slow down when bulk PCIe copies run beside them, the
 * DMMA-bound phase in the middle (the big-core Gram pass) does not.  After this
 * call, work enqueued on `cuda_stream` (a cudaStream_t of the caller: its copy stream) waits —
 * on the device, without a host synchronisation — until the most recently SUBMITTED tk_round /
 * tk_apply_round of this context has reached that phase (at the latest: has finished, also
 * when it failed).  With the asynchronous boundary (tk_ctx_set_async) the rounding is still
 * queued or running when the call is made and the transfers of the neighbouring pipeline steps
 * land inside its window; in synchronous mode, or when no rounding was submitted yet, the
 * condition already holds and the stream is not delayed.  The gate only ever waits for work
 * that is already queued: no call order can leave the stream waiting forever.  Returns 1 if
 * the wait was enqueued, 0 if the driver has no stream memory operations (the stream is not
 * gated: transfers simply start at once), or a negative error.  The first call loads every
 * kernel of the library and synchronises the context once. */
int tk_ctx_gate_stream(tk_ctx* ctx, void* cuda_stream);
int tk_sync_ranks(tk_ctx* ctx, tk_tt* x);
/* Upper bound (bytes) of the library scratch of one tk_round on ranks (R1, R2), or one
 * tk_apply_round whose grown ranks are (R1, R2), with these mode sizes; the caller-owned cores
 * are not included.  tk_ctx_reserve pre-reserves that much of the stream-ordered pool
 * (synchronous); tk_ctx_scratch_high_water reports the measured peak (reset != 0 restarts it). */
size_t tk_round_workspace_bytes(int64_t n_x, int64_t n_xi, int64_t n_t, int64_t R1, int64_t R2);
int tk_ctx_reserve(tk_ctx* ctx, size_t bytes);
int64_t tk_ctx_scratch_high_water(tk_ctx* ctx, int reset);

/* The dense contraction of the path (north star: "Gram/TSQR on FP64 DMMA tensor cores fed via
 * TMA"; the Grams W = X^T Y of the rounding and of the TT dot):
 *   C (M x N, ldc) = alpha op(A) op(B) + beta C,  op(A) M x K, op(B) K x N, fp64, DEVICE
 * pointers, row-major: transA == 0: A is M x K (lda >= K); != 0: A is stored K x M (lda >= M);
 * transB == 0: B is K x N (ldb >= N); != 0: B is stored N x K (ldb >= K).  sym != 0 (needs
 * M == N, B^T A == A^T B): only the upper tiles are computed and mirrored (symmetric Gram).
 * Asynchronous on the context stream; split-K partial sums are reduced in a fixed order, so
 * results are bitwise reproducible run to run (per feed).  Errors: TK_EARG (null pointer,
 * sym with M != N, K == 0 with beta != 0), TK_ECUDA.
 * tk_ctx_set_gemm_feed: how the heavy products (>= 1e8 flops, beta == 0) get their operand
 * tiles: 1 = TMA tensor tiles (cp.async.bulk.tensor + mbarrier, 128B-swizzled shared memory;
 * default), 0 = cp.async.  Operands that are not 16-byte aligned or have an odd leading
 * dimension always take the cp.async kernel.  Both feeds compute the same sums in a different
 * (fixed) order. */
int tk_gemm(tk_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
            const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
            int64_t ldc, int sym);
int tk_ctx_set_gemm_feed(tk_ctx* ctx, int mode);
/* Schedule of the block-Jacobi eigensolver behind the bond SVDs (the truncated
 * SVDs of the rounding): 1 = dataflow (default: the CTAs that solve the 64 x 64 pair problems
 * and the CTAs that apply the tile updates run one round apart, ordered by counters in global
 * memory), 0 = two grid-wide barriers per round.  Same rotations, same products, same order:
 * results are bitwise identical.  Errors: TK_EARG. */
int tk_ctx_set_jacobi_schedule(tk_ctx* ctx, int mode);

/* Operator descriptor  A = sum_{k<T} T_k (x) G_k (x) K_k.
 *   K_k : n_x x n_x CSR, HOST arrays: rowptr[n_x+1] (int32), col[nnz_k] (int32, 0-based),
 *         val[nnz_k] (float64).
 *   G_k : n_xi x n_xi dense, HOST, row-major.
 *   T_k : n_t x n_t banded, HOST, LAPACK general band storage, column major with
 *         ldab = kl+ku+1: T[i][j] = band[j*ldab + ku + i - j] for j-ku <= i <= j+kl.
 * The descriptor is copied to the device; the host arrays may be freed afterwards.
 * Synchronous (setup, not on the hot path). */
int tk_op_create(tk_ctx* ctx, tk_op** op, int T, int64_t n_x, int64_t n_xi, int64_t n_t,
                 const int32_t* const* K_rowptr, const int32_t* const* K_col,
                 const double* const* K_val, const double* const* G, const int* T_kl,
                 const int* T_ku, const double* const* T_band);
int tk_op_destroy(tk_op* op);
int tk_op_terms(const tk_op* op);
/* Select the spatial SpMM kernel of row a1: kernel 0 = the column-merged multi-term sweep
 * (default; available when every row of the merged pattern has <= 32 distinct columns),
 * kernel 1 = the per-term CSR kernel.  Returns 1 if the merged kernel will run, 0 if the
 * per-term kernel will, TK_EARG on a bad argument.  Not thread-safe against concurrent
 * applies of the same operator. */
int tk_op_set_spmm_kernel(tk_op* op, int kernel);
/* Optional exact factor grouping of the space core (OFF by default — the literal
 * T r rank growth is the primary shape).  At tk_op_create the library groups terms whose K_k
 * has the same CSR structure as an earlier term's and is BITWISE proportional to it
 * (K_k = c K_j checked entry by entry in fp64, e.g. nu_l L with nu_l = nu_0 2^-l), so that
 * K_k U1 = c (K_j U1) exactly.  With enable != 0, tk_apply_round then stores the grown space
 * core in the factored form Y1 = Y1' E (Y1' = [K_g U1] over the G group representatives) and
 * runs bond 1 on Y1' with L2' = E L2 — the same operator, the same rounded result up to
 * rounding order, fewer flops.  tk_apply_op and tk_round are unaffected.  Returns G (== T when
 * nothing groups; enabling is then a no-op) or TK_EARG. */
int tk_op_group_space(tk_op* op, int enable);

/* Concatenation A = sum_i A_i of n >= 1 operators with equal mode sizes: the terms of
 * ops[0], then ops[1], ... (e.g. the Picard matrix F(u) + C = fixed terms + N(u),
 * PAPER.md:157-161).  Device arrays are copied (the inputs may be destroyed afterwards).
 * TK_ESHAPE if the mode sizes differ.  Synchronous (setup). */
int tk_op_concat(tk_ctx* ctx, int n, const tk_op* const* ops, tk_op** out);

/* NEXT-1: the TT-format convection operator of eq:N_kron, built on the
 * device from a device-resident velocity TT.
 *
 * tk_conv_create fixes the discretisation once: the spatial mode is [v_1; ...; v_d; rest]
 * with d velocity components of n_v dofs each (d n_v <= n_x; rows >= d n_v, e.g. the
 * pressure, do not convect), D_c (c < d) are the n_v x n_v difference operators of the
 * convective derivative (HOST CSR, int32, 0-based; every row of their union pattern has
 * <= 32 distinct columns), and H (HOST, n_xi^3 doubles, H[(l n_xi + r) n_xi + s] =
 * <psi_l psi_r psi_s>) the chaos triple products.  Copied to the device.
 *
 * tk_op_convection builds, for the velocity TT u (DEVICE cores, modes (n_x, n_xi, n_t)),
 *   N(u) = sum_{a < u.r1, b < u.r2} diag(U3[b, :]) (x) (sum_l U2[a, l, b] H_l) (x) N(U1[:, a])
 *   N(w) = blkdiag_{s < d}( sum_c diag(w_c) D_c ),  w_c = w[c n_v : (c+1) n_v]
 * (this repo's core order, R18): u.r1 u.r2 terms, term k = a u.r2 + b, the
 * kappa -> kappa^2 growth of PAPER.md:331.  Values are computed by kernels from u's device
 * cores (no host round trip of u); the result is an ordinary operator (tk_apply_op,
 * tk_apply_round, tk_op_concat, tk_op_destroy), whose SpMM computes each N(U1[:, a]) U1
 * product once and writes it to the u.r2 blocks of its terms.  It has no per-term CSR
 * (tk_op_set_spmm_kernel(op, 1) returns TK_EARG).  Asynchronous except for the allocations. */
int tk_conv_create(tk_ctx* ctx, tk_conv** conv, int64_t n_x, int64_t n_xi, int64_t n_t, int d,
                   int64_t n_v, const int32_t* const* D_rowptr, const int32_t* const* D_col,
                   const double* const* D_val, const double* H);
int tk_conv_destroy(tk_conv* conv);
int tk_op_convection(tk_ctx* ctx, const tk_conv* conv, const tk_tt* u, tk_op** op);

/* y = A x   (PAPER.md:239-244 eq:Xz).  Per term k: K_k U1, G_k x_2 U2,
 * U3 T_k^T; terms are concatenated: y ranks = (T*x.r1, T*x.r2), y.U1 = [K_0 U1 | ... ],
 * y.U2 block diagonal (zeros off the diagonal blocks), y.U3 = [U3 T_0^T; U3 T_1^T; ...].
 * y must have cap1 >= T*x.r1 and cap2 >= T*x.r2 (else TK_ECAP); on success y->r1, y->r2
 * are set.  Asynchronous. */
int tk_apply_op(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y);

/* In-place TT rounding T_eps: on return ||x_new - x||_F <= tol ||x||_F
 * unless rmax binds, with delta_1 = delta_2 = tol ||x||_F / sqrt(2) and the
 * rank rule "smallest r >= 1 whose discarded tail (sum_{j>r} s_j^2)^{1/2} <= delta", capped
 * at rmax when rmax > 0 (R2-R5).  Space bond first, then time bond (north-star
 * direction).  Output cores: U1 and reshape(U2, r1 n_xi, r2) have orthonormal columns and
 * ||U3||_F = ||x_new||_F.  The zero tensor canonicalises to ranks (1,1), zero cores.
 * sigma1_out / sigma2_out (nullable HOST arrays of length >= x->r1 and >= x->r2 on entry)
 * receive the singular values of the two bonds (descending; entries past the numerical
 * dimension are 0); discarded_out (nullable HOST, 2 doubles) the discarded tail norms;
 * norm_out (nullable HOST) ||x||_F of the input.  Blocks the host to read the chosen ranks,
 * except in async mode (tk_ctx_set_async).
 */
int tk_round(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
             double* sigma2_out, double* discarded_out, double* norm_out);

/* y = T_eps(A x): tk_apply_op followed by tk_round on y, fused: the block
 * diagonal middle core of A x is never written densely — its T diagonal blocks G_k x_2 U2 stay
 * in scratch and the right-to-left step U2 x_3 L3 runs block by block (T-fold fewer flops).
 * Same contract, outputs and results as the two calls in sequence; y needs cap1 >= T*x.r1,
 * cap2 >= T*x.r2 and holds the rounded TT on return (in async mode: after tk_sync_ranks).
 * Blocks the host except in async mode. */
int tk_apply_round(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y, double tol,
                   int64_t rmax, double* sigma1_out, double* sigma2_out, double* discarded_out,
                   double* norm_out);

/* <x, y>_F contracted core by core (Alg. 3 line 7):
 * W1 = X1^T Y1, W2 = sum_i X2(:,i,:)^T W1 Y2(:,i,:), <x,y> = sum(W2 .* (X3 Y3^T)).
 * out_dev: DEVICE pointer to one double.  Asynchronous. */
int tk_dot(tk_ctx* ctx, const tk_tt* x, const tk_tt* y, double* out_dev);
/* ||x||_F = sqrt(<x,x>) into a DEVICE double.  Asynchronous. */
int tk_norm(tk_ctx* ctx, const tk_tt* x, double* out_dev);

/* z = a x + b y by core concatenation: z.U1 = [x.U1 | y.U1],
 * z.U2 = blockdiag(x.U2, y.U2), z.U3 = [a x.U3; b y.U3].  z ranks = sums (TK_ECAP if they
 * exceed z's capacity).  a_dev / b_dev are DEVICE pointers to one double each (so GMRES
 * coefficients never leave the device); tk_axpby_host takes host scalars.  Asynchronous.
 * z must not alias x or y. */
int tk_axpby(tk_ctx* ctx, const double* a_dev, const tk_tt* x, const double* b_dev,
             const tk_tt* y, tk_tt* z);
int tk_axpby_host(tk_ctx* ctx, double a, const tk_tt* x, double b, const tk_tt* y, tk_tt* z);
/* x <- s x (scales U3); s_dev DEVICE double; if invert != 0 uses 1/s.  Asynchronous. */
int tk_scale(tk_ctx* ctx, tk_tt* x, const double* s_dev, int invert);

/* One cycle of low-rank GMRES, Alg. 3 with P = I, z_0 = 0 and the
 * c5 reading of DESIGN.md R15: x = T(A v_k); MGS with h_ik = <x, v_i>, x = T(x - h_ik v_i);
 * h_{k+1,k} = ||x||; v_{k+1} = x / h_{k+1,k}; Givens least squares on the host.
 *   history_out (HOST, steps+1 doubles): beta, then |g_{k+1}| after every step.
 *   steps_done  (HOST): number of Arnoldi steps performed (< steps on breakdown).
 *   explicit_out (HOST, nullable): ||T(b - A z)||_F for the returned iterate.
 *   step_ms_out (HOST, nullable, steps doubles): wall time of each Krylov step (host clock
 *   around a stream synchronisation).
 * Blocking. */
int tk_gmres_cycle(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int steps, double tol,
                   double* history_out, int* steps_done, double* explicit_out,
                   double* step_ms_out);

/* Complete, restarted low-rank GMRES: Alg. 3 with
 * P = I, restarted every `restart` Arnoldi steps with z_0 <- z, the stopping test
 * ||s_k|| <= tol_gmres ||b|| (line 2) and the truncated solution update
 * z <- T_eps_soln(z + sum_i y_i v_i) of eq:eps_soln; reading R19 of
 * within a cycle the test uses the Givens least-squares residual, z_k and the
 * explicit s_k = T_tol(b - A z_k) (lines 13-14) are formed at the end of each cycle.
 *   tol        : truncation tolerance eps_gmres of every T (line 5, MGS, lines 10, 14)
 *   eps_soln   : tolerance of the solution update (< 0: use tol)
 *   z          : OUT, caller-owned TT with capacity (TK_ECAP if the solution's ranks exceed
 *                it); mode sizes must be the operator's
 *   explicit_out (HOST, max_cycles + 1): ||s_0|| = ||T(b)||, then ||s|| after every cycle
 *   ls_out (HOST, nullable, max_cycles * (restart + 1)): per cycle the least-squares history
 *   cycles_done (HOST), steps_out (HOST, nullable, max_cycles): Arnoldi steps per cycle.
 * Blocking. */
int tk_gmres_solve(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int restart, int max_cycles,
                   double tol, double tol_gmres, double eps_soln, tk_tt* z, double* explicit_out,
                   double* ls_out, int* cycles_done, int* steps_out);

/* ===================================================================================== NEXT-3
 * The mean-based preconditioner of PAPER.md section 5.
 *
 * tk_bt: a direct solver for a sparse spatial matrix K (n x n, n = nb * N) that is BLOCK
 * TRIDIAGONAL in blocks of N consecutive rows (entries only between block rows i-1, i, i+1 —
 * the lexicographic 5-point finite-difference structure of the configs, R10, with N
 * the grid line length).  The factorisation is block LU (block Thomas) on the device:
 *   S_0 = D_0,  S_i = D_i - L_i S_{i-1}^{-1} U_{i-1};  E_i = S_i^{-1}, F_i = E_i U_i,
 *   G_i = E_i L_i   (dense N x N blocks; E_i from a Householder QR of S_i: R^{-1} Q^T)
 * and a solve is  y_i = E_i b_i - G_i y_{i-1}  (forward),  x_i = y_i - F_i x_{i+1}  (back).
 * Storage 3 nb N^2 doubles.  Singular or badly conditioned blocks are not detected beyond
 * non-finite results (TK_ENUMERIC from the GMRES / rounding calls that consume them).
 *
 * tk_bt_create: K = A + shift * I for the HOST CSR A (int32, 0-based).  TK_EARG if A has an
 *   entry outside the block-tridiagonal band or n != nb N.  Synchronous (setup).
 * tk_bt_create_gram: K = B B^T for the HOST CSR B (n x ncols); TK_EARG if a column of B
 *   couples rows more than one block row apart.  (The pressure Laplacian B M*^{-1} B^T of
 *   eq:mean_lsc, with M* = I.)  Synchronous (setup).
 * tk_bt_solve: y = (I (x) I (x) K^{-1}) x restricted to the rows [row0, row0 + reps n) of the
 *   space core: K^{-1} applied to each of the reps consecutive n-row blocks of U1 (x's r1
 *   columns), zero elsewhere; y.U2, y.U3 = x's (ranks unchanged, PAPER.md:244 with a single
 *   spatial factor).  y needs cap >= x's ranks and must not alias x.  Asynchronous. */
typedef struct tk_bt tk_bt;
int tk_bt_create(tk_ctx* ctx, tk_bt** bt, int64_t nb, int64_t N, const int32_t* rowptr,
                 const int32_t* col, const double* val, double shift);
int tk_bt_create_gram(tk_ctx* ctx, tk_bt** bt, int64_t nb, int64_t N, int64_t ncols,
                      const int32_t* rowptr, const int32_t* col, const double* val);
int tk_bt_destroy(tk_bt* bt);
int tk_bt_solve(tk_ctx* ctx, const tk_bt* bt, const tk_tt* x, int64_t row0, int reps, tk_tt* y);

/* tk_prec: the right preconditioner P^{-1} of eq:prec on the stacked spatial
 * mode [u1; u2; p] (R8, R20) with the two approximations of section 5:
 *   S^{-1} ~ S_LSC,0^{-1} = (B B^T)^{-1} B (F0 + C) B^T (B B^T)^{-1}    (eq:mean_lsc, M* = I)
 *   (F + C)^{-1} ~ inner low-rank GMRES on (F0 + C) u = w to tol_in (eq:11_sys), itself right
 *   preconditioned by M = (I - C) (x) I (x) (tau^-1 I + F0s) (eq:11_prec; w_avg = w0, R20)
 * F0 + C = ((I - C)/tau) (x) I (x) blkdiag(I, I, 0) + I (x) I (x) blkdiag(F0s, F0s, 0).
 * Inputs (HOST CSR, int32): F0s (n_v x n_v, n_v = grid^2) the mean convection-diffusion block
 * nu_0 L + N(w_0) of one velocity component; B (n_p x 2 n_v, n_p = grid^2) the divergence
 * [B1 B2]; n_x = 2 n_v + n_p.  tol: truncation eps of every T inside P^{-1}; inner GMRES:
 * restart_in steps per cycle, max_cycles_in cycles, stop at ||s|| <= tol_in ||w||.
 * Block size of both spatial solves: grid.  Synchronous (setup).
 *
 * tk_prec_apply: part 0 = P^{-1} v (steps 1-7 of DESIGN.md R20); part 1 = M^{-1} v (the
 * eq:11_prec solve: cumulative sum over time, K_s^{-1} on both velocity blocks, zero pressure
 * rows); part 2 = S_LSC,0^{-1} v_p on the pressure rows of v (positive sign, velocity rows
 * ignored).  out: caller TT, TK_ECAP if the result's ranks exceed its capacity.  Blocking
 * (the inner GMRES reads its Hessenberg entries on the host). */
typedef struct tk_prec tk_prec;
int tk_prec_create_lsc(tk_ctx* ctx, tk_prec** P, int64_t n_xi, int64_t n_t, int64_t grid,
                       const int32_t* F_rowptr, const int32_t* F_col, const double* F_val,
                       const int32_t* B_rowptr, const int32_t* B_col, const double* B_val,
                       double tau, double tol, double tol_in, int restart_in, int max_cycles_in);
int tk_prec_destroy(tk_prec* P);
int tk_prec_apply(tk_ctx* ctx, const tk_prec* P, int part, const tk_tt* v, tk_tt* out);
/* The preconditioner's operators (owned by P; valid while P lives): which = 0: F0 + C,
 * 1: the embedded B^T (pressure rows -> velocity rows), 2: the embedded B. */
const tk_op* tk_prec_operator(const tk_prec* P, int which);

/* tk_gmres_cycle / tk_gmres_solve with the right preconditioner P (flexible GMRES: Alg. 3 line
 * 4 v^_k = P^{-1} v_k, z = z_0 + sum_i y_i v^_i).  Same outputs; P must not be NULL. */
int tk_gmres_cycle_p(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b, int steps,
                     double tol, double* history_out, int* steps_done, double* explicit_out,
                     double* step_ms_out);
int tk_gmres_solve_p(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b,
                     int restart, int max_cycles, double tol, double tol_gmres, double eps_soln,
                     tk_tt* z, double* explicit_out, double* ls_out, int* cycles_done,
                     int* steps_out);

/* ===================================================================================== NEXT-4
 * The inexact Picard iteration of PAPER.md Alg. 1 (alg:picard, :199-213) for the all-at-once
 * stochastic Galerkin Navier-Stokes system eq:ns_sys_all (:148-156), reading R21 of DESIGN.md:
 *   line 1: z_0 = GMRES solve of stokes z = f to ||s|| <= tol_gmres ||f|| (:538)
 *           L = stokes + N(T_eps_conv(z_0)) (eq:N_kron from the iterate's cores on the device,
 *           eq:eps_conv), r_0 = T(f - L z_0)
 *   while ||r_i|| > tol_picard ||f|| and i < maxit:                                (line 2)
 *     dz = GMRES solve of L dz = r_{i-1} to ||s|| <= tol_gmres ||r_{i-1}|| (eq:inexact_solve)
 *     z_i = T(z_{i-1} + dz); L = stokes + N(T_eps_conv(z_i)); r_i = T(f - L z_i)  (lines 5-7)
 * Every T at eps_gmres (eps_conv < 0: eps_gmres); GMRES restarted every `restart` steps, at
 * most max_cycles cycles, right-preconditioned by P when P != NULL (NEXT-3).
 *   stokes: the fixed part (time-mass + Stokes block + KL viscosity terms, no convection)
 *   conv:   the discretisation of N(u) (tk_conv_create, d = 2 velocity components)
 *   f:      the right-hand side [f^u; f^p] (DEVICE TT)
 *   z_out:  OUT, caller TT (TK_ECAP if the solution's ranks exceed its capacity)
 *   residuals_out (HOST, maxit + 1): ||r_0||, ||r_1||, ...;  iterations (HOST): i on exit
 *   ranks_out (HOST, nullable, 2 (maxit + 1)): (r1, r2) of every iterate.
 * Blocking. */
int tk_picard(tk_ctx* ctx, const tk_op* stokes, const tk_conv* conv, const tk_prec* P,
              const tk_tt* f, double tol_picard, int maxit, double tol_gmres, double eps_gmres,
              double eps_conv, int restart, int max_cycles, tk_tt* z_out, double* residuals_out,
              int* iterations, int64_t* ranks_out);

#ifdef __cplusplus
}
#endif
#endif /* TTK_H */
