// Symmetric eigen-decomposition by two-sided BLOCK Jacobi (fp64, on device), as ONE
// persistent cooperative kernel.
//
// Used for PASS 2 of the two-pass Gram-Jacobi rounding: eigenvalues
// of the graded Gram W^T W with RELATIVE accuracy — Jacobi with the relative skip test
// |a_pq| <= rel * sqrt(|a_pp a_qq|) provides that (Demmel-Veselic); tridiagonal QR does not.
//
// Layout: the matrix is embedded in an n_pad x n_pad buffer (n_pad = 64 * ceil(n/64), zero
// padding — padded indices never rotate since their couplings are 0), split into
// nb = n_pad/32 blocks of 32 rows/cols.  One sweep = nb-1 rounds of a round-robin
// tournament over blocks; a round handles nb/2 disjoint block pairs (I, J) in two phases
// separated by grid-wide barriers:
//   inner  one CTA per pair: S = G[I u J, I u J] (64 x 64) in shared memory, one scalar
//          cyclic Jacobi sweep (parallel ordering, Rutishauser updates of each 2x2 pivot)
//          accumulating Q (64 x 64); Q and the rotated S go to global memory.
//   update G[IJ_t, IJ_s] <- Q_t^T G[IJ_t, IJ_s] Q_s for t < s (written to both triangles: G
//          stays exactly symmetric), G[IJ_t, IJ_t] <- S_t (the inner result, so annihilated
//          entries stay exactly 0), and V[:, IJ_t] <- V[:, IJ_t] Q_t   (64 x 64 DMMA tiles)
// Rotation counts per sweep end the loop (all CTAs read the counter after the barrier).
//
// Cluster skip (disabled: tk_jacobi_eig callers pass lskip = nullptr): when lskip >= 0, rotations between two indices whose
// diagonal entries are both <= lskip are skipped.  lskip is chosen (cluster_skip_k) so the
// skipped cluster's total mass is <= delta^2/4: its internal structure cannot move the rank
// decision (only its trace enters the discarded tail, and the trace is invariant); couplings
// between the cluster and the rest are still annihilated.  tk_round verifies afterwards that
// the chosen rank lies above the cluster and otherwise re-runs without the skip.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ttk_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int JB = 32;        // block size
constexpr int JS = 2 * JB;    // pair size (64)
constexpr int JLD = JS + 1;   // shared-memory leading dimension
constexpr int JT = 512;       // threads per CTA

struct JacArgs {
  int n_pad, nb, npairs;
  int v_tiles;          // 64-row tiles of V (V is v_tiles*64 x n_pad, ld n_pad)
  double* G;
  double* V;
  double* Qb;
  double* Sb;
  const double* d_maxdiag;
  const double* abs_floor;  // nullable: absolute skip floor (rounding-noise level of the data)
  double abs_scale, rel_tol;
  const double* lskip;  // nullable
  int max_inner, max_sweeps;
  int* stats;           // rotation count per sweep
  unsigned long long* offmax;  // per sweep: max |a_pq|/sqrt(a_pp a_qq) over applied rotations
  double stop_rel;      // stop after a sweep whose offmax <= stop_rel (0: only when no rotation)
  int n;                // real (unpadded) size
  double rs_tol;        // rank-aware skip: tol of the rank rule (<= 0: off)
  long long rs_rmax;    // rank cap of the rank rule (<= 0: none)
  double* lskip_io;     // nullable: [0] in: static cluster threshold / out: effective one
  unsigned long long* tstamp;  // nullable: per-phase time sums of CTA 0 (TTK_DEBUG)
  int* sweeps_out;
};

__host__ __device__ __forceinline__ int rr_player(int pos, int r, int ne) {
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (ne - 1);
}
__device__ __forceinline__ void pair_blocks(int t, int r, int nb, int& I, int& J) {
  int a = rr_player(t, r, nb), b = rr_player(nb - 1 - t, r, nb);
  I = min(a, b);
  J = max(a, b);
}
// global index of local index l (0..63) of the pair (I, J)
__device__ __forceinline__ int gidx(int l, int I, int J) {
  return l < JB ? I * JB + l : J * JB + (l - JB);
}
// upper-triangle position of (i, j) in the inner solve's shared S
__device__ __forceinline__ int uidx(int i, int j) {
  return i <= j ? i * JLD + j : j * JLD + i;
}

struct InnerShared {
  double rc[JB], rs[JB], rt[JB], rapp[JB], raqq[JB], rapq[JB];
  int rp[JB], rq[JB], ract[JB];
  int nrot;
  double offmax;
};

// skip test without a square root: rotate iff |a_pq| > thr, thr = max(abs, rel sqrt(a_pp a_qq)),
// i.e. a_pq^2 > max(abs^2, rel^2 |a_pp a_qq|); cluster pairs never rotate.
__device__ __forceinline__ bool needs_rot(double app, double aqq, double apq, double abs_tol,
                                          double rel, double lsk) {
  if (app <= lsk && aqq <= lsk) return false;
  const double a2 = apq * apq;
  return a2 > abs_tol * abs_tol && a2 > rel * rel * fabs(app * aqq);
}

// Rotation annihilating a_pq: t = sgn(d) e / u with u = |d| + h, h = sqrt(d^2 + e^2),
// d = a_qq - a_pp, e = 2 a_pq;  c = u / sqrt(u^2 + e^2), s = sgn(d) e / sqrt(u^2 + e^2).
// Two dependent special functions (h = x rsqrt(x), then rsqrt(u^2 + e^2) with the division
// e / u in parallel); c^2 + s^2 = 1 to rounding whatever the accuracy of h.
__device__ __forceinline__ void rot_params(double app, double aqq, double apq, double& c,
                                           double& sn, double& tt) {
  const double d = aqq - app, e2 = 2.0 * apq;
  const double es = d >= 0.0 ? e2 : -e2;
  const double x = fma(d, d, e2 * e2);
  const double u = fabs(d) + x * rsqrt(x);
  const double rn = rsqrt(fma(u, u, e2 * e2));
  tt = es / u;
  c = u * rn;
  sn = es * rn;
}

// The 32 cross rounds of one pair (p in block I, q in block J): in inner round ir pair k is
// (p = k, q = 32 + (k + ir) % 32).  Lean version of the generic round below:
//   * warp 0 computes the 32 rotations and applies them to its own diagonal 2 x 2 blocks at
//     once (it holds a_pp, a_qq, a_pq, t), so the other threads only see the strictly upper
//     pair-blocks (P1 < P2): 496 of them, one per thread — warp w owns rows P1 = w (lanes > w)
//     and P1 = 31 - w (lanes < w) — with fixed p1, p2 and incrementally known q1, q2: no index
//     loads, and the (p1, p2) element stays in a register for all 32 rounds;
//   * Q lives in registers: thread (warp w, lane l) holds rows w + 16 m of column l and of
//     column 32 + (l + ir) % 32; after each round the partner columns move one lane down.
//   * the largest rotated relative coupling is tracked as a fraction (a_pq^2 / |a_pp a_qq|
//     compared by cross-multiplication), one division and square root at the end.
__device__ __forceinline__ void inner_cross(const JacArgs& a, double* S, double* Q, InnerShared& sh,
                                            double abs_tol, double lsk, int& my_rot,
                                            double& my_off) {
  const int tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
  const bool has_blk = lane != wq;
  const int P1 = lane > wq ? wq : 31 - wq, P2 = lane > wq ? lane : 31 - lane;
  double x00 = has_blk ? S[P1 * JLD + P2] : 0.0;
  double qr_p[4], qr_q[4];
#pragma unroll
  for (int m = 0; m < 4; m++) {
    qr_p[m] = (wq + 16 * m == lane) ? 1.0 : 0.0;
    qr_q[m] = (wq + 16 * m == JB + lane) ? 1.0 : 0.0;
  }
  double off_num = 0.0, off_den = 1.0;  // warp 0: max of a_pq^2 / |a_pp a_qq| as a fraction
  for (int ir = 0; ir < JB; ir++) {
    if (tid < JB) {
      const int p = tid, q = JB + ((tid + ir) & (JB - 1));
      const double app = S[p * JLD + p], aqq = S[q * JLD + q], apq = S[p * JLD + q];
      double c = 1.0, sn = 0.0;
      int act = 0;
      if (needs_rot(app, aqq, apq, abs_tol, a.rel_tol, lsk)) {
        double tt;
        rot_params(app, aqq, apq, c, sn, tt);
        act = 1;
        S[p * JLD + p] = app - tt * apq;
        S[q * JLD + q] = aqq + tt * apq;
        S[p * JLD + q] = 0.0;
        const double num = apq * apq, den = fmax(fabs(app * aqq), 1e-300);
        if (num * off_den > off_num * den) {
          off_num = num;
          off_den = den;
        }
        my_rot++;
      }
      sh.rc[tid] = c;
      sh.rs[tid] = sn;
      sh.ract[tid] = act;
    }
    __syncthreads();
    {
      const double c2 = sh.rc[lane], s2 = sh.rs[lane];
      const int act2 = sh.ract[lane];
      if (has_blk) {
        const int actb = sh.ract[P1] | sh.ract[P2];
        if (actb) {
          const double c1 = sh.rc[P1], s1 = sh.rs[P1], cb = sh.rc[P2], sb = sh.rs[P2];
          const int q1 = JB + ((P1 + ir) & (JB - 1)), q2 = JB + ((P2 + ir) & (JB - 1));
          const int i01 = P1 * JLD + q2, i10 = P2 * JLD + q1;
          const int i11 = q1 <= q2 ? q1 * JLD + q2 : q2 * JLD + q1;
          const double x01 = S[i01], x10 = S[i10], x11 = S[i11];
          const double y00 = cb * x00 - sb * x01, y01 = sb * x00 + cb * x01;
          const double y10 = cb * x10 - sb * x11, y11 = sb * x10 + cb * x11;
          x00 = c1 * y00 - s1 * y10;
          S[i10] = s1 * y00 + c1 * y10;
          S[i01] = c1 * y01 - s1 * y11;
          S[i11] = s1 * y01 + c1 * y11;
        }
      }
#pragma unroll
      for (int m = 0; m < 4; m++) {
        if (act2) {
          const double qp = qr_p[m], qq = qr_q[m];
          qr_p[m] = c2 * qp - s2 * qq;
          qr_q[m] = s2 * qp + c2 * qq;
        }
        qr_q[m] = __shfl_sync(0xffffffffu, qr_q[m], (lane + 1) & 31);
      }
    }
    __syncthreads();
  }
  if (has_blk) S[P1 * JLD + P2] = x00;
  // after JB rounds lane l holds column JB + l again
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const int i = wq + 16 * m;
    Q[i * JLD + lane] = qr_p[m];
    Q[i * JLD + JB + lane] = qr_q[m];
  }
  if (tid < JB) my_off = fmax(my_off, sqrt(off_num / off_den));
  __syncthreads();
}

// One pair's inner problem, by one CTA (JT = 512 threads).  Per inner round: (a) warp 0
// computes the 32 disjoint rotations; (b) every thread applies J^T S J to two 2x2 blocks
// (rows of one pair x columns of another: each element belongs to exactly one block, so the
// update is in place) and Q <- Q J to four (row, pair) items.  Two barriers per round.
// staged: S (full symmetric) and Q = I are already in shared memory (the dataflow schedule builds
// the pair's block itself); Qout / Sout: where this pair's Q and rotated S go.
__device__ void inner_solve(const JacArgs& a, int t, int r, double* sm, InnerShared& sh,
                            double abs_tol, double lsk, bool staged = false,
                            double* Qout = nullptr, double* Sout = nullptr) {
  double* S = sm;
  double* Q = sm + JS * JLD;
  int I, J;
  pair_blocks(t, r, a.nb, I, J);
  const double* G = a.G;
  const int n_pad = a.n_pad;
  const int tid = threadIdx.x;
  if (!Qout) Qout = a.Qb;
  if (!Sout) Sout = a.Sb;
  if (!staged) {
    for (int e = tid; e < JS * JS; e += blockDim.x) {
      int i = e / JS, j = e % JS;
      int gi = gidx(i, I, J), gj = gidx(j, I, J);
      S[i * JLD + j] = 0.5 * (G[(int64_t)gi * n_pad + gj] + G[(int64_t)gj * n_pad + gi]);
      Q[i * JLD + j] = (i == j) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  {
    int any = 0;
    for (int e = tid; e < JS * JS; e += blockDim.x) {
      int i = e / JS, j = e % JS;
      if (j <= i) continue;
      any |= needs_rot(S[i * JLD + i], S[j * JLD + j], S[i * JLD + j], abs_tol, a.rel_tol, lsk);
    }
    any = __syncthreads_or(any);
    if (!any) {
      double* Qo = Qout + (int64_t)t * JS * JS;
      double* So = Sout + (int64_t)t * JS * JS;
      for (int e = tid; e < JS * JS; e += blockDim.x) {
        Qo[e] = Q[(e / JS) * JLD + e % JS];
        So[e] = S[uidx(e / JS, e % JS)];
      }
      __syncthreads();
      return;
    }
  }
  int my_rot = 0;          // warp 0 lanes: rotations applied (this call)
  double my_off = 0.0;     // warp 0 lanes: largest relative coupling rotated away
  // The first outer round of a sweep (r == 0, every block appears once) runs the full
  // 63-round inner sweep; later rounds only rotate the 32 x 32 cross pairs (i in I, j in J):
  // 32 inner rounds of 32 disjoint pairs.  Every index pair is still visited once per sweep.
  const bool cross = (r != 0) && (a.npairs > 1);
  const int lane = tid & 31, wq = tid >> 5;
  if (cross) {
    inner_cross(a, S, Q, sh, abs_tol, lsk, my_rot, my_off);
  } else {
    for (int sweep = 0; sweep < a.max_inner; sweep++) {
      int sweep_rot = 0;
      for (int ir = 0; ir < JS - 1; ir++) {
        if (tid < JB) {
          const int k = tid;
          const int pa = rr_player(k, ir, JS), pb = rr_player(JS - 1 - k, ir, JS);
          const int p = min(pa, pb), q = max(pa, pb);
          const double app = S[p * JLD + p], aqq = S[q * JLD + q], apq = S[p * JLD + q];
          double c = 1.0, sn = 0.0, tt = 0.0;
          int act = 0;
          if (needs_rot(app, aqq, apq, abs_tol, a.rel_tol, lsk)) {
            rot_params(app, aqq, apq, c, sn, tt);
            act = 1;
          }
          sh.rc[k] = c;
          sh.rs[k] = sn;
          sh.rt[k] = tt;
          sh.rapp[k] = app;
          sh.raqq[k] = aqq;
          sh.rapq[k] = apq;
          sh.rp[k] = p;
          sh.rq[k] = q;
          sh.ract[k] = act;
          sweep_rot += act;
        }
        __syncthreads();
        // S <- J^T S J on 2x2 blocks (pair P1 rows, pair P2 cols) and Q <- Q J.  Only the upper
        // triangle of S is kept (uidx): block (P1, P2) for P1 <= P2 covers each element once.
        // Thread map: P2 = lane (parameters loaded once), P1 = warp and warp + 16; Q rows
        // warp + 16 m (m < 4) of pair lane.
        {
          const double c2 = sh.rc[lane], s2 = sh.rs[lane];
          const int p2 = sh.rp[lane], q2 = sh.rq[lane], act2 = sh.ract[lane];
          if (wq == 0 && act2)
            my_off = fmax(my_off, fabs(sh.rapq[lane]) *
                                      rsqrt(fmax(fabs(sh.rapp[lane] * sh.raqq[lane]), 1e-300)));
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int P1 = wq + 16 * h;
            if (P1 > lane) continue;
            const int act1 = sh.ract[P1];
            if (!act1 && !act2) continue;
            const int p1 = sh.rp[P1], q1 = sh.rq[P1];
            if (P1 == lane) {
              const double t1 = sh.rt[P1], a1 = sh.rapq[P1];
              S[p1 * JLD + p1] = sh.rapp[P1] - t1 * a1;
              S[q1 * JLD + q1] = sh.raqq[P1] + t1 * a1;
              S[p1 * JLD + q1] = 0.0;  // p1 < q1
              continue;
            }
            const double c1 = sh.rc[P1], s1 = sh.rs[P1];
            const int i00 = uidx(p1, p2), i01 = uidx(p1, q2), i10 = uidx(q1, p2),
                      i11 = uidx(q1, q2);
            const double x00 = S[i00], x01 = S[i01], x10 = S[i10], x11 = S[i11];
            const double y00 = c2 * x00 - s2 * x01, y01 = s2 * x00 + c2 * x01;
            const double y10 = c2 * x10 - s2 * x11, y11 = s2 * x10 + c2 * x11;
            S[i00] = c1 * y00 - s1 * y10;
            S[i10] = s1 * y00 + c1 * y10;
            S[i01] = c1 * y01 - s1 * y11;
            S[i11] = s1 * y01 + c1 * y11;
          }
          if (act2) {
#pragma unroll
            for (int m = 0; m < 4; m++) {
              const int i = wq + 16 * m;
              const double qp = Q[i * JLD + p2], qq = Q[i * JLD + q2];
              Q[i * JLD + p2] = c2 * qp - s2 * qq;
              Q[i * JLD + q2] = s2 * qp + c2 * qq;
            }
          }
        }
        __syncthreads();
      }
      // inner convergence (only matters when max_inner > 1)
      if (tid < JB) {
        int v = sweep_rot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (tid == 0) sh.nrot = v;
        my_rot += sweep_rot;
      }
      __syncthreads();
      const bool done = (sh.nrot == 0);
      __syncthreads();
      if (done) break;
    }
  }
  double* Qo = Qout + (int64_t)t * JS * JS;
  double* So = Sout + (int64_t)t * JS * JS;
  for (int e = tid; e < JS * JS; e += blockDim.x) {
    Qo[e] = Q[(e / JS) * JLD + e % JS];
    So[e] = S[uidx(e / JS, e % JS)];
  }
  if (tid < JB) {
    int v = my_rot;
    double o = my_off;
#pragma unroll
    for (int w = 16; w > 0; w >>= 1) {
      v += __shfl_xor_sync(0xffffffffu, v, w);
      o = fmax(o, __shfl_xor_sync(0xffffffffu, o, w));
    }
    if (tid == 0 && v) {
      atomicAdd(a.stats, v);
      atomicMax(a.offmax, (unsigned long long)__double_as_longlong(o));
    }
  }
  __syncthreads();
}

constexpr int TLD = JS + 4;  // tile leading dimension (68): conflict-free DMMA fragments

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// acc <- this warp's (8 FI) x (8 FJ) block at (wm, wn) of C = op(A) B (64 x 64 x 64, A / B in
// shared memory with leading dimension TLD; transA: op(A)[m][k] = A[k][m]).  An output element is
// the same chain of k-steps whatever FI, FJ and the warp map: sub-block products are bitwise
// equal to the corresponding entries of the full product.
template <int FI, int FJ>
__device__ __forceinline__ void tile_mma_at(const double* As, bool transA, const double* Bs,
                                            double acc[FI][FJ][2], int wm, int wn) {
  const int lane = threadIdx.x & 31;
  const int lr = lane >> 2, lc = lane & 3;
#pragma unroll
  for (int i = 0; i < FI; i++)
#pragma unroll
    for (int j = 0; j < FJ; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < JS; k += 4) {
    double av[FI], bv[FJ];
#pragma unroll
    for (int i = 0; i < FI; i++) {
      const int m = wm + 8 * i + lr, kk = k + lc;
      av[i] = transA ? As[kk * TLD + m] : As[m * TLD + kk];
    }
#pragma unroll
    for (int j = 0; j < FJ; j++) bv[j] = Bs[(k + lc) * TLD + wn + 8 * j + lr];
#pragma unroll
    for (int i = 0; i < FI; i++)
#pragma unroll
      for (int j = 0; j < FJ; j++) dmma884(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
  }
}
// the full 64 x 64 product: 16 warps, each a 16 x 16 block
__device__ __forceinline__ void tile_mma(const double* As, bool transA, const double* Bs,
                                         double acc[2][2][2]) {
  const int warp = threadIdx.x >> 5;
  tile_mma_at<2, 2>(As, transA, Bs, acc, (warp >> 2) * 16, (warp & 3) * 16);
}

// 64-row tile of M[:, I u J] <- M[:, I u J] Q   (DMMA)
__device__ void col_tile(const JacArgs& a, double* M, int row0, int t, int r, double* sm) {
  double* Qs = sm;
  double* Ts = sm + JS * TLD;
  int I, J;
  pair_blocks(t, r, a.nb, I, J);
  const double* Q = a.Qb + (int64_t)t * JS * JS;
  const int n_pad = a.n_pad;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    Qs[i * TLD + j] = Q[e];
    Ts[i * TLD + j] = M[(int64_t)(row0 + i) * n_pad + gidx(j, I, J)];
  }
  __syncthreads();
  double acc[2][2][2];
  tile_mma(Ts, false, Qs, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int m = wm + 8 * i + (lane >> 2), n = wn + 8 * j + 2 * (lane & 3) + h;
        M[(int64_t)(row0 + m) * n_pad + gidx(n, I, J)] = acc[i][j][h];
      }
  __syncthreads();
}

// Two-sided block of G for pairs t < s:  G[IJ_t, IJ_s] <- Q_t^T G[IJ_t, IJ_s] Q_s, written to
// both G[IJ_t, IJ_s] and (transposed) G[IJ_s, IJ_t]; for t == s the block is the inner solve's S.
// One work item per unordered pair of pairs replaces the former column phase on G and the row
// phase (G stays exactly symmetric, one grid barrier less per round).
__device__ void sym_tile(const JacArgs& a, int t, int s, int r, double* sm) {
  double* G = a.G;
  const int n_pad = a.n_pad;
  int It, Jt, Is, Js;
  pair_blocks(t, r, a.nb, It, Jt);
  pair_blocks(s, r, a.nb, Is, Js);
  if (t == s) {
    const double* S = a.Sb + (int64_t)t * JS * JS;
    for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
      const int i = e / JS, j = e % JS;
      G[(int64_t)gidx(i, It, Jt) * n_pad + gidx(j, It, Jt)] = S[e];
    }
    return;
  }
  double* Qs = sm;                 // Q_s
  double* Xs = sm + JS * TLD;      // G block, then G block Q_s
  double* Qt = sm + 2 * JS * TLD;  // Q_t
  const double* Qsg = a.Qb + (int64_t)s * JS * JS;
  const double* Qtg = a.Qb + (int64_t)t * JS * JS;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    const int i = e / JS, j = e % JS;
    Qs[i * TLD + j] = Qsg[e];
    Qt[i * TLD + j] = Qtg[e];
    Xs[i * TLD + j] = G[(int64_t)gidx(i, It, Jt) * n_pad + gidx(j, Is, Js)];
  }
  __syncthreads();
  double acc[2][2][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;
  tile_mma(Xs, false, Qs, acc);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        Xs[(wm + 8 * i + (lane >> 2)) * TLD + wn + 8 * j + 2 * (lane & 3) + h] = acc[i][j][h];
  __syncthreads();
  tile_mma(Qt, true, Xs, acc);
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int m = wm + 8 * i + (lane >> 2), n = wn + 8 * j + 2 * (lane & 3) + h;
        const int gm = gidx(m, It, Jt), gn = gidx(n, Is, Js);
        G[(int64_t)gm * n_pad + gn] = acc[i][j][h];
        G[(int64_t)gn * n_pad + gm] = acc[i][j][h];
      }
  __syncthreads();
}

// CTA 0: lskip = (r + 32)-th largest diagonal entry, r = rank rule (tail of the clamped
// diagonal <= delta^2 = tol^2 trace / 2, capped at rmax) — written to a.lskip_io[0].
__device__ void rank_skip_update(const JacArgs& a, double* sm, double& sh_out) {
  const int n = a.n;
  double* d = sm;       // n values
  double* srt = sm + n; // n values, descending
  if (2 * n > 2 * JS * JLD) {
    if (threadIdx.x == 0) a.lskip_io[0] = -1.0;
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    d[i] = fmax(a.G[(int64_t)i * a.n_pad + i], 0.0);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int rk = 0;
    const double di = d[i];
    for (int j = 0; j < n; j++) rk += (d[j] > di) || (d[j] == di && j < i);
    srt[rk] = di;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int i = n - 1; i >= 0; i--) tr += srt[i];
    const double d2 = a.rs_tol * a.rs_tol * tr * 0.5;
    int r = n;
    double tail = 0.0;
    for (int cand = n; cand >= 1; cand--) {
      if (tail <= d2)
        r = cand;
      else
        break;
      tail += srt[cand - 1];
    }
    if (a.rs_rmax > 0 && r > a.rs_rmax) r = (int)a.rs_rmax;
    const int idx = r + 32;
    a.lskip_io[0] = idx < n ? srt[idx] : -1.0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(JT) jacobi_persistent_k(JacArgs a, int coop) {
  extern __shared__ double sm[];
  __shared__ InnerShared sh;
  const double abs_tol =
      fmax(fmax(a.abs_scale * a.d_maxdiag[0], a.abs_floor ? a.abs_floor[0] : 0.0), 1e-300);
  const double lsk_static = a.lskip ? a.lskip[0] : -1.0;
  double lsk = lsk_static;
  __shared__ double sh_lsk;
  unsigned long long tsum[6] = {0, 0, 0, 0, 0, 0}, tprev = 0;
  const bool rec = a.tstamp && blockIdx.x == 0 && threadIdx.x == 0;
  auto mark = [&](int k) {
    if (rec) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (k >= 0) tsum[k] += now - tprev;
      tprev = now;
    }
  };
  int sweep = 0;
  for (; sweep < a.max_sweeps; sweep++) {
    if (a.rs_tol > 0.0 && sweep > 0 && a.lskip_io) {
      // rank-aware skip: indices whose diagonal lies below the (r + 32)-th largest current
      // diagonal, r the rank rule applied to the current diagonal, only matter through their
      // trace; their mutual rotations are skipped from now on (checked after convergence)
      if (blockIdx.x == 0) rank_skip_update(a, sm, sh_lsk);
      if (coop) cg::this_grid().sync(); else __syncthreads();
      lsk = fmax(lsk_static, *((volatile double*)a.lskip_io));
    }
    JacArgs as = a;
    as.stats = a.stats + sweep;
    as.offmax = a.offmax + sweep;
    for (int r = 0; r < a.nb - 1; r++) {
      mark(-1);
      for (int t = blockIdx.x; t < a.npairs; t += gridDim.x) inner_solve(as, t, r, sm, sh, abs_tol, lsk);
      mark(0);
      if (coop) cg::this_grid().sync(); else __syncthreads();
      mark(1);
      // G: two-sided blocks for t <= s (heavier items first); V: column tiles V[:, IJ_t] Q_t
      const int nsym = a.npairs * (a.npairs + 1) / 2;
      const int nitems = nsym + a.v_tiles * a.npairs;
      for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        if (w < nsym) {
          // w -> (t, s), t <= s, row-major over the upper triangle
          int t = 0, rem = w;
          while (rem >= a.npairs - t) {
            rem -= a.npairs - t;
            t++;
          }
          sym_tile(as, t, t + rem, r, sm);
        } else {
          const int v = w - nsym;
          col_tile(as, a.V, (v % a.v_tiles) * JS, v / a.v_tiles, r, sm);
        }
      }
      mark(2);
      if (coop) cg::this_grid().sync(); else __syncthreads();
      mark(3);
      mark(4);
      mark(5);
    }
    const int rot = *((volatile int*)(a.stats + sweep));
    const double om = __longlong_as_double(
        (long long)*((volatile unsigned long long*)(a.offmax + sweep)));
    if (rot == 0 || a.npairs == 1 || om <= a.stop_rel) {
      sweep++;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.sweeps_out[0] = sweep;
    if (a.lskip_io) a.lskip_io[0] = lsk;  // effective final threshold
  }
  if (rec)
    for (int k = 0; k < 6; k++) a.tstamp[k] = tsum[k];  // [6], [7]: inner phase cycles
}


// ---------------------------------------------------------------------------------------------
// Dataflow schedule ("flow"): the same rounds, pairs, rotations and tile products as
// jacobi_persistent_k, without grid-wide barriers.  CTAs 0..npairs-1 only solve pairs, the others
// only apply tile updates, and the two groups run one round apart:
//   * G is double buffered: G_R (the state after the tile phase of global round R) lives in
//     Gbuf[R & 1], the embedded input G_{-1} in Gbuf[1]; tile phase R reads G_{R-1} and writes G_R
//     (every block belongs to exactly one (t, s) item per round, so all of G_R is written).
//   * The pair CTA of round R builds its own 64 x 64 input block of G_{R-1} instead of waiting
//     for tile phase R-1: the two diagonal 32 x 32 blocks come from the rotated S of the pairs
//     (a, b) that held blocks I and J in round R-1, the coupling block is the (I, J) part of
//     Q_a^T G_{R-2}[IJ_a, IJ_b] Q_b (the same DMMA products, in the same order, the tile phase
//     uses: the values are bitwise those of G_{R-1}).  So inner(R) depends on inner(R-1) (all
//     pairs) and on tile phase R-2 only, and overlaps tile phase R-1.
//   * Q and S of the pairs are double buffered by round parity (tile phase R-1 still reads
//     Q_{R-1} while inner(R) writes Q_R).
// Ordering is by two monotonic counters in global memory (finished inner solves, finished tile
// items): writers __syncthreads + __threadfence + atomicAdd, readers ld.acquire.gpu spin by one
// thread + __syncthreads; data shared between CTAs is read with ld.global.cg.  All CTAs must be
// co-resident (cooperative launch; no grid.sync is used).
struct FlowArgs {
  JacArgs a;            // a.G unused; a.Qb / a.Sb: [2][npairs * 64 * 64]
  double* Gbuf[2];
  unsigned int* cnt;    // [0] finished inner solves, [1] finished tile items
  double* diag_out;     // n_pad: diagonal of the final G
};

__device__ __forceinline__ void flow_wait(const unsigned int* c, unsigned int target) {
  if (threadIdx.x == 0) {
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}
__device__ __forceinline__ void flow_signal(unsigned int* c, unsigned int inc) {
  __syncthreads();
  if (threadIdx.x == 0 && inc) {
    __threadfence();
    atomicAdd(c, inc);
  }
}

// slot and half (0: rows 0..31 of the pair, 1: rows 32..63) of block B in tournament round r:
// the inverse of rr_player (position of B), its partner sits at position nb - 1 - pos
__device__ __forceinline__ void find_block(int B, int r, int nb, int& slot, int& half) {
  const int ne1 = nb - 1;
  int pos = 0;
  if (B != 0) {
    int d = (B - 1 - r) % ne1;
    if (d < 0) d += ne1;
    pos = 1 + d;
  }
  const int ppos = nb - 1 - pos;
  slot = min(pos, ppos);
  half = B < rr_player(ppos, r, nb) ? 0 : 1;
}

// Two-sided tile product shared by the tile phase and the pair CTAs' input construction:
// acc <- (Q_t^T (X Q_s)) fragments, X = Gin[IJ_t, IJ_s]; Qs/Xs/Qt: three 64 x TLD tiles in sm.
__device__ __forceinline__ void two_sided_tile(const double* __restrict__ Gin, int n_pad,
                                               const double* __restrict__ Qtg,
                                               const double* __restrict__ Qsg, int It, int Jt,
                                               int Is, int Js, double* sm, double acc[2][2][2]) {
  double* Qs = sm;
  double* Xs = sm + JS * TLD;
  double* Qt = sm + 2 * JS * TLD;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    const int i = e / JS, j = e % JS;
    Qs[i * TLD + j] = __ldcg(Qsg + e);
    Qt[i * TLD + j] = __ldcg(Qtg + e);
    Xs[i * TLD + j] = __ldcg(Gin + (int64_t)gidx(i, It, Jt) * n_pad + gidx(j, Is, Js));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;
  tile_mma(Xs, false, Qs, acc);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        Xs[(wm + 8 * i + (lane >> 2)) * TLD + wn + 8 * j + 2 * (lane & 3) + h] = acc[i][j][h];
  __syncthreads();
  tile_mma(Qt, true, Xs, acc);
}

__device__ void flow_sym_tile(const FlowArgs& f, int R, int t, int s, int r, double* sm) {
  const JacArgs& a = f.a;
  const int n_pad = a.n_pad;
  const double* Gin = f.Gbuf[(R + 1) & 1];
  double* Gout = f.Gbuf[R & 1];
  const int64_t qoff = (int64_t)(R & 1) * a.npairs * JS * JS;
  int It, Jt, Is, Js;
  pair_blocks(t, r, a.nb, It, Jt);
  pair_blocks(s, r, a.nb, Is, Js);
  if (t == s) {
    const double* S = a.Sb + qoff + (int64_t)t * JS * JS;
    for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
      const int i = e / JS, j = e % JS;
      Gout[(int64_t)gidx(i, It, Jt) * n_pad + gidx(j, It, Jt)] = __ldcg(S + e);
    }
    return;
  }
  double acc[2][2][2];
  two_sided_tile(Gin, n_pad, a.Qb + qoff + (int64_t)t * JS * JS, a.Qb + qoff + (int64_t)s * JS * JS,
                 It, Jt, Is, Js, sm, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int m = wm + 8 * i + (lane >> 2), n = wn + 8 * j + 2 * (lane & 3) + h;
        const int gm = gidx(m, It, Jt), gn = gidx(n, Is, Js);
        Gout[(int64_t)gm * n_pad + gn] = acc[i][j][h];
        Gout[(int64_t)gn * n_pad + gm] = acc[i][j][h];
      }
  __syncthreads();
}

// 64-row tile of V[:, I u J] <- V[:, I u J] Q_t (in place; Q of global round R)
__device__ void flow_col_tile(const FlowArgs& f, int R, int row0, int t, int r, double* sm) {
  const JacArgs& a = f.a;
  double* Qs = sm;
  double* Ts = sm + JS * TLD;
  int I, J;
  pair_blocks(t, r, a.nb, I, J);
  const double* Q = a.Qb + (int64_t)(R & 1) * a.npairs * JS * JS + (int64_t)t * JS * JS;
  double* M = a.V;
  const int n_pad = a.n_pad;
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    int i = e / JS, j = e % JS;
    Qs[i * TLD + j] = __ldcg(Q + e);
    Ts[i * TLD + j] = __ldcg(M + (int64_t)(row0 + i) * n_pad + gidx(j, I, J));
  }
  __syncthreads();
  double acc[2][2][2];
  tile_mma(Ts, false, Qs, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp >> 2) * 16, wn = (warp & 3) * 16;
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int m = wm + 8 * i + (lane >> 2), n = wn + 8 * j + 2 * (lane & 3) + h;
        M[(int64_t)(row0 + m) * n_pad + gidx(n, I, J)] = acc[i][j][h];
      }
  __syncthreads();
}

// Stage the pair's input block S = G_{R-1}[I u J, I u J] and Q = I in shared memory.  For R >= 1
// in two parts: part 0 (needs only tile phase R-2) loads the G_{R-2} block — issued before the
// wait for the pair solves of round R-1, whose imbalance hides its latency; part 1 the rest.
__device__ void flow_stage_input(const FlowArgs& f, int R, int t, int r, double* sm, int part) {
  const JacArgs& a = f.a;
  const int n_pad = a.n_pad, nrounds = a.nb - 1;
  double* S = sm;
  double* Q = sm + JS * JLD;
  int I, J;
  pair_blocks(t, r, a.nb, I, J);
  if (R == 0) {
    if (part == 0) return;
    const double* G = f.Gbuf[1];
    for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
      int i = e / JS, j = e % JS;
      int gi = gidx(i, I, J), gj = gidx(j, I, J);
      S[i * JLD + j] = 0.5 * (G[(int64_t)gi * n_pad + gj] + G[(int64_t)gj * n_pad + gi]);
      Q[i * JLD + j] = (i == j) ? 1.0 : 0.0;
    }
    return;
  }
  const int rp = (r + nrounds - 1) % nrounds;
  int ta, ha, tb, hb;
  find_block(I, rp, a.nb, ta, ha);
  find_block(J, rp, a.nb, tb, hb);
  int Ia, Ja, Ib, Jb;
  pair_blocks(ta, rp, a.nb, Ia, Ja);
  pair_blocks(tb, rp, a.nb, Ib, Jb);
  const int64_t qoff = (int64_t)((R - 1) & 1) * a.npairs * JS * JS;
  const double* Qa = a.Qb + qoff + (int64_t)ta * JS * JS;
  const double* Qbb = a.Qb + qoff + (int64_t)tb * JS * JS;
  const double* Sa = a.Sb + qoff + (int64_t)ta * JS * JS;
  const double* Sbb = a.Sb + qoff + (int64_t)tb * JS * JS;
  // coupling block: the tile phase computes item (min, max) of the two slots, Y = Q_t^T (X Q_s)
  // with X = G_{R-2}[IJ_t, IJ_s], and mirrors it; only the (hr, hc) quarter of Y is needed —
  // the 32 columns hc of X Q_s (16 warps x (16 x 8)), then the 32 x 32 quarter of Q_t^T (.)
  // (16 warps x (8 x 8)): the same k-chains as the tile phase, so the values are bitwise its.
  const bool ab = ta < tb;
  const int It = ab ? Ia : Ib, Jt = ab ? Ja : Jb, Is = ab ? Ib : Ia, Js = ab ? Jb : Ja;
  const double* Qtg = ab ? Qa : Qbb;
  const double* Qsg = ab ? Qbb : Qa;
  const int hr = ab ? ha : hb, hc = ab ? hb : ha;  // wanted half of the rows / columns of Y
  const double* Gin = f.Gbuf[R & 1];
  double* Qs = sm;
  double* Xs = sm + JS * TLD;
  double* Qt = sm + 2 * JS * TLD;
  if (part == 0) {
    for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
      const int i = e / JS, j = e % JS;
      Xs[i * TLD + j] = __ldcg(Gin + (int64_t)gidx(i, It, Jt) * n_pad + gidx(j, Is, Js));
    }
    return;
  }
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    const int i = e / JS, j = e % JS;
    Qs[i * TLD + j] = __ldcg(Qsg + e);
    Qt[i * TLD + j] = __ldcg(Qtg + e);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    double acc1[2][1][2];
    const int wm = (warp >> 2) * 16, wn = hc * JB + (warp & 3) * 8;
    tile_mma_at<2, 1>(Xs, false, Qs, acc1, wm, wn);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        Xs[(wm + 8 * i + (lane >> 2)) * TLD + wn + 2 * (lane & 3) + h] = acc1[i][0][h];
    __syncthreads();
  }
  double acc[1][1][2];
  const int wm = hr * JB + (warp >> 2) * 8, wn = hc * JB + (warp & 3) * 8;
  tile_mma_at<1, 1>(Qt, true, Xs, acc, wm, wn);
  __syncthreads();  // tiles consumed: S / Q alias them
  for (int e = threadIdx.x; e < JS * JS; e += blockDim.x) {
    const int i = e / JS, j = e % JS;
    Q[i * JLD + j] = (i == j) ? 1.0 : 0.0;
    if (i < JB && j < JB)
      S[i * JLD + j] = __ldcg(Sa + (ha * JB + i) * JS + ha * JB + j);
    else if (i >= JB && j >= JB)
      S[i * JLD + j] = __ldcg(Sbb + (hb * JB + i - JB) * JS + hb * JB + j - JB);
  }
  // Y rows belong to slot min(ta, tb)'s pair: to I when ab, else to J
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int m = wm + (lane >> 2), n = wn + 2 * (lane & 3) + h;
    const int li = ab ? (m & 31) : (n & 31), lj = ab ? (n & 31) : (m & 31);
    S[li * JLD + JB + lj] = acc[0][0][h];
    S[(JB + lj) * JLD + li] = acc[0][0][h];
  }
}

__global__ void __launch_bounds__(JT) jacobi_flow_k(FlowArgs f) {
  extern __shared__ double sm[];
  __shared__ InnerShared sh;
  const JacArgs& a = f.a;
  const double abs_tol =
      fmax(fmax(a.abs_scale * a.d_maxdiag[0], a.abs_floor ? a.abs_floor[0] : 0.0), 1e-300);
  const int nrounds = a.nb - 1, npairs = a.npairs;
  const int nsym = npairs * (npairs + 1) / 2;
  const int nitems = nsym + a.v_tiles * npairs;
  const bool is_inner = (int)blockIdx.x < npairs;
  const int ntile = (int)gridDim.x - npairs, tile_id = (int)blockIdx.x - npairs;
  unsigned int* c_inner = f.cnt;
  unsigned int* c_tile = f.cnt + 1;
  int R = 0, sweep = 0;
  for (; sweep < a.max_sweeps; sweep++) {
    JacArgs as = a;
    as.stats = a.stats + sweep;
    as.offmax = a.offmax + sweep;
    for (int r = 0; r < nrounds; r++, R++) {
      if (is_inner) {
        if (R >= 2) flow_wait(c_tile, (unsigned)((R - 1) * nitems));  // G_{R-2} complete
        flow_stage_input(f, R, blockIdx.x, r, sm, 0);
        flow_wait(c_inner, (unsigned)(R * npairs));                   // Q, S of round R - 1
        flow_stage_input(f, R, blockIdx.x, r, sm, 1);
        const int64_t qoff = (int64_t)(R & 1) * npairs * JS * JS;
        inner_solve(as, blockIdx.x, r, sm, sh, abs_tol, -1.0, true, a.Qb + qoff, a.Sb + qoff);
        flow_signal(c_inner, 1);
      } else {
        flow_wait(c_inner, (unsigned)((R + 1) * npairs));  // Q, S of round R
        flow_wait(c_tile, (unsigned)(R * nitems));         // G_{R-1}, V complete
        int done = 0;
        for (int w = tile_id; w < nitems; w += ntile, done++) {
          if (w < nsym) {
            int t = 0, rem = w;
            while (rem >= npairs - t) {
              rem -= npairs - t;
              t++;
            }
            flow_sym_tile(f, R, t, t + rem, r, sm);
          } else {
            const int v = w - nsym;
            flow_col_tile(f, R, (v % a.v_tiles) * JS, v / a.v_tiles, r, sm);
          }
        }
        flow_signal(c_tile, (unsigned)done);
      }
    }
    // the sweep's rotation statistics are complete once all of its pair solves are
    flow_wait(c_inner, (unsigned)(R * npairs));
    const int rot = __ldcg(a.stats + sweep);
    const double om = __longlong_as_double((long long)__ldcg(a.offmax + sweep));
    if (rot == 0 || om <= a.stop_rel) {
      sweep++;
      break;
    }
  }
  if (blockIdx.x == 0) {
    flow_wait(c_tile, (unsigned)(R * nitems));
    const double* G = f.Gbuf[(R + 1) & 1];  // G_{R-1}
    for (int i = threadIdx.x; i < a.n_pad; i += blockDim.x)
      f.diag_out[i] = __ldcg(G + (int64_t)i * a.n_pad + i);
    if (threadIdx.x == 0) a.sweeps_out[0] = sweep;
  }
}

// G <- A zero-padded to n_pad x n_pad; V <- V0 (mv x n, zero-padded to mv_pad x n_pad) or, when
// V0 is null, the identity.
__global__ void embed_k(int n, int n_pad, const double* __restrict__ A, double* __restrict__ G,
                        double* __restrict__ V, const double* __restrict__ V0, int mv, int mv_pad) {
  const int64_t nn = (int64_t)n_pad * n_pad, nv = (int64_t)mv_pad * n_pad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nn || e < nv;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n_pad), j = (int)(e % n_pad);
    if (e < nn) G[e] = (i < n && j < n) ? A[(int64_t)i * n + j] : 0.0;
    if (e < nv)
      V[e] = V0 ? ((i < mv && j < n) ? V0[(int64_t)i * n + j] : 0.0) : ((i == j) ? 1.0 : 0.0);
  }
}

// Sort eigenvalues descending (stable by index) and permute eigenvector columns.
// (diag[i * dstride]: the eigenvalues — G's diagonal with dstride = n_pad + 1, or a packed copy)
__global__ void eig_sort_k(int n, int n_pad, int mv, const double* __restrict__ diag,
                           int64_t dstride, const double* __restrict__ Vp,
                           double* __restrict__ lam, double* __restrict__ Vout) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double li = diag[i * dstride];
    int rank = 0;
    for (int j = 0; j < n; j++) {
      double lj = diag[j * dstride];
      rank += (lj > li) || (lj == li && j < i);
    }
    lam[rank] = li;
    for (int k = 0; k < mv; k++) Vout[(int64_t)k * n + rank] = Vp[(int64_t)k * n_pad + i];
  }
}

__global__ void max_abs_diag_k(int n, const double* A, double* out) {
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(A[(int64_t)i * n + i]));
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

}  // namespace

int tk_jacobi_eig(tk_ctx* ctx, int n, double* A, double* lam, double* V, double abs_tol_scale,
                  double rel_tol, int max_sweeps, int* sweeps_out, double* lskip_dev,
                  double rs_tol, int64_t rs_rmax, const double* abs_floor_dev, const double* V0,
                  int mv, double stop_rel) {
  if (n <= 0) return TK_OK;
  const int n_pad = ((n + JS - 1) / JS) * JS;
  if (!V0) mv = n;
  const int mv_pad = ((mv + JS - 1) / JS) * JS;
  const int nb = n_pad / JB;
  const int npairs = nb / 2;
  // dataflow schedule (jacobi_flow_k): >= 2 pairs, no cluster skip, room for the pair CTAs plus
  // at least as many tile CTAs
  const bool flow = ctx->jacobi_flow && npairs >= 2 && !lskip_dev && 2 * npairs <= ctx->num_sms;
  DevBuf Gp, Vp, Qb, Sb, scr, G2, dg;
  TK_TRY(Gp.get(ctx, (size_t)n_pad * n_pad));
  TK_TRY(Vp.get(ctx, (size_t)std::max(mv_pad, n_pad) * n_pad));
  TK_TRY(Qb.get(ctx, (size_t)(flow ? 2 : 1) * npairs * JS * JS));
  TK_TRY(Sb.get(ctx, (size_t)(flow ? 2 : 1) * npairs * JS * JS));
  if (flow) {
    TK_TRY(G2.get(ctx, (size_t)n_pad * n_pad));
    TK_TRY(dg.get(ctx, (size_t)n_pad + 1));  // diagonal + the two counters
  }
  TK_TRY(scr.get(ctx, 2 + 2 * (size_t)max_sweeps));
  double* d_maxdiag = scr.p;
  unsigned long long* offmax = (unsigned long long*)(scr.p + 1);
  int* stats = (int*)(scr.p + 1 + max_sweeps);
  int* d_sweeps = stats + max_sweeps;
  TK_TRY(tk_zero(ctx, scr.p + 1, 1, sizeof(double) * (1 + 2 * (int64_t)max_sweeps),
                 sizeof(double) * (1 + 2 * (int64_t)max_sweeps)));
  const int prof_id = tk_prof_begin(ctx, "jacobi", 0.0, 0.0);
  max_abs_diag_k<<<1, 256, 0, ctx->stream>>>(n, A, d_maxdiag);
  TK_LAUNCH_CHECK(ctx);
  {
    int64_t nn = (int64_t)std::max(mv_pad, n_pad) * n_pad;
    int g = (int)std::min<int64_t>((nn + 255) / 256, 8LL * ctx->num_sms);
    embed_k<<<g, 256, 0, ctx->stream>>>(n, n_pad, A, Gp.p, Vp.p, V0, mv, mv_pad);
    TK_LAUNCH_CHECK(ctx);
  }
  const size_t smem = 3 * (size_t)JS * TLD * sizeof(double);
  static int max_grid = -1;
  if (max_grid < 0) {
    cudaFuncSetAttribute(jacobi_persistent_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_persistent_k, JT, smem);
    max_grid = std::max(1, per_sm) * ctx->num_sms;
  }
  JacArgs a;
  a.n_pad = n_pad;
  a.v_tiles = mv_pad / JS;
  a.nb = nb;
  a.npairs = npairs;
  a.G = Gp.p;
  a.V = Vp.p;
  a.Qb = Qb.p;
  a.Sb = Sb.p;
  a.d_maxdiag = d_maxdiag;
  a.abs_floor = abs_floor_dev;
  a.abs_scale = abs_tol_scale;
  a.rel_tol = rel_tol;
  a.lskip = lskip_dev;
  a.lskip_io = lskip_dev;
  a.n = n;
  a.rs_tol = 0.0;  // (rank-aware skip: off)
  a.rs_rmax = rs_rmax;
  a.offmax = offmax;
  // relative mode: a sweep whose largest applied relative coupling is <= 1e-10 leaves
  // couplings of O(1e-20) behind (quadratic convergence): stop after it
  a.stop_rel = rel_tol > 0.0 ? (stop_rel > 0.0 ? stop_rel : 1e-10) : 0.0;
  a.tstamp = nullptr;
  a.max_inner = (npairs == 1) ? 60 : 1;
  a.max_sweeps = max_sweeps;
  a.stats = stats;
  a.sweeps_out = d_sweeps;
  const int rtiles = n_pad / JS;
  int grid = std::min(max_grid, std::max(npairs, (rtiles + mv_pad / JS) * npairs));
  grid = std::min(grid, ctx->num_sms);
  int coop = grid > 1 ? 1 : 0;
  if (flow) {
    static int flow_grid = -1;
    if (flow_grid < 0) {
      cudaFuncSetAttribute(jacobi_flow_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_flow_k, JT, smem);
      flow_grid = std::max(1, per_sm) * ctx->num_sms;
    }
    FlowArgs f;
    f.a = a;
    f.Gbuf[0] = G2.p;
    f.Gbuf[1] = Gp.p;  // embed_k wrote the input here
    f.cnt = (unsigned int*)(dg.p + n_pad);
    f.diag_out = dg.p;
    TK_TRY(tk_zero(ctx, dg.p + n_pad, 1, sizeof(double), sizeof(double)));
    const int nitems = npairs * (npairs + 1) / 2 + a.v_tiles * npairs;
    int fgrid = std::min(std::min(flow_grid, ctx->num_sms), npairs + nitems);
    void* args[] = {&f};
    TK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((void*)jacobi_flow_k, dim3(fgrid), dim3(JT),
                                                 args, smem, ctx->stream));
    ctx->launches++;
  } else if (coop) {
    void* args[] = {&a, &coop};
    TK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((void*)jacobi_persistent_k, dim3(grid),
                                                 dim3(JT), args, smem, ctx->stream));
    ctx->launches++;
  } else {
    jacobi_persistent_k<<<1, JT, smem, ctx->stream>>>(a, 0);
    TK_LAUNCH_CHECK(ctx);
  }
  int sg = (int)std::min<int64_t>((n + 127) / 128, 4LL * ctx->num_sms);
  eig_sort_k<<<sg, 128, 0, ctx->stream>>>(n, n_pad, mv, flow ? dg.p : Gp.p,
                                          flow ? 1 : (int64_t)n_pad + 1, Vp.p, lam, V);
  TK_LAUNCH_CHECK(ctx);
  tk_prof_end(ctx, prof_id);
  if (sweeps_out) {
    TK_TRY(tk_read_host(ctx, ctx->stream, sweeps_out, d_sweeps, sizeof(int)));
  }
  return TK_OK;
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_k_jacobi_k() {}
const void* tk_anchor_k_jacobi() { return (const void*)tk_anchor_k_jacobi_k; }
