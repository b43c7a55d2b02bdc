// Symmetric eigen-decomposition by parallel cyclic two-sided Jacobi (fp64, on device).
//
// Used for the small R x R Gram matrices of the rounding: pass 1
// needs an ORTHOGONAL eigenbasis to absolute accuracy, pass 2 needs eigenvalues with
// RELATIVE accuracy on a graded matrix — Jacobi with the relative skip test
// |a_pq| <= rel * sqrt(|a_pp a_qq|) provides that (Demmel-Veselic), which tridiagonal QR
// does not.
//
// Parallel ordering: round-robin tournament, n_e = n + (n odd) players, n_e - 1 rounds per
// sweep, n_e/2 disjoint pairs per round.  One round = every CTA recomputes the n_e/2
// rotations from the current matrix into shared memory, then updates its share of the
// n x n elements  A' = J^T A J  (double buffered) and of V' = V J (in place, one thread per
// (row, pair)).  One grid-wide barrier per round (cooperative launch); a single-CTA launch
// uses __syncthreads instead.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "ttk_internal.h"

namespace cg = cooperative_groups;

namespace {

constexpr int JT = 256;

__device__ __forceinline__ int rr_player(int pos, int r, int ne) {
  return pos == 0 ? 0 : 1 + (pos - 1 + r) % (ne - 1);
}
__device__ __forceinline__ int rr_pos(int player, int r, int ne) {
  if (player == 0) return 0;
  int m = ne - 1;
  return 1 + (((player - 1 - r) % m) + m) % m;
}

struct Rot {
  double c, s, t;
  int active;
};

__device__ __forceinline__ void grid_barrier(bool coop) {
  if (coop)
    cg::this_grid().sync();
  else
    __syncthreads();
}

// partner of row i in round r (or -1), and whether i is the "p" (smaller) element
__device__ __forceinline__ int partner_of(int i, int r, int n, int ne) {
  int pos = rr_pos(i, r, ne);
  int pp = ne - 1 - pos;
  int j = rr_player(pp, r, ne);
  return j < n ? j : -1;
}

__global__ void __launch_bounds__(JT) jacobi_kernel(int n, double* A0, double* A1, double* V,
                                                    const double* d_maxdiag, double abs_scale,
                                                    double rel_tol,
                                                    int max_sweeps, int* counters, int* sweeps_out,
                                                    int coop) {
  extern __shared__ double jsm[];
  const int ne = n + (n & 1);
  const int npairs = ne / 2;
  double* rc = jsm;               // c per pair-slot
  double* rs = jsm + npairs;      // s
  double* rt = jsm + 2 * npairs;  // t
  __shared__ int block_active;

  const double abs_tol = fmax(abs_scale * d_maxdiag[0], 1e-300);
  double* Acur = A0;
  double* Anext = A1;
  const int64_t nn = (int64_t)n * n;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  int sweep = 0;
  for (; sweep < max_sweeps; sweep++) {
    for (int r = 0; r < ne - 1; r++) {
      // (1) rotations for all pairs of this round, from Acur (redundantly per CTA)
      if (threadIdx.x == 0) block_active = 0;
      __syncthreads();
      int local_active = 0;
      for (int t = threadIdx.x; t < npairs; t += blockDim.x) {
        int a = rr_player(t, r, ne), b = rr_player(ne - 1 - t, r, ne);
        int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0, tt = 0.0;
        if (q < n) {
          double app = Acur[(int64_t)p * n + p], aqq = Acur[(int64_t)q * n + q];
          double apq = Acur[(int64_t)p * n + q];
          double thr = fmax(abs_tol, rel_tol * sqrt(fabs(app * aqq)));
          if (fabs(apq) > thr) {
            double theta = (aqq - app) / (2.0 * apq);
            double at = fabs(theta);
            if (at > 1e150) {
              tt = 0.5 / theta;
            } else {
              tt = 1.0 / (at + sqrt(1.0 + at * at));
              if (theta < 0) tt = -tt;
            }
            c = 1.0 / sqrt(1.0 + tt * tt);
            s = tt * c;
            local_active++;
          }
        }
        rc[t] = c;
        rs[t] = s;
        rt[t] = tt;
      }
      if (local_active) atomicAdd(&block_active, local_active);
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x == 0 && block_active)
        atomicAdd(&counters[sweep], block_active);

      // (2) A' = J^T A J, element-wise from Acur into Anext
      for (int64_t e = gtid; e < nn; e += gstride) {
        int i = (int)(e / n), j = (int)(e % n);
        int pi = partner_of(i, r, n, ne), pj = partner_of(j, r, n, ne);
        // coefficient of column i of J on i (ci) and on its partner (di)
        double ci = 1.0, di = 0.0, cj = 1.0, dj = 0.0;
        int ti = -1, tj = -1;
        if (pi >= 0) {
          int pos = rr_pos(i, r, ne);
          ti = pos < npairs ? pos : ne - 1 - pos;
          ci = rc[ti];
          di = (i < pi) ? -rs[ti] : rs[ti];
        }
        if (pj >= 0) {
          int pos = rr_pos(j, r, ne);
          tj = pos < npairs ? pos : ne - 1 - pos;
          cj = rc[tj];
          dj = (j < pj) ? -rs[tj] : rs[tj];
        }
        double v;
        if (ti >= 0 && ti == tj && rs[ti] != 0.0) {
          // inside an active pair's 2x2 block: Rutishauser's formulas
          if (i == j) {
            int p = min(i, pi), q = max(i, pi);
            double apq = Acur[(int64_t)p * n + q];
            v = Acur[e] + ((i == p) ? -rt[ti] * apq : rt[ti] * apq);
          } else {
            v = 0.0;
          }
        } else {
          v = ci * cj * Acur[e];
          if (dj != 0.0) v += ci * dj * Acur[(int64_t)i * n + pj];
          if (di != 0.0) v += di * cj * Acur[(int64_t)pi * n + j];
          if (di != 0.0 && dj != 0.0) v += di * dj * Acur[(int64_t)pi * n + pj];
        }
        Anext[e] = v;
      }
      // (3) V' = V J  (one thread per (row k, pair t))
      const int64_t nv = (int64_t)n * npairs;
      for (int64_t e = gtid; e < nv; e += gstride) {
        int k = (int)(e / npairs), t = (int)(e % npairs);
        double s = rs[t];
        if (s == 0.0) continue;
        int a = rr_player(t, r, ne), b = rr_player(ne - 1 - t, r, ne);
        int p = min(a, b), q = max(a, b);
        double c = rc[t];
        double vp = V[(int64_t)k * n + p], vq = V[(int64_t)k * n + q];
        V[(int64_t)k * n + p] = c * vp - s * vq;
        V[(int64_t)k * n + q] = s * vp + c * vq;
      }
      grid_barrier(coop);
      double* tmp = Acur;
      Acur = Anext;
      Anext = tmp;
    }
    // sweep finished: all CTAs read the counter (written before the last barrier)
    int act = *((volatile int*)&counters[sweep]);
    if (act == 0) {
      sweep++;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sweeps_out[0] = sweep;
    sweeps_out[1] = (Acur == A0) ? 0 : 1;  // which buffer holds the result
  }
}

// Sort eigenvalues descending (stable by index) and permute eigenvector columns.
__global__ void eig_sort(int n, const double* __restrict__ A0, const double* __restrict__ A1,
                         const int* __restrict__ which, const double* __restrict__ Vin,
                         double* __restrict__ lam, double* __restrict__ Vout) {
  const double* A = which[1] ? A1 : A0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double li = A[(int64_t)i * n + i];
    int rank = 0;
    for (int j = 0; j < n; j++) {
      double lj = A[(int64_t)j * n + j];
      rank += (lj > li) || (lj == li && j < i);
    }
    lam[rank] = li;
    for (int k = 0; k < n; k++) Vout[(int64_t)k * n + rank] = Vin[(int64_t)k * n + i];
  }
}

__global__ void max_abs_diag(int n, const double* A, double* out) {
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
                  double rel_tol, int max_sweeps, int* sweeps_out) {
  if (n <= 0) return TK_OK;
  if (n == 1) {
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(lam, A, sizeof(double), cudaMemcpyDeviceToDevice,
                                     ctx->stream));
    return tk_eye(ctx, V, 1);
  }
  const int ne = n + (n & 1);
  DevBuf A1, Vtmp, scratch;
  TK_TRY(A1.get(ctx, (size_t)n * n));
  TK_TRY(Vtmp.get(ctx, (size_t)n * n));
  // scratch: [maxdiag (1 double)] [counters: max_sweeps ints] [sweeps_out: 2 ints]
  TK_TRY(scratch.get(ctx, 1 + (size_t)(max_sweeps + 2 + 1) / 2 + 1));
  double* d_maxdiag = scratch.p;
  int* counters = (int*)(scratch.p + 1);
  int* info = counters + max_sweeps;
  TK_CUDA_TRY(ctx, cudaMemsetAsync(counters, 0, (max_sweeps + 2) * sizeof(int), ctx->stream));
  TK_TRY(tk_eye(ctx, Vtmp.p, n));
  // absolute skip threshold = abs_tol_scale * max|a_ii|, read on device by the kernel
  max_abs_diag<<<1, 256, 0, ctx->stream>>>(n, A, d_maxdiag);
  TK_LAUNCH_CHECK(ctx);

  const int npairs = ne / 2;
  size_t smem = 3 * (size_t)npairs * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t work = (int64_t)n * n;
  int grid = 1;
  if (n > 96) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, JT, smem);
    per_sm = std::max(1, std::min(per_sm, 2));
    grid = (int)std::min<int64_t>((work + JT * 4 - 1) / (JT * 4), (int64_t)per_sm * ctx->num_sms);
    grid = std::max(grid, 1);
  }
  int coop = grid > 1 ? 1 : 0;
  double* a0 = A;
  double* a1 = A1.p;
  double* vv = Vtmp.p;
  if (coop) {
    void* args[] = {&n, &a0, &a1, &vv, &d_maxdiag, &abs_tol_scale, &rel_tol, &max_sweeps, &counters, &info, &coop};
    TK_CUDA_TRY(ctx, cudaLaunchCooperativeKernel((void*)jacobi_kernel, dim3(grid), dim3(JT), args,
                                                 smem, ctx->stream));
    ctx->launches++;
  } else {
    jacobi_kernel<<<1, JT, smem, ctx->stream>>>(n, a0, a1, vv, d_maxdiag, abs_tol_scale, rel_tol, max_sweeps,
                                                counters, info, 0);
    TK_LAUNCH_CHECK(ctx);
  }
  int sg = (int)std::min<int64_t>((n + 127) / 128, 4LL * ctx->num_sms);
  eig_sort<<<sg, 128, 0, ctx->stream>>>(n, a0, a1, info, vv, lam, V);
  TK_LAUNCH_CHECK(ctx);
  if (sweeps_out) {
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->pinned, info, sizeof(int), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    *sweeps_out = *(int*)ctx->pinned;
  }
  return TK_OK;
}
