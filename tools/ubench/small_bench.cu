// Stand-alone timing of the latency-bound internal routines of libttk (Householder pass 1,
// pivoted Cholesky, triangular inverse, Jacobi) on synthetic SPD matrices, through the library's
// own (non-ABI, internal) entry points.  Diagnostic only.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_1906_06785_b200/csrc/ttk_internal.h"

static int g_rank = -1;  // < n: exact rank of the synthetic H (eigenvalues beyond it are 0)
static void spd(int n, std::vector<double>& H, double span) {
  // H = B diag(d) B^T with B random, d graded over `span` decades
  std::vector<double> B((size_t)n * n);
  srand(1);
  for (auto& v : B) v = (rand() / (double)RAND_MAX) - 0.5;
  H.assign((size_t)n * n, 0.0);
  std::vector<double> d(n);
  for (int i = 0; i < n; i++) d[i] = (g_rank >= 0 && i >= g_rank) ? 0.0 : pow(10.0, -span * i / n);
  for (int i = 0; i < n; i++)
    for (int j = 0; j <= i; j++) {
      double s = 0;
      for (int k = 0; k < n; k++) s += B[(size_t)i * n + k] * d[k] * B[(size_t)j * n + k];
      H[(size_t)i * n + j] = H[(size_t)j * n + i] = s;
    }
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 896;
  const char* what = argc > 2 ? argv[2] : "qr";
  if (argc > 3) g_rank = atoi(argv[3]);
  if (!strcmp(what, "gemm") || !strcmp(what, "gram")) {
    // c4 bond-1 shapes: W = Y P (786432 x 640 x 896) and G_W = W^T W (sym)
    const int64_t M = 786432, K = 896, N = 640;
    tk_ctx* c2;
    cudaStream_t st2;
    cudaStreamCreate(&st2);
    tk_ctx_create(&c2, st2);
    double *Y, *P, *W, *G;
    cudaMalloc(&Y, sizeof(double) * M * K);
    cudaMalloc(&P, sizeof(double) * K * N);
    cudaMalloc(&W, sizeof(double) * M * N);
    cudaMalloc(&G, sizeof(double) * N * N);
    cudaMemset(Y, 0, sizeof(double) * M * K);
    cudaMemset(P, 0, sizeof(double) * K * N);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0, st2);
      if (!strcmp(what, "gemm"))
        tk_dgemm(c2, false, false, M, N, K, 1.0, Y, K, P, N, 0.0, W, N);
      else
        tk_dgemm(c2, true, false, N, N, M, 1.0, W, N, W, N, 0.0, G, N, true);
      cudaEventRecord(e1, st2);
      cudaStreamSynchronize(st2);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fl = !strcmp(what, "gemm") ? 2.0 * M * N * K : (double)N * (N + 1) * M;
      printf("%s %.3f ms  %.2f TF/s\n", what, ms, fl / ms / 1e9);
    }
    return 0;
  }
  if (!strcmp(what, "gemmsmall")) {
    // latency of the small DMMA GEMMs of the Cholesky trailing updates: sym n x n x 32, and a
    // plain n x n x 32 product, 200 back-to-back launches each (profiling off)
    tk_ctx* c2;
    cudaStream_t st2;
    cudaStreamCreate(&st2);
    tk_ctx_create(&c2, st2);
    double *A, *C;
    cudaMalloc(&A, sizeof(double) * 32 * n);
    cudaMalloc(&C, sizeof(double) * n * n);
    cudaMemset(A, 0, sizeof(double) * 32 * n);
    cudaMemset(C, 0, sizeof(double) * n * n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int sym = 1; sym >= 0; sym--) {
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(e0, st2);
        for (int i = 0; i < 200; i++)
          tk_dgemm(c2, true, false, n, n, 32, -1.0, A, n, A, n, 1.0, C, n, sym != 0);
        cudaEventRecord(e1, st2);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("gemm n=%d K=32 sym=%d: %.2f us per launch\n", n, sym, ms * 1e3 / 200);
      }
    }
    return 0;
  }
  tk_ctx* ctx;
  cudaStream_t st;
  cudaStreamCreate(&st);
  tk_ctx_create(&ctx, st);
  std::vector<double> H;
  spd(n, H, 12.0);
  double *dH, *dQ, *dR;
  int *piv, *state;
  cudaMalloc(&dH, sizeof(double) * n * n);
  cudaMalloc(&dQ, sizeof(double) * n * n);
  cudaMalloc(&dR, sizeof(double) * n * n);
  cudaMalloc(&piv, sizeof(double) * (n + 2) * 2);
  cudaMalloc(&state, sizeof(int) * (n + 2));
  cudaMemcpy(dH, H.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; rep++) {
    tk_ctx_profile(ctx, 1);
    cudaEventRecord(a, st);
    int rc = 0;
    if (!strcmp(what, "qr")) rc = tk_householder_q(ctx, n, dH, dQ);
    else if (!strcmp(what, "pchol")) rc = tk_pchol(ctx, n, dH, 1e-28, nullptr, dR, piv, state, true);
    else if (!strcmp(what, "jacobi")) {
      // pass-2-like relative Jacobi on the graded SPD matrix (destroys dR's copy of H)
      cudaMemcpyAsync(dR, dH, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st);
      cudaEventRecord(a, st);
      int sw = 0;
      rc = tk_jacobi_eig(ctx, n, dR, (double*)piv, dQ, 4.93e-32, 32 * 2.220446049250313e-16, 40, &sw);
      printf("  sweeps %d\n", sw);
    } else if (!strcmp(what, "triinv")) {
      tk_pchol(ctx, n, dH, 1e-28, nullptr, dR, piv, state, false);
      cudaEventRecord(a, st);
      rc = tk_tri_inv(ctx, n, dR, n, dQ, n);
    }
    cudaEventRecord(b, st);
    cudaStreamSynchronize(st);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s n=%d rc=%d total %.3f ms\n", what, n, rc, ms);
    if (rep == 2 && !strcmp(what, "triinv")) {
      // X R = I for the upper triangular R (unpivoted Cholesky factor of H), on the host
      std::vector<double> ro((size_t)n * n), xi((size_t)n * n);
      cudaMemcpy(ro.data(), dR, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      cudaMemcpy(xi.data(), dQ, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      double e = 0.0;
      for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
          double s2 = 0.0;
          for (int t = 0; t < n; t++) s2 += xi[(size_t)i * n + t] * ro[(size_t)t * n + j];
          e = std::max(e, fabs(s2 - (i == j ? 1.0 : 0.0)));
        }
      printf("   max |X R - I| = %.2e\n", e);
    }
    if (rep == 2 && !strcmp(what, "pchol")) {
      // reconstruction H ~ Ro^T Ro over the first k rows, on the host
      std::vector<double> ro((size_t)n * n);
      int st[2];
      cudaMemcpy(ro.data(), dR, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      cudaMemcpy(st, state, sizeof(st), cudaMemcpyDeviceToHost);
      const int k = st[0];
      double hn = 0.0, e = 0.0;
      for (double v : H) hn = std::max(hn, fabs(v));
      for (int i = 0; i < n; i++)
        for (int j = 0; j <= i; j++) {
          double s2 = 0.0;
          for (int t = 0; t < k; t++) s2 += ro[(size_t)t * n + i] * ro[(size_t)t * n + j];
          e = std::max(e, fabs(s2 - H[(size_t)i * n + j]));
        }
      printf("   rank %d  max |H - Ro^T Ro| / max|H| = %.2e\n", k, e / hn);
    }
    if (rep == 2 && !strcmp(what, "qr")) {
      // orthogonality of Q and the triangularity of Q^T H (first 64 columns), on the host
      std::vector<double> hq((size_t)n * n);
      cudaMemcpy(hq.data(), dQ, sizeof(double) * n * n, cudaMemcpyDeviceToHost);
      double eo = 0.0, et = 0.0;
      for (int i = 0; i < n; i++)
        for (int j = 0; j <= i; j++) {
          double s = 0.0;
          for (int k = 0; k < n; k++) s += hq[(size_t)k * n + i] * hq[(size_t)k * n + j];
          eo = std::max(eo, fabs(s - (i == j ? 1.0 : 0.0)));
        }
      double hn = 0.0;
      for (double v : H) hn = std::max(hn, fabs(v));
      for (int j = 0; j < std::min(n, 64); j++)
        for (int i = j + 1; i < n; i++) {  // (Q^T H)[i, j] for i > j must vanish
          double s = 0.0;
          for (int k = 0; k < n; k++) s += hq[(size_t)k * n + i] * H[(size_t)k * n + j];
          et = std::max(et, fabs(s) / hn);
        }
      printf("   max |Q^T Q - I| = %.2e   max |(Q^T H)_{i>j}| / max|H| = %.2e\n", eo, et);
      if (g_rank >= 0) {
        // range(H) inside span(Q[:, :rank]): rows >= rank of Q^T H vanish
        double el = 0.0;
        for (int i = g_rank; i < n; i++)
          for (int j = 0; j < n; j++) {
            double s2 = 0.0;
            for (int k = 0; k < n; k++) s2 += hq[(size_t)k * n + i] * H[(size_t)k * n + j];
            el = std::max(el, fabs(s2) / hn);
          }
        printf("   rank %d: max |(Q^T H)_{i>=rank}| / max|H| = %.2e\n", g_rank, el);
      }
    }
    if (rep == 2) {
      static char buf[1 << 22];
      tk_ctx_profile_dump(ctx, buf, sizeof(buf));
      // aggregate by category
      std::vector<std::pair<std::string, std::pair<double, int>>> agg;
      char* line = strtok(buf, "\n");
      while (line) {
        char cat[128];
        double t;
        if (sscanf(line, "%127s %lf", cat, &t) == 2) {
          bool f = false;
          for (auto& x : agg)
            if (x.first == cat) { x.second.first += t; x.second.second++; f = true; }
          if (!f) agg.push_back({cat, {t, 1}});
        }
        line = strtok(nullptr, "\n");
      }
      for (auto& x : agg) printf("   %-16s n=%5d %8.3f ms\n", x.first.c_str(), x.second.second, x.second.first);
    }
  }
  return 0;
}
