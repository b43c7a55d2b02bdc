// libttk C ABI: context, operator descriptor, apply, round, dot, axpby, GMRES cycle.
// See include/ttk.h for the contract of every entry point and DESIGN.md for the algorithms.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "ttk_internal.h"

static const double kEps = 2.220446049250313e-16;

// ============================================================================ memory
int tk_alloc(tk_ctx* ctx, void** p, size_t bytes) {
  cudaError_t e = cudaMallocAsync(p, bytes, ctx->stream);
  if (e != cudaSuccess) {
    ctx->err = std::string("cudaMallocAsync(") + std::to_string(bytes) + "): " +
               cudaGetErrorString(e);
    *p = nullptr;
    return TK_ECUDA;
  }
  ctx->live[*p] = bytes;
  ctx->live_bytes += bytes;
  ctx->high_bytes = std::max(ctx->high_bytes, ctx->live_bytes);
  return TK_OK;
}
void tk_free(tk_ctx* ctx, void* p) {
  if (!p) return;
  auto it = ctx->live.find(p);
  if (it != ctx->live.end()) {
    ctx->live_bytes -= it->second;
    ctx->live.erase(it);
  }
  cudaFreeAsync(p, ctx->stream);
}

// Called at the end of the top-level entry points.  Once the scratch high-water mark of a call
// is known, the stream-ordered pool is given one free block of 1.5x that size: later calls
// carve their scratch from it instead of mapping new memory mid-call (a pool growth costs
// hundreds of ms at the c4 sizes and showed up as step-time outliers, profiles/r01/README.md).
static void pool_settle(tk_ctx* ctx) {
  if (ctx->high_bytes <= ctx->reserved_for) return;
  const size_t want = ctx->high_bytes + ctx->high_bytes / 2;
  void* p = nullptr;
  if (cudaMallocAsync(&p, want, ctx->stream) == cudaSuccess) cudaFreeAsync(p, ctx->stream);
  cudaGetLastError();  // a failed reservation is not an error: growth just stays on demand
  ctx->reserved_for = want;
}

// ============================================================================ context
extern "C" const char* tk_version(void) { return "ttk 0.1 (sm_100a, fp64 DMMA)"; }

extern "C" int tk_ctx_create(tk_ctx** out, void* stream) {
  if (!out) return TK_EARG;
  auto* ctx = new tk_ctx();
  ctx->stream = (cudaStream_t)stream;
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e == cudaSuccess)
    e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (e == cudaSuccess) {
    // keep freed pool memory cached: stream-ordered allocations stay cheap in steady state
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    ctx->pinned_bytes = 1 << 16;
    e = cudaHostAlloc(&ctx->pinned, ctx->pinned_bytes, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ctx->pinned_dev, ctx->pinned, 0);
  }
  if (e != cudaSuccess) {
    delete ctx;
    return TK_ECUDA;
  }
  *out = ctx;
  return TK_OK;
}

int tk_aux_streams(tk_ctx* ctx, size_t n_events) {
  // highest priority, like ctx->crit: the QR's trailing updates are on the critical path and
  // must not queue behind the side stream's big GEMMs
  // (one level below ctx->crit, whose QR panel kernels need a whole SM: when an SM frees up,
  // the pending panel is dispatched before more update blocks)
  int lo = 0, hi = 0;
  TK_CUDA_TRY(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  const int pr = hi >= lo ? hi : hi + 1;
  for (auto& s : ctx->aux)
    if (!s) TK_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, pr));
  while (ctx->fork_ev.size() < n_events) {
    cudaEvent_t e;
    TK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->fork_ev.push_back(e);
  }
  return TK_OK;
}

CritScope::CritScope(tk_ctx* ctx) : c(ctx) {
  if (!ctx->crit) {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return;
    if (cudaStreamCreateWithPriority(&ctx->crit, cudaStreamNonBlocking, hi) != cudaSuccess) {
      ctx->crit = nullptr;
      return;
    }
    for (auto& e : ctx->crit_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  user = ctx->stream;
  cudaEventRecord(ctx->crit_ev[0], user);
  cudaStreamWaitEvent(ctx->crit, ctx->crit_ev[0], 0);
  ctx->stream = ctx->crit;
  on = true;
}
CritScope::~CritScope() {
  if (!on) return;
  cudaEventRecord(c->crit_ev[1], c->crit);
  cudaStreamWaitEvent(user, c->crit_ev[1], 0);
  c->stream = user;
}

int tk_side_fork(tk_ctx* ctx) {
  if (!ctx->side) {
    int lo = 0, hi = 0;
    TK_CUDA_TRY(ctx, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TK_CUDA_TRY(ctx, cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, lo));
    for (auto& e : ctx->side_ev) TK_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  TK_CUDA_TRY(ctx, cudaEventRecord(ctx->side_ev[0], ctx->stream));
  TK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->side, ctx->side_ev[0], 0));
  return TK_OK;
}
int tk_side_join(tk_ctx* ctx) {
  if (!ctx->side) return TK_OK;
  TK_CUDA_TRY(ctx, cudaEventRecord(ctx->side_ev[1], ctx->side));
  TK_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->side_ev[1], 0));
  return TK_OK;
}

extern "C" int tk_ctx_destroy(tk_ctx* ctx) {
  if (!ctx) return TK_OK;
  tk_async_destroy(ctx);
  tk_gate_destroy(ctx);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
    for (auto e : ctx->side_ev) cudaEventDestroy(e);
  }
  if (ctx->crit) {
    cudaStreamSynchronize(ctx->crit);
    cudaStreamDestroy(ctx->crit);
    for (auto e : ctx->crit_ev) cudaEventDestroy(e);
  }
  for (auto& s : ctx->aux)
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  for (auto e : ctx->fork_ev) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  delete ctx;
  return TK_OK;
}

// ============================================================================ profiling
int tk_prof_begin(tk_ctx* ctx, const char* cat, double flops, double bytes) {
  if (!ctx->prof) return -1;
  // level 1: the event pairs of the many small launches of the latency-bound chain cost ~2 ms
  // per c4 step; only the heavy launches are recorded
  if (ctx->prof_level < 2 && flops < 1e8 && bytes < 1e8) return -1;
  while (ctx->ev_pool.size() < ctx->ev_used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    ctx->ev_pool.push_back(e);
  }
  ProfRec r{cat, flops, bytes, ctx->ev_pool[ctx->ev_used], ctx->ev_pool[ctx->ev_used + 1]};
  ctx->ev_used += 2;
  cudaEventRecord(r.a, ctx->stream);
  ctx->recs.push_back(r);
  return (int)ctx->recs.size() - 1;
}
void tk_prof_end(tk_ctx* ctx, int id) {
  if (id < 0 || !ctx->prof) return;
  cudaEventRecord(ctx->recs[id].b, ctx->stream);
}

extern "C" int tk_ctx_profile(tk_ctx* ctx, int enable) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx) return TK_EARG;
  ctx->prof = enable != 0;
  ctx->prof_level = enable == 2 ? 1 : 2;  // enable == 2: heavy launches only
  ctx->prof_timeline = enable == 3;       // enable == 3: every launch + start offsets
  if (enable) {
    ctx->recs.clear();
    ctx->ev_used = 0;
  }
  return TK_OK;
}

extern "C" int tk_ctx_profile_dump(tk_ctx* ctx, char* buf, size_t len) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx) return TK_EARG;
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  std::string out;
  const bool tl = ctx->prof_timeline;
  for (auto& r : ctx->recs) {
    float ms = 0.f, t0 = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    char line[256];
    if (tl) {  // timeline: start offset (ms) from the first record, for overlap analysis
      cudaEventElapsedTime(&t0, ctx->recs[0].a, r.a);
      snprintf(line, sizeof(line), "%s %.6f %.6e %.6e %.4f\n", r.cat, ms, r.flops, r.bytes, t0);
    } else {
      snprintf(line, sizeof(line), "%s %.6f %.6e %.6e\n", r.cat, ms, r.flops, r.bytes);
    }
    out += line;
  }
  if (buf && len) {
    size_t n = std::min(len - 1, out.size());
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int)ctx->recs.size();
}

// Upper bound of the library scratch (stream-ordered pool) of one tk_round on ranks (R1, R2), or
// of one tk_apply_round whose grown ranks are (R1, R2): every temporary of round_impl,
// orth_rows, the bond SVDs and the fused apply counted as if live at once (they are not), in
// doubles, plus 1 MiB for small buffers.  tests/test_gpu_parity.py checks it against the
// measured high-water mark.
extern "C" size_t tk_round_workspace_bytes(int64_t n_x, int64_t n_xi, int64_t n_t, int64_t R1,
                                           int64_t R2) {
  if (n_x < 1 || n_xi < 1 || n_t < 1 || R1 < 1 || R2 < 1) return 0;
  const double k3 = (double)std::min(n_t, R2), N2 = (double)n_xi * k3;
  const double k2 = std::min((double)R1, N2), r1 = R1, r2 = R2, nx = n_x, nt = n_t;
  const double time_core = 12 * r2 * r2 + 4 * nt * r2 + 2 * nt * nt;
  const double mid = 3 * r1 * N2 + 12 * r1 * r1 + 4 * N2 * r1;
  const double bond1 = nx * k2 + r1 * r1 + 3 * r1 * k2 + 16 * k2 * k2 + 2 * k2 * N2;
  const double bond2 = 3 * k2 * n_xi * k3 + 16 * k3 * k3 + 2 * k2 * k3;
  const double fused = 2 * r1 * n_xi * r2 + r1 * r1;
  return (size_t)(8.0 * (time_core + mid + bond1 + bond2 + fused)) + ((size_t)1 << 20);
}

// Reserve `bytes` of the stream-ordered pool for the context's scratch (the pool keeps freed
// memory, so later calls up to that size map nothing new; cf. pool_settle).  Synchronous.
extern "C" int tk_ctx_reserve(tk_ctx* ctx, size_t bytes) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx) return TK_EARG;
  if (bytes <= ctx->reserved_for) return TK_OK;
  void* p = nullptr;
  TK_CUDA_TRY(ctx, cudaMallocAsync(&p, bytes, ctx->stream));
  TK_CUDA_TRY(ctx, cudaFreeAsync(p, ctx->stream));
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  ctx->reserved_for = bytes;
  return TK_OK;
}

// High-water mark of the library scratch since creation or the last reset (bytes).
extern "C" int64_t tk_ctx_scratch_high_water(tk_ctx* ctx, int reset) {
  if (!ctx) return 0;
  if (ctx->async) tk_async_drain(ctx);
  const int64_t h = (int64_t)ctx->high_bytes;
  if (reset) ctx->high_bytes = ctx->live_bytes;
  return h;
}

extern "C" const char* tk_last_error(const tk_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }
extern "C" int64_t tk_ctx_launch_count(const tk_ctx* ctx) { return ctx ? ctx->launches : 0; }

extern "C" int tk_ctx_set_gemm_feed(tk_ctx* ctx, int mode) {
  if (!ctx) return TK_EARG;
  if (mode != 0 && mode != 1) {
    ctx->err = "tk_ctx_set_gemm_feed: mode must be 0 (cp.async) or 1 (TMA)";
    return TK_EARG;
  }
  TK_ASYNC_GUARD(ctx);
  ctx->gemm_tma = mode;
  return TK_OK;
}

extern "C" int tk_ctx_set_jacobi_schedule(tk_ctx* ctx, int mode) {
  if (!ctx) return TK_EARG;
  if (mode != 0 && mode != 1) {
    ctx->err = "tk_ctx_set_jacobi_schedule: mode must be 0 (grid barriers) or 1 (dataflow)";
    return TK_EARG;
  }
  TK_ASYNC_GUARD(ctx);
  ctx->jacobi_flow = mode;
  return TK_OK;
}

extern "C" int tk_gemm(tk_ctx* ctx, int transA, int transB, int64_t M, int64_t N, int64_t K,
                       double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                       double beta, double* C, int64_t ldc, int sym) {
  if (!ctx) return TK_EARG;
  if (M < 0 || N < 0 || K < 0 || ((!A || !B) && K > 0 && M > 0 && N > 0) || (!C && M > 0 && N > 0)) {
    ctx->err = "tk_gemm: null pointer or negative size";
    return TK_EARG;
  }
  TK_ASYNC_GUARD(ctx);
  const char* tag0 = ctx->tag;
  ctx->tag = "tk_gemm";
  const int st = tk_dgemm(ctx, transA != 0, transB != 0, M, N, K, alpha, A, lda, B, ldb, beta, C,
                          ldc, sym != 0);
  ctx->tag = tag0;
  return st;
}

static int sync_read(tk_ctx* ctx, void* host, const void* dev, size_t bytes);
int tk_sync_read(tk_ctx* ctx, void* host, const void* dev, size_t bytes) {
  return sync_read(ctx, host, dev, bytes);
}
namespace {
// bytes -> the mapped pinned buffer (8-byte words when aligned)
__global__ void read_to_host_k(const void* __restrict__ src, void* dst, size_t n) {
  if ((((uintptr_t)src | (uintptr_t)dst) & 7) == 0) {
    const size_t w = n / 8;
    for (size_t i = threadIdx.x; i < w; i += blockDim.x)
      ((volatile unsigned long long*)dst)[i] = ((const unsigned long long*)src)[i];
    for (size_t i = 8 * w + threadIdx.x; i < n; i += blockDim.x)
      ((volatile unsigned char*)dst)[i] = ((const unsigned char*)src)[i];
  } else {
    for (size_t i = threadIdx.x; i < n; i += blockDim.x)
      ((volatile unsigned char*)dst)[i] = ((const unsigned char*)src)[i];
  }
}
}  // namespace

int tk_read_host(tk_ctx* ctx, cudaStream_t stream, void* host, const void* dev, size_t bytes) {
  if (bytes == 0) return TK_OK;
  if (bytes > ctx->pinned_bytes || !ctx->pinned_dev) {
    TK_CUDA_TRY(ctx, cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream));
    TK_CUDA_TRY(ctx, cudaStreamSynchronize(stream));
    return TK_OK;
  }
  read_to_host_k<<<1, 256, 0, stream>>>(dev, ctx->pinned_dev, bytes);
  TK_LAUNCH_CHECK(ctx);
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(stream));
  memcpy(host, ctx->pinned, bytes);
  return TK_OK;
}

static int sync_read(tk_ctx* ctx, void* host, const void* dev, size_t bytes) {
  return tk_read_host(ctx, ctx->stream, host, dev, bytes);
}

// ============================================================================ operator
// Column-merged records of T spatial factors for spmm_merged_k (k_apply.cu): per row, the
// distinct columns over all T in ascending order, each as col | (mask << 32), and the values
// in (column, factor) order.  Duplicate (column, factor) entries are summed.  Returns false
// (no records) when a row has more than 32 distinct columns (then the per-term kernel runs).
static bool merge_records(int T, int64_t n_x, const int32_t* const* K_rowptr,
                          const int32_t* const* K_col, const double* const* K_val,
                          std::vector<int64_t>& recptr, std::vector<int64_t>& rec) {
  if (n_x >= ((int64_t)1 << 31) || T > 32) return false;
  // merged per-row lists (distinct columns with term masks, values in (column, term) order)
  std::vector<int64_t> wptr(n_x + 1, 0), vptr(n_x + 1, 0), words, vals_all;
  int64_t tot = 0;
  for (int k = 0; k < T; k++) tot += K_rowptr[k][n_x];
  words.reserve(tot / 2 + 16);
  vals_all.reserve(tot);
  struct E {
    int32_t c;
    int32_t k;
    double v;
  };
  std::vector<E> ents;
  for (int64_t i = 0; i < n_x; i++) {
    ents.clear();
    for (int k = 0; k < T; k++)
      for (int32_t p = K_rowptr[k][i]; p < K_rowptr[k][i + 1]; p++)
        ents.push_back({K_col[k][p], k, K_val[k][p]});
    std::stable_sort(ents.begin(), ents.end(), [](const E& a, const E& b) {
      return a.c != b.c ? a.c < b.c : a.k < b.k;
    });
    size_t q = 0;
    while (q < ents.size()) {
      const int32_t c = ents[q].c;
      uint32_t mask = 0;
      while (q < ents.size() && ents[q].c == c) {
        const int k = ents[q].k;
        double v = 0.0;
        while (q < ents.size() && ents[q].c == c && ents[q].k == k) v += ents[q++].v;
        mask |= 1u << k;
        int64_t b;
        memcpy(&b, &v, sizeof(b));
        vals_all.push_back(b);
      }
      words.push_back((int64_t)(uint32_t)c | ((int64_t)mask << 32));
    }
    wptr[i + 1] = (int64_t)words.size();
    vptr[i + 1] = (int64_t)vals_all.size();
    // the merged kernel keeps one row's distinct columns in one warp's lanes
    if (wptr[i + 1] - wptr[i] > 32) return false;
  }
  // processing order: breadth-first over the symmetrised merged pattern (Cuthill-McKee, no
  // reversal), each component from its lowest unvisited row
  std::vector<int32_t> order;
  order.reserve(n_x);
  {
    std::vector<int64_t> tptr(n_x + 1, 0);
    for (int64_t i = 0; i < n_x; i++)
      for (int64_t w = wptr[i]; w < wptr[i + 1]; w++) tptr[(words[w] & 0xffffffffLL) + 1]++;
    for (int64_t i = 0; i < n_x; i++) tptr[i + 1] += tptr[i];
    std::vector<int32_t> tcol(tptr[n_x]);
    std::vector<int64_t> fill(tptr.begin(), tptr.end() - 1);
    for (int64_t i = 0; i < n_x; i++)
      for (int64_t w = wptr[i]; w < wptr[i + 1]; w++)
        tcol[fill[words[w] & 0xffffffffLL]++] = (int32_t)i;
    std::vector<char> seen(n_x, 0);
    std::vector<int32_t> nb;
    for (int64_t s0 = 0; s0 < n_x; s0++) {
      if (seen[s0]) continue;
      seen[s0] = 1;
      size_t head = order.size();
      order.push_back((int32_t)s0);
      while (head < order.size()) {
        const int32_t u = order[head++];
        nb.clear();
        for (int64_t w = wptr[u]; w < wptr[u + 1]; w++) nb.push_back((int32_t)(words[w] & 0xffffffffLL));
        for (int64_t t = tptr[u]; t < tptr[u + 1]; t++) nb.push_back(tcol[t]);
        std::sort(nb.begin(), nb.end());
        for (int32_t v : nb)
          if (!seen[v]) {
            seen[v] = 1;
            order.push_back(v);
          }
      }
    }
  }
  recptr.assign(n_x + 1, 0);
  rec.clear();
  rec.reserve(words.size() + vals_all.size() + n_x + 16);
  for (int64_t pos = 0; pos < n_x; pos++) {
    const int64_t i = order[pos];
    const int64_t gn = wptr[i + 1] - wptr[i];
    rec.push_back(i | (gn << 32));
    rec.insert(rec.end(), words.begin() + wptr[i], words.begin() + wptr[i + 1]);
    rec.insert(rec.end(), vals_all.begin() + vptr[i], vals_all.begin() + vptr[i + 1]);
    recptr[pos + 1] = (int64_t)rec.size();
  }
  return true;
}

void tk_free_chunks(std::vector<SpmmChunk>& cs) {
  for (auto& c : cs) {
    if (!c.owns) continue;
    cudaFree(c.recptr);
    cudaFree(c.rec);
    cudaFree(c.tk);
    cudaFree(c.tg);
    cudaFree(c.tc);
  }
  cs.clear();
}

// Device copy of a chunk's term list (terms tk[t] of local group tg[t] with coefficient
// tc[t]), stored sorted by group with the group offsets goff (ng + 1) in c.tg.
int tk_upload_terms(tk_ctx* ctx, SpmmChunk& c, const std::vector<int>& tk,
                    const std::vector<int>& tg, const std::vector<double>& tc) {
  auto up = [&](void** d, const void* h, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(d, b ? b : 8));
    if (b) TK_CUDA_TRY(ctx, cudaMemcpy(*d, h, b, cudaMemcpyHostToDevice));
    return TK_OK;
  };
  c.nterm = (int)tk.size();
  std::vector<int> ord(tk.size());
  for (size_t t = 0; t < ord.size(); t++) ord[t] = (int)t;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return tg[a] < tg[b]; });
  std::vector<int> sk(tk.size()), goff(c.ng + 1, 0);
  std::vector<double> sc(tk.size());
  for (size_t t = 0; t < ord.size(); t++) {
    sk[t] = tk[ord[t]];
    sc[t] = tc[ord[t]];
    goff[tg[ord[t]] + 1]++;
  }
  for (int g = 0; g < c.ng; g++) goff[g + 1] += goff[g];
  c.h_tk = sk;
  c.h_goff = goff;
  c.h_tc = sc;
  TK_TRY(up((void**)&c.tk, sk.data(), sizeof(int) * sk.size()));
  TK_TRY(up((void**)&c.tg, goff.data(), sizeof(int) * goff.size()));
  TK_TRY(up((void**)&c.tc, sc.data(), sizeof(double) * sc.size()));
  return TK_OK;
}

// Device copy of one chunk: its records and its term list (tk_upload_terms).
int tk_upload_chunk(tk_ctx* ctx, SpmmChunk& c, const std::vector<int64_t>& recptr,
                    const std::vector<int64_t>& rec, const std::vector<int>& tk,
                    const std::vector<int>& tg, const std::vector<double>& tc) {
  auto up = [&](void** d, const void* h, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(d, b ? b : 8));
    if (b) TK_CUDA_TRY(ctx, cudaMemcpy(*d, h, b, cudaMemcpyHostToDevice));
    return TK_OK;
  };
  TK_TRY(up((void**)&c.recptr, recptr.data(), sizeof(int64_t) * recptr.size()));
  TK_TRY(up((void**)&c.rec, rec.data(), sizeof(int64_t) * rec.size()));
  return tk_upload_terms(ctx, c, tk, tg, tc);
}

// Merged-SpMM chunks over the factors reps[0..G) (each the representative CSR of one output
// column block g, coefficient 1, identity output map: chunk c writes blocks c*16 ..), in chunks
// of <= 16.  Leaves `out` empty when some merged row exceeds 32 distinct columns.
static int build_chunks(tk_ctx* ctx, std::vector<SpmmChunk>& out, int64_t n_x,
                        const int32_t* const* K_rowptr, const int32_t* const* K_col,
                        const double* const* K_val, const std::vector<int>& reps) {
  const int G = (int)reps.size();
  for (int g0 = 0; g0 < G; g0 += 16) {
    const int ng = std::min(16, G - g0);
    std::vector<const int32_t*> rp, cl;
    std::vector<const double*> vl;
    for (int g = g0; g < g0 + ng; g++) {
      rp.push_back(K_rowptr[reps[g]]);
      cl.push_back(K_col[reps[g]]);
      vl.push_back(K_val[reps[g]]);
    }
    std::vector<int64_t> recptr, rec;
    if (!merge_records(ng, n_x, rp.data(), cl.data(), vl.data(), recptr, rec)) {
      tk_free_chunks(out);
      return TK_OK;
    }
    std::vector<int> tk, tg;
    std::vector<double> tc;
    for (int g = 0; g < ng; g++) {
      tk.push_back(g0 + g);
      tg.push_back(g);
      tc.push_back(1.0);
    }
    SpmmChunk c;
    c.g0 = g0;
    c.ng = ng;
    c.ident = true;
    c.k0 = g0;
    out.push_back(c);
    TK_TRY(tk_upload_chunk(ctx, out.back(), recptr, rec, tk, tg, tc));
  }
  return TK_OK;
}

// Spatial groups: term k joins the group of an earlier representative j when K_k has the same
// CSR structure and K_k = c K_j BITWISE (c = val_k[0] / val_j[0], every entry checked in fp64),
// e.g. the KL terms nu_l L with nu_l = nu_0 2^-l.  Then K_k U1 = c (K_j U1) exactly.
static void find_groups(int T, int64_t n_x, const int32_t* const* rp, const int32_t* const* cl,
                        const double* const* vl, std::vector<int>& group,
                        std::vector<double>& coef, std::vector<int>& reps) {
  group.assign(T, -1);
  coef.assign(T, 1.0);
  reps.clear();
  for (int k = 0; k < T; k++) {
    const int64_t nnz = rp[k][n_x];
    for (size_t g = 0; g < reps.size() && group[k] < 0; g++) {
      const int j = reps[g];
      if (rp[j][n_x] != nnz || nnz == 0) continue;
      if (memcmp(rp[j], rp[k], sizeof(int32_t) * (n_x + 1)) != 0) continue;
      if (memcmp(cl[j], cl[k], sizeof(int32_t) * nnz) != 0) continue;
      if (vl[j][0] == 0.0) continue;
      const double c = vl[k][0] / vl[j][0];
      bool ok = std::isfinite(c) && c != 0.0;
      for (int64_t e = 0; ok && e < nnz; e++) ok = (c * vl[j][e] == vl[k][e]);
      if (ok) {
        group[k] = (int)g;
        coef[k] = c;
      }
    }
    if (group[k] < 0) {
      group[k] = (int)reps.size();
      reps.push_back(k);
    }
  }
}

extern "C" int tk_op_create(tk_ctx* ctx, tk_op** out, int T, int64_t n_x, int64_t n_xi,
                            int64_t n_t, const int32_t* const* K_rowptr,
                            const int32_t* const* K_col, const double* const* K_val,
                            const double* const* G, const int* T_kl, const int* T_ku,
                            const double* const* T_band) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out) return TK_EARG;
  if (T < 1 || n_x < 1 || n_xi < 1 || n_t < 1) {
    ctx->err = "tk_op_create: T, n_x, n_xi, n_t must be >= 1";
    return TK_EARG;
  }
  if (n_x >= INT32_MAX) {
    ctx->err = "tk_op_create: n_x must fit int32 CSR indices";
    return TK_EARG;
  }
  // (partial device allocations are freed by tk_op_destroy on every error return)
  struct OpDel {
    void operator()(tk_op* o) const { tk_op_destroy(o); }
  };
  std::unique_ptr<tk_op, OpDel> op(new tk_op());
  op->ctx = ctx;
  op->T = T;
  op->n_x = n_x;
  op->n_xi = n_xi;
  op->n_t = n_t;
  std::vector<int64_t> nnz_off(T + 1, 0), band_off(T + 1, 0);
  for (int k = 0; k < T; k++) {
    if (!K_rowptr[k] || !G[k] || !T_band[k] || T_kl[k] < 0 || T_ku[k] < 0) {
      ctx->err = "tk_op_create: null descriptor array or negative band width";
      return TK_EARG;
    }
    int64_t nnz = K_rowptr[k][n_x] - K_rowptr[k][0];
    if (K_rowptr[k][0] != 0 || nnz < 0) {
      ctx->err = "tk_op_create: rowptr must start at 0 and be non-decreasing";
      return TK_EARG;
    }
    // every row pointer in [rowptr[i], nnz]: the merged-record builder and the SpMM kernels
    // index col/val by them
    for (int64_t i = 0; i < n_x; i++)
      if (K_rowptr[k][i + 1] < K_rowptr[k][i] || K_rowptr[k][i + 1] > nnz) {
        ctx->err = "tk_op_create: rowptr must be non-decreasing and <= nnz";
        return TK_EARG;
      }
    if (nnz > 0 && (!K_col[k] || !K_val[k])) {
      ctx->err = "tk_op_create: null CSR arrays";
      return TK_EARG;
    }
    for (int64_t c = 0; c < nnz; c++)
      if (K_col[k][c] < 0 || K_col[k][c] >= n_x) {
        ctx->err = "tk_op_create: CSR column index out of range";
        return TK_EARG;
      }
    nnz_off[k + 1] = nnz_off[k] + nnz;
    band_off[k + 1] = band_off[k] + (int64_t)(T_kl[k] + T_ku[k] + 1) * n_t;
    op->max_kl = std::max(op->max_kl, T_kl[k]);
    op->max_ku = std::max(op->max_ku, T_ku[k]);
    op->h_nnz.push_back(nnz);
  }
  const int64_t tot = nnz_off[T];
  auto dmal = [&](void** p, size_t b) -> int {
    TK_CUDA_TRY(ctx, cudaMalloc(p, b ? b : 8));
    return TK_OK;
  };
  TK_TRY(dmal((void**)&op->rowptr, sizeof(int32_t) * T * (n_x + 1)));
  TK_TRY(dmal((void**)&op->col, sizeof(int32_t) * tot));
  TK_TRY(dmal((void**)&op->val, sizeof(double) * tot));
  TK_TRY(dmal((void**)&op->nnz_off, sizeof(int64_t) * (T + 1)));
  TK_TRY(dmal((void**)&op->G, sizeof(double) * T * n_xi * n_xi));
  TK_TRY(dmal((void**)&op->band_kl, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->band_ku, sizeof(int) * T));
  TK_TRY(dmal((void**)&op->band_off, sizeof(int64_t) * (T + 1)));
  TK_TRY(dmal((void**)&op->band, sizeof(double) * band_off[T]));
  for (int k = 0; k < T; k++) {
    TK_CUDA_TRY(ctx, cudaMemcpy(op->rowptr + (int64_t)k * (n_x + 1), K_rowptr[k],
                                sizeof(int32_t) * (n_x + 1), cudaMemcpyHostToDevice));
    int64_t nnz = nnz_off[k + 1] - nnz_off[k];
    if (nnz) {
      TK_CUDA_TRY(ctx, cudaMemcpy(op->col + nnz_off[k], K_col[k], sizeof(int32_t) * nnz,
                                  cudaMemcpyHostToDevice));
      TK_CUDA_TRY(ctx, cudaMemcpy(op->val + nnz_off[k], K_val[k], sizeof(double) * nnz,
                                  cudaMemcpyHostToDevice));
    }
    TK_CUDA_TRY(ctx, cudaMemcpy(op->G + (int64_t)k * n_xi * n_xi, G[k],
                                sizeof(double) * n_xi * n_xi, cudaMemcpyHostToDevice));
    TK_CUDA_TRY(ctx, cudaMemcpy(op->band + band_off[k], T_band[k],
                                sizeof(double) * (band_off[k + 1] - band_off[k]),
                                cudaMemcpyHostToDevice));
  }
  TK_CUDA_TRY(ctx, cudaMemcpy(op->nnz_off, nnz_off.data(), sizeof(int64_t) * (T + 1),
                              cudaMemcpyHostToDevice));
  {
    // merged-SpMM chunks over the terms (the literal output), and over the spatial groups
    // (bitwise-proportional K_k) for the optional group-space output
    std::vector<int> group, reps, all(T);
    std::vector<double> coef;
    for (int k = 0; k < T; k++) all[k] = k;
    TK_TRY(build_chunks(ctx, op->chunks, n_x, K_rowptr, K_col, K_val, all));
    find_groups(T, n_x, K_rowptr, K_col, K_val, group, coef, reps);
    op->n_groups = (int)reps.size();
    if (op->n_groups < T && !op->chunks.empty())
      TK_TRY(build_chunks(ctx, op->gchunks, n_x, K_rowptr, K_col, K_val, reps));
    if (op->gchunks.empty()) op->n_groups = T;  // (no group-space output)
    TK_CUDA_TRY(ctx, cudaMalloc((void**)&op->d_group, sizeof(int) * T));
    TK_CUDA_TRY(ctx, cudaMalloc((void**)&op->d_coef, sizeof(double) * T));
    TK_CUDA_TRY(ctx, cudaMemcpy(op->d_group, group.data(), sizeof(int) * T,
                                cudaMemcpyHostToDevice));
    TK_CUDA_TRY(ctx, cudaMemcpy(op->d_coef, coef.data(), sizeof(double) * T,
                                cudaMemcpyHostToDevice));
  }
  TK_CUDA_TRY(ctx, cudaMemcpy(op->band_kl, T_kl, sizeof(int) * T, cudaMemcpyHostToDevice));
  TK_CUDA_TRY(ctx, cudaMemcpy(op->band_ku, T_ku, sizeof(int) * T, cudaMemcpyHostToDevice));
  TK_CUDA_TRY(ctx, cudaMemcpy(op->band_off, band_off.data(), sizeof(int64_t) * (T + 1),
                              cudaMemcpyHostToDevice));
  *out = op.release();
  return TK_OK;
}

extern "C" int tk_op_destroy(tk_op* op) {
  { tk_ctx* _gc = op ? op->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  if (!op) return TK_OK;
  cudaFree(op->rowptr);
  cudaFree(op->col);
  cudaFree(op->val);
  cudaFree(op->nnz_off);
  cudaFree(op->G);
  cudaFree(op->band_kl);
  cudaFree(op->band_ku);
  cudaFree(op->band_off);
  cudaFree(op->band);
  tk_free_chunks(op->gchunks);
  tk_free_chunks(op->chunks);
  cudaFree(op->d_group);
  cudaFree(op->d_coef);
  delete op;
  return TK_OK;
}
extern "C" int tk_op_terms(const tk_op* op) { return op ? op->T : 0; }
extern "C" int tk_op_set_spmm_kernel(tk_op* op, int kernel) {
  { tk_ctx* _gc = op ? op->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  if (!op || kernel < 0 || kernel > 1) return TK_EARG;
  if (kernel == 1 && !op->rowptr) return TK_EARG;  // (no per-term CSR: merged only)
  if (kernel == 0 && op->chunks.empty()) return 0;
  op->spmm_perterm = kernel == 1;
  return op->chunks.empty() ? 0 : 1 - (int)op->spmm_perterm;
}
extern "C" int tk_op_group_space(tk_op* op, int enable) {
  { tk_ctx* _gc = op ? op->ctx : nullptr; TK_ASYNC_GUARD(_gc); }
  if (!op) return TK_EARG;
  op->group_space = enable != 0 && op->n_groups < op->T && !op->gchunks.empty();
  return op->n_groups;
}

// ============================================================================ validation
static int check_tt(tk_ctx* ctx, const tk_tt* x, const char* who) {
  if (!x || !x->U1 || !x->U2 || !x->U3) {
    ctx->err = std::string(who) + ": null TT or core pointer";
    return TK_EARG;
  }
  if (x->n_x < 1 || x->n_xi < 1 || x->n_t < 1 || x->r1 < 1 || x->r2 < 1) {
    ctx->err = std::string(who) + ": mode sizes and ranks must be >= 1";
    return TK_EARG;
  }
  if (x->r1 > x->cap1 || x->r2 > x->cap2) {
    ctx->err = std::string(who) + ": rank exceeds capacity";
    return TK_ECAP;
  }
  return TK_OK;
}

// ============================================================================ apply
// The space and time cores of y = A x: Y1 = [K_k U1]_k (SpMM), Y3 = [U3 T_k^T]_k (band).
// side: the SpMM runs on the side stream (forked here; the caller joins before it reads Y1)
static int apply_space_time(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y,
                            bool side = false, bool grouped = false) {
  const int64_t R2 = op->T * x->r2;
  const int64_t R1 = (grouped ? op->n_groups : op->T) * x->r1;  // columns the SpMM writes
  if (side) TK_TRY(tk_side_fork(ctx));
  {
    std::unique_ptr<OnSide> on;
    if (side) on.reset(new OnSide(ctx));
    // algorithmic bytes: read U1 once, write Y1 once, read the CSR (12 B/nnz + rowptr)
    double nnz = 0;
    for (auto v : op->h_nnz) nnz += (double)v;
    if (grouped) nnz *= (double)op->n_groups / op->T;  // (approximate: group representatives)
    double bytes = 8.0 * x->n_x * x->r1 + 8.0 * x->n_x * R1 + 12.0 * nnz +
                   4.0 * (grouped ? op->n_groups : op->T) * (x->n_x + 1);
    int id = tk_prof_begin(ctx, grouped ? "spmm_grouped" : "spmm_multi", 2.0 * nnz * x->r1,
                           bytes);
    TK_TRY(tk_launch_spmm_multi(ctx, op, (int)x->r1, x->U1, y->U1, grouped));
    tk_prof_end(ctx, id);
  }
  {
    int id = tk_prof_begin(ctx, "time_apply", 0.0, 8.0 * (R2 + x->r2) * x->n_t);
    TK_TRY(tk_launch_time_apply(ctx, op, (int)x->r2, x->U3, y->U3));
    tk_prof_end(ctx, id);
  }
  return TK_OK;
}

extern "C" int tk_apply_op(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !op) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_apply_op(x)"));
  if (!y || !y->U1 || !y->U2 || !y->U3) {
    ctx->err = "tk_apply_op: null output TT";
    return TK_EARG;
  }
  if (x->n_x != op->n_x || x->n_xi != op->n_xi || x->n_t != op->n_t || y->n_x != op->n_x ||
      y->n_xi != op->n_xi || y->n_t != op->n_t) {
    ctx->err = "tk_apply_op: mode sizes differ from the operator's";
    return TK_ESHAPE;
  }
  const int64_t R1 = op->T * x->r1, R2 = op->T * x->r2;
  if (R1 > y->cap1 || R2 > y->cap2) {
    ctx->err = "tk_apply_op: output capacity < (T r1, T r2)";
    return TK_ECAP;
  }
  TK_TRY(apply_space_time(ctx, op, x, y));
  {
    double bytes = 8.0 * (R1 * x->n_xi * R2 + x->r1 * x->n_xi * x->r2);
    int id = tk_prof_begin(ctx, "stoch_apply", 2.0 * op->T * x->r1 * x->n_xi * x->n_xi * x->r2,
                           bytes);
    TK_TRY(tk_launch_stoch_apply(ctx, op, (int)x->r1, (int)x->r2, x->U2, y->U2));
    tk_prof_end(ctx, id);
  }
  y->r1 = R1;
  y->r2 = R2;
  return TK_OK;
}

// ============================================================================ rounding
namespace {

struct EigOpts {
  double abs_scale, rel;
};
// Pass 2 needs relative accuracy: skip when |g_pq| <= 32 eps sqrt(g_pp g_qq) (second-order
// effect on the eigenvalues: ~1e-29).

// Pass 1: an exactly orthogonal basis V of R^n whose leading columns follow the dominant
// eigenvectors of the Gram G: Q of the Householder QR of G (one orthogonal-iteration step;
// direct, O(n^3) on DMMA).  lam is unused (kept for the call sites' buffer shape).
int pass1_basis(tk_ctx* ctx, int n, const double* G, double* /*lam*/, double* V) {
  return tk_householder_q(ctx, n, G, V);
}
const EigOpts kPass2{kEps * kEps, 32 * kEps};
const int kMaxSweeps = 40;
const int64_t kOrth3MinRank = 128;  // orth_rows on the time core from this grown rank on ...
const int64_t kOrth3MinNt = 128;    // ... when n_t is at least this (R2 >= n_t case)
const double kDropThr = 64.0 * kEps;         // numerical-dimension threshold of orth_rows

// A (R x N, row-major, ld N) = L (R x k) * Q (k x N, orthonormal rows) with Q stored
// transposed as Qc (N x k).  Two-pass Gram-Jacobi on B = A^T.
// Outputs are allocated here.  Returns k via *k_out (host; blocks).
int orth_rows(tk_ctx* ctx, int64_t R, int64_t N, const double* A, DevBuf& L, DevBuf& Qc,
              int64_t* k_out) {
  TagScope tag(ctx, "orth_rows");
  DevBuf G, V, W, GW, lam, V2, sig, scr, tmp;
  TK_TRY(G.get(ctx, R * R));
  TK_TRY(V.get(ctx, R * R));
  TK_TRY(lam.get(ctx, R));
  // pass 1: G = A A^T, orthogonal eigenbasis V
  TK_TRY(tk_dgemm(ctx, false, true, R, R, N, 1.0, A, N, A, N, 0.0, G.p, R, true));
  TK_TRY(pass1_basis(ctx, (int)R, G.p, lam.p, V.p));
  // W = A^T V  (N x R)
  TK_TRY(W.get(ctx, N * R));
  TK_TRY(tk_dgemm(ctx, true, false, N, R, R, 1.0, A, N, V.p, R, 0.0, W.p, R));
  TK_TRY(GW.get(ctx, R * R));
  TK_TRY(tk_dgemm(ctx, true, false, R, R, N, 1.0, W.p, R, W.p, R, 0.0, GW.p, R, true));
  if (R <= tk_pchol_max_n()) {
    // pass 2: CholeskyQR2 with diagonal pivoting on the graded W:
    //   W P1 = Q1 R1 (pivoted Cholesky of W^T W, truncated at the numerical rank k1),
    //   Q1 = W P1 R1^{-1},  Q1 = Q2 R2 (second pass: restores orthonormality to O(eps)),
    //   A = L Q2^T  with  L = V (Ro2 Ro1)^T  (Ro = R P^T in original column indexing).
    DevBuf Ro1, pv1, st1, R11, X1, S1, Q1, G2, Ro2, pv2, st2, R22, X2, M;
    TK_TRY(Ro1.get(ctx, R * R));
    TK_TRY(pv1.get(ctx, (R + 1) / 2));
    TK_TRY(st1.get(ctx, (R + 3) / 2));
    TK_TRY(tk_pchol(ctx, (int)R, GW.p, kDropThr * kDropThr, nullptr, Ro1.p, (int*)pv1.p,
                    (int*)st1.p));
    int k1 = 0;
    TK_TRY(sync_read(ctx, &k1, st1.p, sizeof(int)));
    if (k1 > 0) {
      TK_TRY(R11.get(ctx, (int64_t)k1 * k1));
      TK_TRY(tk_gather_cols(ctx, k1, k1, Ro1.p, R, (const int*)pv1.p, R11.p));
      TK_TRY(X1.get(ctx, (int64_t)k1 * k1));
      TK_TRY(tk_tri_inv(ctx, k1, R11.p, k1, X1.p, k1));
      // Q1 = W[:, piv1[:k1]] R11^{-1}: gather W's pivot columns, then a triangular product
      TK_TRY(S1.get(ctx, N * k1));
      TK_TRY(tk_gather_cols(ctx, N, k1, W.p, R, (const int*)pv1.p, S1.p));
      W.release();
      TK_TRY(Q1.get(ctx, N * k1));
      TK_TRY(tk_dgemm(ctx, false, false, N, k1, k1, 1.0, S1.p, k1, X1.p, k1, 0.0, Q1.p, k1, false,
                      true));
      S1.release();
      TK_TRY(G2.get(ctx, (int64_t)k1 * k1));
      TK_TRY(tk_dgemm(ctx, true, false, k1, k1, N, 1.0, Q1.p, k1, Q1.p, k1, 0.0, G2.p, k1, true));
      TK_TRY(Ro2.get(ctx, (int64_t)k1 * k1));
      TK_TRY(pv2.get(ctx, (k1 + 1) / 2));
      TK_TRY(st2.get(ctx, (k1 + 3) / 2));
      // no pivoting in the second pass: Q1's columns are already in the importance order of
      // the first pass, which L = V (Ro2 Ro1)^T inherits (bond 1's pass 1 relies on it)
      TK_TRY(tk_pchol(ctx, k1, G2.p, kDropThr * kDropThr, nullptr, Ro2.p, (int*)pv2.p,
                      (int*)st2.p, false));
      int k2 = 0;
      TK_TRY(sync_read(ctx, &k2, st2.p, sizeof(int)));
      if (k2 > 0) {
        TK_TRY(R22.get(ctx, (int64_t)k2 * k2));
        TK_TRY(tk_gather_cols(ctx, k2, k2, Ro2.p, k1, (const int*)pv2.p, R22.p));
        TK_TRY(X2.get(ctx, (int64_t)k2 * k2));
        TK_TRY(tk_tri_inv(ctx, k2, R22.p, k2, X2.p, k2));
        // unpivoted second pass: piv2 is the identity and R2^{-1} is upper triangular
        TK_TRY(Qc.get(ctx, N * k2));
        TK_TRY(tk_dgemm(ctx, false, false, N, k2, k2, 1.0, Q1.p, k1, X2.p, k2, 0.0, Qc.p, k2,
                        false, true));
        // M = Ro2[:k2] Ro1[:k1]  (k2 x R);  L = V M^T  (R x k2)
        TK_TRY(M.get(ctx, (int64_t)k2 * R));
        TK_TRY(tk_dgemm(ctx, false, false, k2, R, k1, 1.0, Ro2.p, k1, Ro1.p, R, 0.0, M.p, R));
        TK_TRY(L.get(ctx, R * k2));
        TK_TRY(tk_dgemm(ctx, false, true, R, k2, R, 1.0, V.p, R, M.p, R, 0.0, L.p, k2));
        *k_out = k2;
        return TK_OK;
      }
    }
    // zero (or numerically zero) A: the Jacobi path below handles it as before
    if (!W.p) {
      TK_TRY(W.get(ctx, N * R));
      TK_TRY(tk_dgemm(ctx, true, false, N, R, R, 1.0, A, N, V.p, R, 0.0, W.p, R));
    }
  }
  // pass 2: relative eigen-decomposition of GW down to the rounding-noise floor of W
  TK_TRY(V2.get(ctx, R * R));
  DevBuf floor;
  TK_TRY(floor.get(ctx, 1));
  TK_TRY(tk_noise_floor(ctx, G.p, R, 1.0, nullptr, 0, R, R, floor.p));
  TK_TRY(tk_jacobi_eig(ctx, (int)R, GW.p, lam.p, V2.p, kPass2.abs_scale, kPass2.rel,
                       kMaxSweeps, nullptr, nullptr, 0.0, 0, floor.p));
  TK_TRY(sig.get(ctx, R));
  TK_TRY(scr.get(ctx, 8));
  int* info = (int*)scr.p;
  double* dinfo = scr.p + 2;
  TK_TRY(tk_rank_select(ctx, (int)R, lam.p, sig.p, 0.0, nullptr, 0, kDropThr, info, dinfo));
  int hinfo[2];
  TK_TRY(sync_read(ctx, hinfo, info, sizeof(hinfo)));
  const int64_t k = hinfo[1];
  // Qc = W V2[:, :k] diag(1/sig)   (N x k)
  TK_TRY(tmp.get(ctx, R * k));
  TK_TRY(tk_col_scale(ctx, R, k, V2.p, R, tmp.p, k, sig.p, 1));
  TK_TRY(Qc.get(ctx, N * k));
  TK_TRY(tk_dgemm(ctx, false, false, N, k, R, 1.0, W.p, R, tmp.p, k, 0.0, Qc.p, k));
  // L = (V V2)[:, :k] diag(sig)   (R x k)
  DevBuf VV;
  TK_TRY(VV.get(ctx, R * k));
  TK_TRY(tk_dgemm(ctx, false, false, R, k, R, 1.0, V.p, R, V2.p, R, 0.0, VV.p, k));
  TK_TRY(L.get(ctx, R * k));
  TK_TRY(tk_col_scale(ctx, R, k, VV.p, k, L.p, k, sig.p, 0));
  *k_out = k;
  return TK_OK;
}

// SVD of Z = Y L (Y: M x R explicit, ld R; L: R x k, ld k; L == nullptr means identity with
// k = R) by two-pass Gram-Jacobi, first part: pass 1 basis V (k x k, orthogonal),
// W = Z V (M x k) and its Gram GW = W^T W.  pass2() finishes: lam (k, descending
// eigenvalues of GW = squared singular values of Z), V2 (k x k), Vt = V V2.
// floor (out, 1 device double): rounding-noise level of G_W entries for pass 2's skip test.
// Stride of the bond-1 pass-1 row sample (>= 8R rows, s <= 16).
static int64_t pass1_stride(int64_t M, int64_t R) {
  return std::max<int64_t>(1, std::min<int64_t>(16, M / (8 * R)));
}
// The sampled pass-1 Gram Y_s^T Y_s (R x R) of bond 1.
static int pass1_gram(tk_ctx* ctx, int64_t M, int64_t R, const double* Y, double* GY) {
  const int64_t s = pass1_stride(M, R);
  TagScope t(ctx, "bond1.gram_Y");
  return tk_dgemm(ctx, true, false, R, R, (M + s - 1) / s, 1.0, Y, R * s, Y, R * s, 0.0, GY, R,
                  true);
}

// gy_pre (nullable): the sampled Gram of Y, already computed (pass1_gram; tk_apply_round
// computes it on the side stream right after the SpMM).
int svd_two_pass(tk_ctx* ctx, int64_t M, int64_t R, const double* Y, const double* Lm,
                 int64_t k, DevBuf& W, DevBuf& GW, DevBuf& V, DevBuf& floor,
                 const double* gy_pre = nullptr) {
  DevBuf GY, GZ, T1, P, lam;
  TK_TRY(GZ.get(ctx, k * k));
  TK_TRY(floor.get(ctx, 1));
  int64_t s = 1;
  const double* gy = nullptr;
  TagScope tag0(ctx, Lm ? "bond1.small" : "bond2.small");
  if (Lm) {
    // Pass 1 only has to supply an orthogonal basis that roughly follows the dominant
    // directions (accuracy comes from pass 2 on the explicit W), so its Gram is taken over
    // a strided sample of >= 8R rows (every s-th spatial row, s <= 16): 1/s of the flops
    // with the same pass-2 convergence.
    s = pass1_stride(M, R);
    gy = gy_pre;
    if (!gy) {
      TK_TRY(GY.get(ctx, R * R));
      TK_TRY(pass1_gram(ctx, M, R, Y, GY.p));
      gy = GY.p;
    }
    TK_TRY(T1.get(ctx, R * k));
    TK_TRY(tk_dgemm(ctx, false, false, R, k, R, 1.0, gy, R, Lm, k, 0.0, T1.p, k));
    TK_TRY(tk_dgemm(ctx, true, false, k, k, R, 1.0, Lm, k, T1.p, k, 0.0, GZ.p, k));
    TK_TRY(tk_symmetrize(ctx, k, GZ.p));
  } else {
    TagScope t(ctx, "bond2.gram_C");
    TK_TRY(tk_dgemm(ctx, true, false, k, k, M, 1.0, Y, R, Y, R, 0.0, GZ.p, k, true));
  }
  TK_TRY(V.get(ctx, k * k));
  TK_TRY(lam.get(ctx, k));
  TK_TRY(pass1_basis(ctx, (int)k, GZ.p, lam.p, V.p));
  // W = Y (L V)
  const double* PV = V.p;
  if (Lm) {
    TK_TRY(P.get(ctx, R * k));
    TK_TRY(tk_dgemm(ctx, false, false, R, k, k, 1.0, Lm, k, V.p, k, 0.0, P.p, k));
    PV = P.p;
    // ||Y||_F^2 ~ s * trace(sampled Gram); P = L V
    TK_TRY(tk_noise_floor(ctx, gy, R, (double)s, P.p, R * k, R, k, floor.p));
  } else {
    TK_TRY(tk_noise_floor(ctx, GZ.p, k, 1.0, nullptr, 0, R, k, floor.p));  // P = V orthogonal
  }
  GZ.release();
  TK_TRY(W.get(ctx, M * k));
  {
    TagScope t(ctx, Lm ? "bond1.form_W" : "bond2.form_W");
    if (Lm) tk_gate_open(ctx);  // the DMMA-bound phase starts: open the copy-window gate
    TK_TRY(tk_dgemm(ctx, false, false, M, k, R, 1.0, Y, R, PV, k, 0.0, W.p, k));
  }
  TK_TRY(GW.get(ctx, k * k));
  {
    TagScope t(ctx, Lm ? "bond1.gram_W" : "bond2.gram_W");
    TK_TRY(tk_dgemm(ctx, true, false, k, k, M, 1.0, W.p, k, W.p, k, 0.0, GW.p, k, true));
  }
  return TK_OK;
}

// Q (rows x c) <- A (rows x c) R^{-1} with R from the unpivoted Cholesky of A^T A: one
// CholeskyQR pass (used twice on an already well-conditioned basis).
int cholqr_pass(tk_ctx* ctx, int64_t rows, int64_t c, const double* A, double* Q) {
  DevBuf G, Ro, pv, st, X;
  TK_TRY(G.get(ctx, c * c));
  TK_TRY(tk_dgemm(ctx, true, false, c, c, rows, 1.0, A, c, A, c, 0.0, G.p, c, true));
  TK_TRY(Ro.get(ctx, c * c));
  TK_TRY(pv.get(ctx, (c + 1) / 2));
  TK_TRY(st.get(ctx, (c + 3) / 2));
  TK_TRY(tk_pchol(ctx, (int)c, G.p, 0.0, nullptr, Ro.p, (int*)pv.p, (int*)st.p, false));
  int rank = 0;
  TK_TRY(sync_read(ctx, &rank, st.p, sizeof(int)));
  if (rank < c) {  // a Schur diagonal <= 1e-300 or NaN: R is singular, R^{-1} would spread inf
    ctx->err = "cholqr_pass: Gram not positive definite";
    return TK_ENUMERIC;
  }
  TK_TRY(X.get(ctx, c * c));
  TK_TRY(tk_tri_inv(ctx, (int)c, Ro.p, c, X.p, c));
  TK_TRY(tk_dgemm(ctx, false, false, rows, c, c, 1.0, A, c, X.p, c, 0.0, Q, c));
  return TK_OK;
}

// Pass 2 of a bond SVD, Cholesky-preconditioned:
//   (1) pivoted Cholesky P^T G_W P = R^T R, truncated at the noise floor (rank kc; the dropped
//       Schur trace `rem` stays in the tail);
//   (2) relative Jacobi on X = R R^T (graded by the pivoting: 6-9 sweeps instead of 14-16), its
//       rotations accumulated onto R^T, so the columns become sigma_i v_i (the eigenvectors of
//       G_W, one-sided-Jacobi style) and are normalised;
//   (3) that basis, made orthonormal by a CholeskyQR pass, turns G_W into Q^T G_W Q, which
//       one more relative Jacobi (1-3 sweeps) diagonalises to the pass-2 accuracy; V2 = Q V2'.
// lam (k): eigenvalues descending, then rem, then zeros; V2 (k x k): zero columns >= kc.
// Returns TK_EARG (caller falls back to plain Jacobi) when the preconditioner does not apply.
int pass2_chol(tk_ctx* ctx, int64_t k, const DevBuf& GW, const double* floor, DevBuf& lam,
               DevBuf& V2, int* rcap) {
  // small problems: one plain Jacobi (a single 64-wide block pair) is cheaper than two
  if (k > tk_pchol_max_n() || k <= 64) return TK_EARG;
  TagScope tag(ctx, "pass2_chol");
  DevBuf Ro, pv, st, rem, X, V0, Y, nrm, V1, Qv, T1, Gp, lam2, V2p;
  TK_TRY(Ro.get(ctx, k * k));
  TK_TRY(pv.get(ctx, (k + 1) / 2));
  TK_TRY(st.get(ctx, (k + 3) / 2));
  TK_TRY(rem.get(ctx, 1));
  TK_TRY(tk_pchol(ctx, (int)k, GW.p, 0.0, floor, Ro.p, (int*)pv.p, (int*)st.p, true, rem.p));
  int kc = 0;
  TK_TRY(sync_read(ctx, &kc, st.p, sizeof(int)));
  if (kc < 1) return TK_EARG;
  // (2) X = Ro Ro^T (kc x kc; column order of Ro is irrelevant), V0 = Ro^T (k x kc)
  TK_TRY(X.get(ctx, (int64_t)kc * kc));
  TK_TRY(tk_dgemm(ctx, false, true, kc, kc, k, 1.0, Ro.p, k, Ro.p, k, 0.0, X.p, kc, true));
  TK_TRY(V0.get(ctx, k * kc));
  TK_TRY(tk_transpose(ctx, kc, k, Ro.p, k, V0.p, kc));
  Ro.release();
  TK_TRY(lam2.get(ctx, kc));
  TK_TRY(Y.get(ctx, k * kc));
  // (the refinement Jacobi of step (3) restores the full accuracy, so this one may stop as
  // soon as the couplings are small: its last, confirming sweep is left to the refinement)
  const double stop1 = 1e-3;
  if (k >= kc + 64) {
    // accumulate the rotations into J (kc x kc) and apply them to V0 = R^T (k x kc) once: the
    // Jacobi's per-round tile phase then updates kc instead of k rows (fewer work items when
    // the factorisation truncated: c5 rounds k ~ 1300, kc ~ 1000)
    DevBuf J;
    TK_TRY(J.get(ctx, (int64_t)kc * kc));
    TK_TRY(tk_jacobi_eig(ctx, kc, X.p, lam2.p, J.p, kPass2.abs_scale, kPass2.rel, kMaxSweeps,
                         nullptr, nullptr, 0.0, 0, floor, nullptr, 0, stop1));
    TK_TRY(tk_dgemm(ctx, false, false, k, kc, kc, 1.0, V0.p, kc, J.p, kc, 0.0, Y.p, kc));
  } else {
    TK_TRY(tk_jacobi_eig(ctx, kc, X.p, lam2.p, Y.p, kPass2.abs_scale, kPass2.rel, kMaxSweeps,
                         nullptr, nullptr, 0.0, 0, floor, V0.p, (int)k, stop1));
  }
  TK_TRY(nrm.get(ctx, kc));
  TK_TRY(tk_col_norms(ctx, k, kc, Y.p, kc, nrm.p));
  TK_TRY(V1.get(ctx, k * kc));
  TK_TRY(tk_col_scale(ctx, k, kc, Y.p, kc, V1.p, kc, nrm.p, 1));
  // (3) orthonormal basis (columns in descending-sigma order), then the refinement Jacobi.  V1
  // is already orthonormal up to ~1e-12 on the kept columns and O(0.1) overall, so one
  // CholeskyQR pass gives O(eps) orthonormality (error ~ eps cond(V1)^2).
  TK_TRY(Qv.get(ctx, k * kc));
  if (cholqr_pass(ctx, k, kc, V1.p, Qv.p) != TK_OK) return TK_EARG;  // -> plain Jacobi
  TK_TRY(T1.get(ctx, k * kc));
  TK_TRY(tk_dgemm(ctx, false, false, k, kc, k, 1.0, GW.p, k, Qv.p, kc, 0.0, T1.p, kc));
  TK_TRY(Gp.get(ctx, (int64_t)kc * kc));
  TK_TRY(tk_dgemm(ctx, true, false, kc, kc, k, 1.0, Qv.p, kc, T1.p, kc, 0.0, Gp.p, kc));
  TK_TRY(tk_symmetrize(ctx, kc, Gp.p));
  TK_TRY(V2p.get(ctx, (int64_t)kc * kc));
  TK_TRY(tk_jacobi_eig(ctx, kc, Gp.p, lam2.p, V2p.p, kPass2.abs_scale, kPass2.rel, kMaxSweeps,
                       nullptr, nullptr, 0.0, 0, floor));
  TK_TRY(lam.get(ctx, k));
  TK_TRY(tk_fill(ctx, lam.p, k, 0.0));
  TK_TRY(tk_copy2d(ctx, 1, kc, lam2.p, kc, lam.p, kc));
  if (kc < k)
    TK_TRY(tk_copy2d(ctx, 1, 1, rem.p, 1, lam.p + kc, 1));
  TK_TRY(V2.get(ctx, k * k));
  TK_TRY(tk_fill(ctx, V2.p, k * k, 0.0));
  TK_TRY(tk_dgemm(ctx, false, false, k, kc, kc, 1.0, Qv.p, kc, V2p.p, kc, 0.0, V2.p, k));
  *rcap = kc;
  return TK_OK;
}

// Pass 2 of a bond SVD: the Cholesky-preconditioned variant when it applies (k > 64), else one
// relative Jacobi on G_W.  *rcap (out): the largest admissible rank — the preconditioned
// variant resolves only kc <= k eigenpairs (the Schur remainder `rem` of the truncated
// Cholesky sits at lam[kc] and counts only in the discarded tail), the plain Jacobi all k.
int pass2(tk_ctx* ctx, int64_t k, const DevBuf& GW, const DevBuf& V, const double* floor,
          DevBuf& lam, DevBuf& V2, DevBuf& Vt, int* rcap) {
  if (pass2_chol(ctx, k, GW, floor, lam, V2, rcap) != TK_OK) {
    TK_TRY(lam.get(ctx, k));
    TK_TRY(V2.get(ctx, k * k));
    TK_TRY(tk_jacobi_eig(ctx, (int)k, GW.p, lam.p, V2.p, kPass2.abs_scale, kPass2.rel,
                         kMaxSweeps, nullptr, nullptr, 0.0, 0, floor));
    *rcap = (int)k;
  }
  TK_TRY(Vt.get(ctx, k * k));
  TK_TRY(tk_dgemm(ctx, false, false, k, k, k, 1.0, V.p, k, V2.p, k, 0.0, Vt.p, k));
  return TK_OK;
}

// pass 2, then the rank rule (tk_rank_select; the chosen rank is capped at pass 2's rcap).
int pass2_and_rank(tk_ctx* ctx, int64_t k, const DevBuf& GW, const DevBuf& V,
                   const DevBuf& floor, double tol, const double* delta_dev, int64_t rmax,
                   DevBuf& lam, DevBuf& V2, DevBuf& Vt, DevBuf& sig, int* info, double* dinfo,
                   int hinfo[3], double hd[3]) {
  TK_TRY(sig.get(ctx, k));
  int rcap = (int)k;
  TK_TRY(pass2(ctx, k, GW, V, floor.p, lam, V2, Vt, &rcap));
  TK_TRY(tk_rank_select(ctx, (int)k, lam.p, sig.p, tol, delta_dev, rmax, kDropThr, info, dinfo,
                        rcap));
  TK_TRY(sync_read(ctx, hinfo, info, 3 * sizeof(int)));
  TK_TRY(sync_read(ctx, hd, dinfo, 3 * sizeof(double)));
  return TK_OK;
}

}  // namespace

int set_zero_tt(tk_ctx* ctx, tk_tt* x) {
  x->r1 = 1;
  x->r2 = 1;
  TK_TRY(tk_fill(ctx, x->U1, x->n_x, 0.0));
  TK_TRY(tk_fill(ctx, x->U2, x->n_xi, 0.0));
  TK_TRY(tk_fill(ctx, x->U3, x->n_t, 0.0));
  return TK_OK;
}


// y2blk (nullable): the middle core is block diagonal with nb = R1 / rb1 diagonal blocks of
// size rb1 x n_xi x rb2, packed in y2blk (the fused apply+round); x->U2 is then output only.
static int round_impl(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
                      double* sigma2_out, double* discarded_out, double* norm_out,
                      const double* y2blk = nullptr, int64_t rb1 = 0, int64_t rb2 = 0,
                      const double* gy_pre = nullptr, const tk_op* gop = nullptr);

int tk_round_now(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
                 double* sigma2_out, double* discarded_out, double* norm_out) {
  if (!ctx) return TK_EARG;
  int st;
  {
    CritScope cs(ctx);
    st = round_impl(ctx, x, tol, rmax, sigma1_out, sigma2_out, discarded_out, norm_out);
  }
  pool_settle(ctx);
  return st;
}

extern "C" int tk_round(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
                        double* sigma2_out, double* discarded_out, double* norm_out) {
  if (!ctx || !x) return TK_EARG;
  const uint32_t gate = tk_gate_claim(ctx);  // this rounding's number (copy-window gate)
  if (ctx->async && !tk_async_on_worker(ctx))  // queued: *x is read when the job runs
    return tk_async_submit(ctx, [=]() {
      GateGuard gg(ctx, gate);
      tk_tt xc = *x;
      const int st = tk_round_now(ctx, &xc, tol, rmax, sigma1_out, sigma2_out, discarded_out,
                                  norm_out);
      if (st == TK_OK) {  // publish the ranks into the caller's struct
        x->r1 = xc.r1;
        x->r2 = xc.r2;
      }
      return st;
    });
  GateGuard gg(ctx, gate);
  return tk_round_now(ctx, x, tol, rmax, sigma1_out, sigma2_out, discarded_out, norm_out);
}

extern "C" int tk_apply_round(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y, double tol,
                              int64_t rmax, double* sigma1_out, double* sigma2_out,
                              double* discarded_out, double* norm_out) {
  if (!ctx || !op || !x || !y) return TK_EARG;
  const uint32_t gate = tk_gate_claim(ctx);
  if (ctx->async && !tk_async_on_worker(ctx))
    return tk_async_submit(ctx, [=]() {
      GateGuard gg(ctx, gate);
      const tk_tt xc = *x;
      tk_tt yc = *y;
      const int st = tk_apply_round_now(ctx, op, &xc, &yc, tol, rmax, sigma1_out, sigma2_out,
                                        discarded_out, norm_out);
      if (st == TK_OK) {
        y->r1 = yc.r1;
        y->r2 = yc.r2;
      }
      return st;
    });
  GateGuard gg(ctx, gate);
  return tk_apply_round_now(ctx, op, x, y, tol, rmax, sigma1_out, sigma2_out, discarded_out,
                            norm_out);
}

int tk_apply_round_now(tk_ctx* ctx, const tk_op* op, const tk_tt* x, tk_tt* y, double tol,
                       int64_t rmax, double* sigma1_out, double* sigma2_out,
                       double* discarded_out, double* norm_out) {
  if (!ctx || !op) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_apply_round(x)"));
  if (!y || !y->U1 || !y->U2 || !y->U3) {
    ctx->err = "tk_apply_round: null output TT";
    return TK_EARG;
  }
  if (x->n_x != op->n_x || x->n_xi != op->n_xi || x->n_t != op->n_t || y->n_x != op->n_x ||
      y->n_xi != op->n_xi || y->n_t != op->n_t) {
    ctx->err = "tk_apply_round: mode sizes differ from the operator's";
    return TK_ESHAPE;
  }
  const int64_t R1 = op->T * x->r1, R2 = op->T * x->r2;
  if (R1 > y->cap1 || R2 > y->cap2) {
    ctx->err = "tk_apply_round: output capacity < (T r1, T r2)";
    return TK_ECAP;
  }
  // the SpMM (HBM-bound, all SMs) overlaps the latency-bound sweep of the small cores; the
  // round joins the side stream before its first read of Y1 (bond 1)
  CritScope cs(ctx);  // (declared before every buffer below: joins back after they are freed)
  // opt-in exact factor grouping (tk_op_group_space): the space core is produced in the
  // factored form Y1 = Y1' E, Y1' = [K_g U1]_g over the G group representatives
  const bool grouped = op->group_space && op->n_groups < op->T;
  const int64_t R1s = (grouped ? op->n_groups : op->T) * x->r1;  // columns of the stored Y1
  TK_TRY(apply_space_time(ctx, op, x, y, true, grouped));
  DevBuf gyb;  // bond 1's sampled pass-1 Gram, also on the side stream behind the SpMM
  {
    OnSide on(ctx);
    TK_TRY(gyb.get(ctx, R1s * R1s));
    TK_TRY(pass1_gram(ctx, op->n_x, R1s, y->U1, gyb.p));
  }
  SideJoin sj(ctx, true);  // (round_impl joins before bond 1; this covers early returns)
  DevBuf blk;
  TK_TRY(blk.get(ctx, R1 * x->n_xi * x->r2));
  {
    // the T diagonal blocks G_k x_2 U2 as ONE DMMA GEMM: [G_0; ...; G_{T-1}] (T n_xi x n_xi)
    // times U2 permuted to (n_xi) x (r1 r2), then (k, i, a, b) -> (k, a, i, b)
    TagScope t(ctx, "stoch_apply");
    const int64_t nxi = x->n_xi, r1 = x->r1, r2 = x->r2;
    DevBuf U2p, C;
    TK_TRY(U2p.get(ctx, nxi * r1 * r2));
    TK_TRY(tk_swap_mid(ctx, 1, r1, nxi, r2, x->U2, U2p.p));
    TK_TRY(C.get(ctx, op->T * nxi * r1 * r2));
    TK_TRY(tk_dgemm(ctx, false, false, op->T * nxi, r1 * r2, nxi, 1.0, op->G, nxi, U2p.p, r1 * r2,
                    0.0, C.p, r1 * r2));
    TK_TRY(tk_swap_mid(ctx, op->T, nxi, r1, r2, C.p, blk.p));
  }
  y->r1 = R1;
  y->r2 = R2;
  const int st = round_impl(ctx, y, tol, rmax, sigma1_out, sigma2_out, discarded_out, norm_out,
                            blk.p, x->r1, x->r2, gyb.p, grouped ? op : nullptr);
  blk.release();
  pool_settle(ctx);
  return st;
}

static int round_impl(tk_ctx* ctx, tk_tt* x, double tol, int64_t rmax, double* sigma1_out,
                      double* sigma2_out, double* discarded_out, double* norm_out,
                      const double* y2blk, int64_t rb1, int64_t rb2, const double* gy_pre,
                      const tk_op* gop) {
  TK_TRY(check_tt(ctx, x, "tk_round"));
  if (!(tol >= 0.0) || !std::isfinite(tol)) {
    ctx->err = "tk_round: tol must be finite and >= 0";
    return TK_EARG;
  }
  const int64_t n_x = x->n_x, n_xi = x->n_xi, n_t = x->n_t, R1 = x->r1, R2 = x->r2;
  // ---- step A: time core  U3 = L3 Q3  (Q3 = identity when n_t <= R2)
  DevBuf L3b, Q3c;
  const double* L3 = x->U3;
  int64_t k3 = n_t;
  bool q3_id = true;
  // Also when R2 >= n_t but the core is large: the rank-revealing orth_rows then finds the
  // NUMERICAL row rank k3 of U3 (terms sharing a time factor, e.g. T_k = I, make it exactly
  // rank-deficient: c4 k3 = 128 instead of n_t = 512), which shrinks the middle core's
  // unfolding (R1 x n_xi k3) and bond 2 four-fold for the price of one orth_rows on R2 x n_t.
  // (n_t < kOrth3MinNt: the rank cannot drop below much less than n_t's worth of columns and
  // the step costs more than it can save — c5, n_t = 64: every MGS rounding has R2 = 128 and
  // full time rank 64, ~1.5 ms of pure overhead per rounding)
  if (n_t > R2 || (R2 >= kOrth3MinRank && n_t >= kOrth3MinNt)) {
    TK_TRY(orth_rows(ctx, R2, n_t, x->U3, L3b, Q3c, &k3));
    L3 = L3b.p;
    q3_id = false;
  }
  // ---- step B: Y2p = U2 x_3 L3   ((R1 n_xi) x R2) (R2 x k3)
  DevBuf Y2p;
  TagScope tagr(ctx, "round.small");
  TK_TRY(Y2p.get(ctx, R1 * n_xi * k3));
  if (y2blk) {
    // block diagonal middle core: row block b of Y2p = B_b (rb1 n_xi x rb2) L3[b rb2 : (b+1) rb2, :]
    // (T-fold fewer flops than the dense product with its zero blocks)
    for (int64_t b = 0; b < R1 / rb1; b++)
      TK_TRY(tk_dgemm(ctx, false, false, rb1 * n_xi, k3, rb2, 1.0, y2blk + b * rb1 * n_xi * rb2,
                      rb2, L3 + b * rb2 * k3, k3, 0.0, Y2p.p + b * rb1 * n_xi * k3, k3));
  } else {
    TK_TRY(tk_dgemm(ctx, false, false, R1 * n_xi, k3, R2, 1.0, x->U2, R2, L3, k3, 0.0, Y2p.p, k3));
  }
  // ---- step C: Y2p as R1 x (n_xi k3) = L2 Q2
  const int64_t N2 = n_xi * k3;
  DevBuf L2b, Q2c;
  const double* L2 = Y2p.p;
  int64_t k2 = N2;
  bool q2_id = true;
  if (N2 > R1) {
    TK_TRY(orth_rows(ctx, R1, N2, Y2p.p, L2b, Q2c, &k2));
    L2 = L2b.p;
    q2_id = false;
  }
  // ---- step D: SVD of Z = U1 L2 (n_x x k2), space bond truncation
  TK_TRY(tk_side_join(ctx));  // U1 written by a side-stream SpMM (tk_apply_round)
  DevBuf W, GW1, V1, V2, Vt, lam, fl1;
  // grouped space core (gop != nullptr): x->U1 holds Y1' (n_x x G rb1) with Y1 = Y1' E, so
  // Z = Y1 L2 = Y1' (E L2): bond 1 runs on Y1' with L2' = E L2 (G rb1 x k2)
  DevBuf L2g;
  const double* L2z = L2;
  int64_t R1z = R1;
  if (gop) {
    R1z = (int64_t)gop->n_groups * rb1;
    TK_TRY(L2g.get(ctx, R1z * k2));
    TK_TRY(tk_group_rows(ctx, gop->T, gop->n_groups, rb1, k2, gop->d_group, gop->d_coef, L2,
                         L2g.p));
    L2z = L2g.p;
  }
  TK_TRY(svd_two_pass(ctx, n_x, R1z, x->U1, L2z, k2, W, GW1, V1, fl1, gy_pre));
  DevBuf sig1, scr;
  TK_TRY(scr.get(ctx, 16));
  int* info1 = (int*)scr.p;
  double* dinfo1 = scr.p + 2;  // [norm, delta, discarded]
  int* info2 = (int*)(scr.p + 6);
  double* dinfo2 = scr.p + 8;
  int hi1[3];
  double hd1[3];
  TK_TRY(pass2_and_rank(ctx, k2, GW1, V1, fl1, tol, nullptr, rmax, lam, V2, Vt, sig1, info1,
                        dinfo1, hi1, hd1));
  GW1.release();
  V1.release();
  if (!std::isfinite(hd1[0])) {
    ctx->err = "tk_round: non-finite norm";
    return TK_ENUMERIC;
  }
  if (norm_out) *norm_out = hd1[0];
  if (hd1[0] == 0.0) {
    if (sigma1_out) memset(sigma1_out, 0, sizeof(double) * R1);
    if (sigma2_out) memset(sigma2_out, 0, sizeof(double) * R2);
    if (discarded_out) discarded_out[0] = discarded_out[1] = 0.0;
    return set_zero_tt(ctx, x);
  }
  const int64_t r1 = hi1[0];
  if (sigma1_out) {
    std::vector<double> s(k2);
    TK_TRY(sync_read(ctx, s.data(), sig1.p, sizeof(double) * k2));
    for (int64_t i = 0; i < R1; i++) sigma1_out[i] = i < k2 ? s[i] : 0.0;
  }
  // U1_new = W V2[:, :r1] diag(1/sig)  -> x->U1 (n_x x r1), on the side stream: the DMMA-bound
  // reconstruction overlaps the latency-bound bond-2 chain (joined before return; W and F1
  // are released only after the join)
  DevBuf F1;
  TK_TRY(F1.get(ctx, k2 * r1));
  TK_TRY(tk_col_scale(ctx, k2, r1, V2.p, k2, F1.p, r1, sig1.p, 1));
  TK_TRY(tk_side_fork(ctx));
  SideJoin sj(ctx, true);  // destroyed before F1 and W
  {
    OnSide on(ctx);
    TagScope t(ctx, "bond1.form_U1");
    TK_TRY(tk_dgemm(ctx, false, false, n_x, r1, k2, 1.0, W.p, k2, F1.p, r1, 0.0, x->U1, r1));
  }
  // C = (Vt[:, :r1] diag(sig))^T Q2   (r1 x N2)
  DevBuf S1, C;
  TK_TRY(S1.get(ctx, k2 * r1));
  TK_TRY(tk_col_scale(ctx, k2, r1, Vt.p, k2, S1.p, r1, sig1.p, 0));
  TK_TRY(C.get(ctx, r1 * N2));
  if (q2_id) {
    TK_TRY(tk_transpose(ctx, k2, r1, S1.p, r1, C.p, N2));  // k2 == N2
  } else {
    TK_TRY(tk_dgemm(ctx, true, true, r1, N2, k2, 1.0, S1.p, r1, Q2c.p, k2, 0.0, C.p, N2));
  }
  // ---- step E: SVD of C as (r1 n_xi) x k3, time bond truncation
  DevBuf W2, GW2, V21, V22, Vt2, lam2, fl2;
  const int64_t M2 = r1 * n_xi;
  TK_TRY(svd_two_pass(ctx, M2, k3, C.p, nullptr, k3, W2, GW2, V21, fl2));
  DevBuf sig2;
  int hi2[3];
  double hd2[3];
  TK_TRY(pass2_and_rank(ctx, k3, GW2, V21, fl2, tol, dinfo1 + 1, rmax, lam2, V22, Vt2, sig2,
                        info2, dinfo2, hi2, hd2));
  const int64_t r2 = hi2[0];
  if (sigma2_out) {
    std::vector<double> s(k3);
    TK_TRY(sync_read(ctx, s.data(), sig2.p, sizeof(double) * k3));
    for (int64_t i = 0; i < R2; i++) sigma2_out[i] = i < k3 ? s[i] : 0.0;
  }
  if (discarded_out) {
    discarded_out[0] = hd1[2];
    discarded_out[1] = hd2[2];
  }
  // U2_new = W2 V22[:, :r2] diag(1/sig2) -> x->U2 ((r1 n_xi) x r2)
  {
    DevBuf F2;
    TK_TRY(F2.get(ctx, k3 * r2));
    TK_TRY(tk_col_scale(ctx, k3, r2, V22.p, k3, F2.p, r2, sig2.p, 1));
    TK_TRY(tk_dgemm(ctx, false, false, M2, r2, k3, 1.0, W2.p, k3, F2.p, r2, 0.0, x->U2, r2));
  }
  // U3_new = (Vt2[:, :r2] diag(sig2))^T Q3   (r2 x n_t)
  {
    DevBuf S2;
    TK_TRY(S2.get(ctx, k3 * r2));
    TK_TRY(tk_col_scale(ctx, k3, r2, Vt2.p, k3, S2.p, r2, sig2.p, 0));
    if (q3_id) {
      TK_TRY(tk_transpose(ctx, k3, r2, S2.p, r2, x->U3, n_t));  // k3 == n_t
    } else {
      TK_TRY(tk_dgemm(ctx, true, true, r2, n_t, k3, 1.0, S2.p, r2, Q3c.p, k3, 0.0, x->U3, n_t));
    }
  }
  TK_TRY(tk_side_join(ctx));
  W.release();
  F1.release();
  x->r1 = r1;
  x->r2 = r2;
  TK_CUDA_TRY(ctx, cudaGetLastError());
  return TK_OK;
}

// ============================================================================ dot / norm
static int same_modes(tk_ctx* ctx, const tk_tt* x, const tk_tt* y, const char* who) {
  if (x->n_x != y->n_x || x->n_xi != y->n_xi || x->n_t != y->n_t) {
    ctx->err = std::string(who) + ": mode sizes differ";
    return TK_ESHAPE;
  }
  return TK_OK;
}

static int dot_impl(tk_ctx* ctx, const tk_tt* x, const tk_tt* y, double* out, int take_sqrt) {
  const int64_t n_x = x->n_x, n_xi = x->n_xi, n_t = x->n_t;
  const int64_t a1 = x->r1, a2 = x->r2, b1 = y->r1, b2 = y->r2;
  DevBuf W1, Tm, W2, W3;
  TK_TRY(W1.get(ctx, a1 * b1));
  TK_TRY(tk_dgemm(ctx, true, false, a1, b1, n_x, 1.0, x->U1, a1, y->U1, b1, 0.0, W1.p, b1));
  TK_TRY(Tm.get(ctx, a1 * n_xi * b2));
  TK_TRY(tk_dgemm(ctx, false, false, a1, n_xi * b2, b1, 1.0, W1.p, b1, y->U2, n_xi * b2, 0.0,
                  Tm.p, n_xi * b2));
  TK_TRY(W2.get(ctx, a2 * b2));
  TK_TRY(tk_dgemm(ctx, true, false, a2, b2, a1 * n_xi, 1.0, x->U2, a2, Tm.p, b2, 0.0, W2.p, b2));
  TK_TRY(W3.get(ctx, a2 * b2));
  TK_TRY(tk_dgemm(ctx, false, true, a2, b2, n_t, 1.0, x->U3, n_t, y->U3, n_t, 0.0, W3.p, b2));
  TK_TRY(tk_dot_final(ctx, a2 * b2, W2.p, W3.p, out, take_sqrt));
  return TK_OK;
}

extern "C" int tk_dot(tk_ctx* ctx, const tk_tt* x, const tk_tt* y, double* out_dev) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out_dev) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_dot(x)"));
  TK_TRY(check_tt(ctx, y, "tk_dot(y)"));
  TK_TRY(same_modes(ctx, x, y, "tk_dot"));
  return dot_impl(ctx, x, y, out_dev, 0);
}

extern "C" int tk_norm(tk_ctx* ctx, const tk_tt* x, double* out_dev) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !out_dev) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_norm"));
  return dot_impl(ctx, x, x, out_dev, 1);
}

// ============================================================================ axpby / scale
extern "C" int tk_axpby(tk_ctx* ctx, const double* a_dev, const tk_tt* x, const double* b_dev,
                        const tk_tt* y, tk_tt* z) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !a_dev || !b_dev) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_axpby(x)"));
  TK_TRY(check_tt(ctx, y, "tk_axpby(y)"));
  TK_TRY(same_modes(ctx, x, y, "tk_axpby"));
  if (!z || !z->U1 || !z->U2 || !z->U3) {
    ctx->err = "tk_axpby: null output";
    return TK_EARG;
  }
  TK_TRY(same_modes(ctx, x, z, "tk_axpby(z)"));
  if (x->r1 + y->r1 > z->cap1 || x->r2 + y->r2 > z->cap2) {
    ctx->err = "tk_axpby: output capacity < rank sums";
    return TK_ECAP;
  }
  {
    // algorithmic bytes: every core entry of x and y read once, every entry of z written once
    // (the zero blocks of z's middle core are written, not read)
    const double R1 = (double)(x->r1 + y->r1), R2 = (double)(x->r2 + y->r2);
    const double bytes = 8.0 * (2.0 * x->n_x * R1 +
                                (x->r1 * x->r2 + y->r1 * y->r2 + R1 * R2) * x->n_xi +
                                2.0 * R2 * x->n_t);
    TagScope ts(ctx, "axpby");
    const int id = tk_prof_begin(ctx, "axpby", 0.0, bytes);
    TK_TRY(tk_axpby_cores(ctx, a_dev, x, b_dev, y, z));
    tk_prof_end(ctx, id);
  }
  z->r1 = x->r1 + y->r1;
  z->r2 = x->r2 + y->r2;
  return TK_OK;
}

extern "C" int tk_axpby_host(tk_ctx* ctx, double a, const tk_tt* x, double b, const tk_tt* y,
                             tk_tt* z) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx) return TK_EARG;
  DevBuf s;
  TK_TRY(s.get(ctx, 2));
  TK_TRY(tk_set_scalar(ctx, s.p, a));
  TK_TRY(tk_set_scalar(ctx, s.p + 1, b));
  return tk_axpby(ctx, s.p, x, s.p + 1, y, z);
}

extern "C" int tk_scale(tk_ctx* ctx, tk_tt* x, const double* s_dev, int invert) {
  TK_ASYNC_GUARD(ctx);
  if (!ctx || !s_dev) return TK_EARG;
  TK_TRY(check_tt(ctx, x, "tk_scale"));
  return tk_scale_rows(ctx, x->U3, x->r2 * x->n_t, s_dev, invert);
}

// ============================================================================ GMRES
int tk_apply_round_owned(tk_ctx* ctx, const tk_op* op, const tk_tt* x, OwnedPtr& y, double tol) {
  y = std::make_unique<OwnedTT>();
  TK_TRY(y->make(ctx, x->n_x, x->n_xi, x->n_t, op->T * x->r1, op->T * x->r2));
  return tk_apply_round_now(ctx, op, x, &y->t, tol, 0, nullptr, nullptr, nullptr, nullptr);
}

// One cycle (tk_gmres_cycle), plus what the restarted solver needs: stop once the Givens
// least-squares residual is <= stop_abs (Alg. 3 line 2, R19) and hand back the
// iterate z = sum_i y_i v^_i (z_out, nullable) instead of / besides its explicit residual.
// prec (nullable): right preconditioner, v^_k = P^{-1} v_k (line 4); the flexible form keeps
// the v^_k and forms z from them (lines 11, 13).
static int gmres_cycle_impl(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int steps, double tol,
                            double stop_abs, const TkPrecFn* prec, double* history_out,
                            int* steps_done, double* explicit_out, double* step_ms_out,
                            OwnedPtr* z_out) {
  if (!ctx || !op || !history_out || !steps_done || steps < 1) return TK_EARG;
  TK_TRY(check_tt(ctx, b, "tk_gmres_cycle(b)"));
  if (b->n_x != op->n_x || b->n_xi != op->n_xi || b->n_t != op->n_t) {
    ctx->err = "tk_gmres_cycle: b mode sizes differ from the operator's";
    return TK_ESHAPE;
  }
  const int64_t n_x = b->n_x, n_xi = b->n_xi, n_t = b->n_t;
  const int T = op->T;
  DevBuf sc;  // device scalars: [beta, hn, nav, h(0..steps), negh(0..steps), one]
  TK_TRY(sc.get(ctx, 4 + 2 * (steps + 1)));
  double* d_beta = sc.p;
  double* d_hn = sc.p + 1;
  double* d_nav = sc.p + 2;
  double* d_h = sc.p + 3;
  double* d_negh = d_h + (steps + 1);
  double* d_one = d_negh + (steps + 1);
  TK_TRY(tk_set_scalar(ctx, d_one, 1.0));

  std::vector<OwnedPtr> V, Vhat;
  V.emplace_back(new OwnedTT());
  TK_TRY(clone_tt(ctx, b, *V[0]));
  TK_TRY(tk_round_now(ctx, &V[0]->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
  TK_TRY(tk_norm(ctx, &V[0]->t, d_beta));
  double beta;
  TK_TRY(sync_read(ctx, &beta, d_beta, sizeof(double)));
  TK_TRY(tk_scale(ctx, &V[0]->t, d_beta, 1));
  std::vector<double> H((size_t)(steps + 1) * steps, 0.0), cs, sn, g(steps + 1, 0.0);
  g[0] = beta;
  history_out[0] = beta;
  int k_done = 0;
  for (int k = 0; k < steps; k++) {
    auto t0 = std::chrono::high_resolution_clock::now();
    const tk_tt* vk = &V[k]->t;
    if (prec) {  // line 4: v^_k = P^{-1} v_k
      OwnedPtr vh;
      TK_TRY((*prec)(vk, vh));
      Vhat.push_back(std::move(vh));
      vk = &Vhat.back()->t;
    }
    OwnedPtr x;
    TK_TRY(tk_apply_round_owned(ctx, op, vk, x, tol));
    TK_TRY(tk_norm(ctx, &x->t, d_nav));
    for (int i = 0; i <= k; i++) {
      TK_TRY(tk_dot(ctx, &x->t, &V[i]->t, d_h + i));
      TK_TRY(tk_neg_scalar(ctx, d_h + i, d_negh + i));
      auto z = std::make_unique<OwnedTT>();
      TK_TRY(z->make(ctx, n_x, n_xi, n_t, x->t.r1 + V[i]->t.r1, x->t.r2 + V[i]->t.r2));
      TK_TRY(tk_axpby(ctx, d_one, &x->t, d_negh + i, &V[i]->t, &z->t));
      TK_TRY(tk_round_now(ctx, &z->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
      x = std::move(z);
    }
    TK_TRY(tk_norm(ctx, &x->t, d_hn));
    std::vector<double> hcol(k + 1);
    double hn, nav;
    TK_TRY(sync_read(ctx, hcol.data(), d_h, sizeof(double) * (k + 1)));
    TK_TRY(sync_read(ctx, &hn, d_hn, sizeof(double)));
    TK_TRY(sync_read(ctx, &nav, d_nav, sizeof(double)));
    // Givens update of column k of H-bar
    std::vector<double> col(k + 2);
    for (int i = 0; i <= k; i++) col[i] = hcol[i];
    col[k + 1] = hn;
    for (int i = 0; i < k; i++) {
      double t0v = cs[i] * col[i] + sn[i] * col[i + 1];
      col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
      col[i] = t0v;
    }
    double c = 1.0, s = 0.0;
    if (col[k + 1] != 0.0) {
      double r = std::hypot(col[k], col[k + 1]);
      c = col[k] / r;
      s = col[k + 1] / r;
    }
    cs.push_back(c);
    sn.push_back(s);
    col[k] = c * col[k] + s * col[k + 1];
    col[k + 1] = 0.0;
    for (int i = 0; i <= k + 1; i++) H[(size_t)i * steps + k] = col[i];
    g[k + 1] = -s * g[k];
    g[k] = c * g[k];
    history_out[k + 1] = std::fabs(g[k + 1]);
    k_done = k + 1;
    bool breakdown = hn <= 1e-14 * nav || history_out[k + 1] <= stop_abs;
    if (!breakdown) {
      TK_TRY(tk_scale(ctx, &x->t, d_hn, 1));
      V.push_back(std::move(x));
    }
    TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    auto t1 = std::chrono::high_resolution_clock::now();
    if (step_ms_out) step_ms_out[k] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (breakdown) break;
  }
  *steps_done = k_done;
  if (explicit_out || z_out) {
    // y = R^{-1} g  (back substitution on the rotated H-bar)
    std::vector<double> y(k_done, 0.0);
    for (int i = k_done - 1; i >= 0; i--) {
      double s = g[i];
      for (int j = i + 1; j < k_done; j++) s -= H[(size_t)i * steps + j] * y[j];
      y[i] = s / H[(size_t)i * steps + i];
    }
    std::vector<OwnedPtr>& B = prec ? Vhat : V;  // the basis z is formed from (line 13)
    auto z = std::make_unique<OwnedTT>();
    TK_TRY(clone_tt(ctx, &B[0]->t, *z));
    TK_TRY(tk_set_scalar(ctx, d_h, y[0]));
    TK_TRY(tk_scale(ctx, &z->t, d_h, 0));
    for (int i = 1; i < k_done; i++) {
      auto z2 = std::make_unique<OwnedTT>();
      TK_TRY(z2->make(ctx, n_x, n_xi, n_t, z->t.r1 + B[i]->t.r1, z->t.r2 + B[i]->t.r2));
      TK_TRY(tk_axpby_host(ctx, 1.0, &z->t, y[i], &B[i]->t, &z2->t));
      TK_TRY(tk_round_now(ctx, &z2->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
      z = std::move(z2);
    }
    if (!explicit_out) {
      *z_out = std::move(z);
      return TK_OK;
    }
    auto az = std::make_unique<OwnedTT>();
    TK_TRY(az->make(ctx, n_x, n_xi, n_t, T * z->t.r1, T * z->t.r2));
    TK_TRY(tk_apply_op(ctx, op, &z->t, &az->t));
    auto r = std::make_unique<OwnedTT>();
    TK_TRY(r->make(ctx, n_x, n_xi, n_t, b->r1 + az->t.r1, b->r2 + az->t.r2));
    TK_TRY(tk_axpby_host(ctx, 1.0, b, -1.0, &az->t, &r->t));
    TK_TRY(tk_round_now(ctx, &r->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
    TK_TRY(tk_norm(ctx, &r->t, d_hn));
    TK_TRY(sync_read(ctx, explicit_out, d_hn, sizeof(double)));
    if (z_out) *z_out = std::move(z);
  }
  return TK_OK;
}

static int gmres_cycle_entry(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b,
                             int steps, double tol, double* history_out, int* steps_done,
                             double* explicit_out, double* step_ms_out) {
  if (!ctx) return TK_EARG;
  TkPrecFn fn;
  if (P) fn = tk_prec_fn(ctx, P, 0);
  return gmres_cycle_impl(ctx, op, b, steps, tol, 0.0, P ? &fn : nullptr, history_out,
                          steps_done, explicit_out, step_ms_out, nullptr);
}

extern "C" int tk_gmres_cycle(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int steps,
                              double tol, double* history_out, int* steps_done,
                              double* explicit_out, double* step_ms_out) {
  TK_ASYNC_GUARD(ctx);
  return gmres_cycle_entry(ctx, op, nullptr, b, steps, tol, history_out, steps_done,
                           explicit_out, step_ms_out);
}

extern "C" int tk_gmres_cycle_p(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b,
                                int steps, double tol, double* history_out, int* steps_done,
                                double* explicit_out, double* step_ms_out) {
  TK_ASYNC_GUARD(ctx);
  if (!P) return TK_EARG;
  return gmres_cycle_entry(ctx, op, P, b, steps, tol, history_out, steps_done, explicit_out,
                           step_ms_out);
}

// Complete, restarted low-rank GMRES (NEXT-2; Alg. 3, eq:eps_soln; R19), flexible
// with a right preconditioner (NEXT-3).
int tk_gmres_solve_core(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int restart,
                        int max_cycles, double tol, double tol_gmres, double eps_soln,
                        const TkPrecFn* prec, OwnedPtr& zt, std::vector<double>& explicit_out,
                        std::vector<double>* ls_out, std::vector<int>* steps_out) {
  if (eps_soln < 0.0) eps_soln = tol;
  const int64_t n_x = b->n_x, n_xi = b->n_xi, n_t = b->n_t;
  const int T = op->T;
  DevBuf sc;
  TK_TRY(sc.get(ctx, 1));
  TK_TRY(tk_norm(ctx, b, sc.p));
  double bnorm, e;
  TK_TRY(sync_read(ctx, &bnorm, sc.p, sizeof(double)));
  // s_0 = T(b)  (z_0 = 0)
  auto s_ = std::make_unique<OwnedTT>();
  TK_TRY(clone_tt(ctx, b, *s_));
  TK_TRY(tk_round_now(ctx, &s_->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
  TK_TRY(tk_norm(ctx, &s_->t, sc.p));
  TK_TRY(sync_read(ctx, &e, sc.p, sizeof(double)));
  explicit_out.assign(1, e);
  zt.reset();
  for (int cyc = 0; cyc < max_cycles; cyc++) {
    if (explicit_out[cyc] <= tol_gmres * bnorm) break;
    std::vector<double> hist(restart + 1, 0.0);
    int done = 0;
    OwnedPtr dz;
    TK_TRY(gmres_cycle_impl(ctx, op, &s_->t, restart, tol, tol_gmres * bnorm, prec, hist.data(),
                            &done, nullptr, nullptr, &dz));
    if (ls_out)
      for (int i = 0; i <= restart; i++) ls_out->push_back(i <= done ? hist[i] : 0.0);
    if (steps_out) steps_out->push_back(done);
    // z <- T_eps_soln(z + dz)   (eq:eps_soln)
    if (!zt) {
      zt = std::move(dz);
    } else {
      auto z2 = std::make_unique<OwnedTT>();
      TK_TRY(z2->make(ctx, n_x, n_xi, n_t, zt->t.r1 + dz->t.r1, zt->t.r2 + dz->t.r2));
      TK_TRY(tk_axpby_host(ctx, 1.0, &zt->t, 1.0, &dz->t, &z2->t));
      zt = std::move(z2);
    }
    TK_TRY(tk_round_now(ctx, &zt->t, eps_soln, 0, nullptr, nullptr, nullptr, nullptr));
    // s = T(b - L z)   (line 14)
    auto az = std::make_unique<OwnedTT>();
    TK_TRY(az->make(ctx, n_x, n_xi, n_t, T * zt->t.r1, T * zt->t.r2));
    TK_TRY(tk_apply_op(ctx, op, &zt->t, &az->t));
    auto s2 = std::make_unique<OwnedTT>();
    TK_TRY(s2->make(ctx, n_x, n_xi, n_t, b->r1 + az->t.r1, b->r2 + az->t.r2));
    TK_TRY(tk_axpby_host(ctx, 1.0, b, -1.0, &az->t, &s2->t));
    TK_TRY(tk_round_now(ctx, &s2->t, tol, 0, nullptr, nullptr, nullptr, nullptr));
    s_ = std::move(s2);
    TK_TRY(tk_norm(ctx, &s_->t, sc.p));
    TK_TRY(sync_read(ctx, &e, sc.p, sizeof(double)));
    explicit_out.push_back(e);
  }
  return TK_OK;
}

static int gmres_solve_entry(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b,
                             int restart, int max_cycles, double tol, double tol_gmres,
                             double eps_soln, tk_tt* z, double* explicit_out, double* ls_out,
                             int* cycles_done, int* steps_out) {
  if (!ctx || !op || !z || !explicit_out || !cycles_done || restart < 1 || max_cycles < 0 ||
      !(tol >= 0.0) || !(tol_gmres >= 0.0))
    return TK_EARG;
  TK_TRY(check_tt(ctx, b, "tk_gmres_solve(b)"));
  if (b->n_x != op->n_x || b->n_xi != op->n_xi || b->n_t != op->n_t || z->n_x != op->n_x ||
      z->n_xi != op->n_xi || z->n_t != op->n_t) {
    ctx->err = "tk_gmres_solve: mode sizes differ from the operator's";
    return TK_ESHAPE;
  }
  TkPrecFn fn;
  if (P) fn = tk_prec_fn(ctx, P, 0);
  OwnedPtr zt;
  std::vector<double> expl, ls;
  std::vector<int> steps;
  TK_TRY(tk_gmres_solve_core(ctx, op, b, restart, max_cycles, tol, tol_gmres, eps_soln,
                             P ? &fn : nullptr, zt, expl, &ls, &steps));
  const int cyc = (int)steps.size();
  *cycles_done = cyc;
  for (size_t i = 0; i < expl.size(); i++) explicit_out[i] = expl[i];
  if (ls_out)
    for (size_t i = 0; i < ls.size(); i++) ls_out[i] = ls[i];
  if (steps_out)
    for (int i = 0; i < cyc; i++) steps_out[i] = steps[i];
  if (!zt) {  // b rounded to (numerically) zero or max_cycles == 0: z = 0
    TK_TRY(set_zero_tt(ctx, z));
    return TK_OK;
  }
  if (zt->t.r1 > z->cap1 || zt->t.r2 > z->cap2) {
    ctx->err = "tk_gmres_solve: solution ranks exceed z's capacity";
    return TK_ECAP;
  }
  const int64_t n_x = b->n_x, n_xi = b->n_xi, n_t = b->n_t;
  z->r1 = zt->t.r1;
  z->r2 = zt->t.r2;
  TK_TRY(tk_copy2d(ctx, n_x, z->r1, zt->t.U1, z->r1, z->U1, z->r1));
  TK_TRY(tk_copy2d(ctx, z->r1 * n_xi, z->r2, zt->t.U2, z->r2, z->U2, z->r2));
  TK_TRY(tk_copy2d(ctx, z->r2, n_t, zt->t.U3, n_t, z->U3, n_t));
  TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TK_OK;
}

extern "C" int tk_gmres_solve(tk_ctx* ctx, const tk_op* op, const tk_tt* b, int restart,
                              int max_cycles, double tol, double tol_gmres, double eps_soln,
                              tk_tt* z, double* explicit_out, double* ls_out, int* cycles_done,
                              int* steps_out) {
  TK_ASYNC_GUARD(ctx);
  return gmres_solve_entry(ctx, op, nullptr, b, restart, max_cycles, tol, tol_gmres, eps_soln,
                           z, explicit_out, ls_out, cycles_done, steps_out);
}

extern "C" int tk_gmres_solve_p(tk_ctx* ctx, const tk_op* op, const tk_prec* P, const tk_tt* b,
                                int restart, int max_cycles, double tol, double tol_gmres,
                                double eps_soln, tk_tt* z, double* explicit_out, double* ls_out,
                                int* cycles_done, int* steps_out) {
  TK_ASYNC_GUARD(ctx);
  if (!P) return TK_EARG;
  return gmres_solve_entry(ctx, op, P, b, restart, max_cycles, tol, tol_gmres, eps_soln, z,
                           explicit_out, ls_out, cycles_done, steps_out);
}

// Module anchor: async.cu loads every kernel of this translation unit through it (lazy module
// loading must not happen while a context stream is gated, see tk_ctx_set_async).
__global__ void tk_anchor_ttk_api_k() {}
const void* tk_anchor_ttk_api() { return (const void*)tk_anchor_ttk_api_k; }
