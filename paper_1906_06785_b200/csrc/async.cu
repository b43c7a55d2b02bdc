// Asynchronous rounding for the C ABI ("all calls are asynchronous on the ctx
// stream; only tk_sync_ranks and host-mode scalars block").
//
// The rank decisions of a rounding are taken on the device, but the launches
// that follow them are sized on the host, so a rounding needs host<->device round trips.  In
// async mode (tk_ctx_set_async) tk_round / tk_apply_round therefore do not run on the calling
// thread: they are queued to a per-context worker thread that drives the GPU on a private
// stream, and the caller's stream is gated in stream order on the job's completion with a
// device-side wait (cuStreamWaitValue32 on a flag the worker's stream writes with
// cuStreamWriteValue32 after the job's last kernel).  The calling thread returns at once; work
// it enqueues afterwards on its stream runs after the rounding.  The new ranks are published
// into the caller's tk_tt by the worker and are valid after tk_sync_ranks; every other entry
// point on the context first waits for the queued jobs (they read ranks on the host).
#include <cuda.h>
#include <cuda_runtime.h>

#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ttk_internal.h"

namespace {
typedef CUresult (*PfnFuncGetModule)(CUmodule*, CUfunction);
typedef CUresult (*PfnModCount)(unsigned int*, CUmodule);
typedef CUresult (*PfnModEnum)(CUfunction*, unsigned int, CUmodule);
typedef CUresult (*PfnFuncLoad)(CUfunction);
typedef CUresult (*PfnWait)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PfnWrite)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PfnWait g_wait = nullptr;
PfnWrite g_write = nullptr;
std::once_flag g_once;

bool memops_available() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    void *w = nullptr, *v = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &w, 12000, cudaEnableDefault,
                                         &q1) == cudaSuccess &&
        cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &v, 12000, cudaEnableDefault,
                                         &q2) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess) {
      g_wait = (PfnWait)w;
      g_write = (PfnWrite)v;
    }
    cudaGetLastError();
  });
  return g_wait && g_write;
}

template <typename F>
bool entry(const char* name, F* out) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12040, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  *out = (F)p;
  return true;
}
}  // namespace

// One kernel of every translation unit (its module anchor).
const void* tk_anchor_k_apply();
const void* tk_anchor_k_gemm();
const void* tk_anchor_k_gemm_tma();
const void* tk_anchor_k_jacobi();
const void* tk_anchor_k_qr();
const void* tk_anchor_k_chol();
const void* tk_anchor_k_small();
const void* tk_anchor_k_conv();
const void* tk_anchor_prec();
const void* tk_anchor_ttk_api();

// Load every kernel of the library now.  With CUDA's lazy module loading a kernel is loaded at
// its first launch, and loading waits for the device — which never idles while a context
// stream is gated on a queued rounding, so the worker's first launch of a new kernel would
// deadlock.  Enumerates each translation unit's module from its anchor kernel.
static int preload_kernels(tk_ctx* ctx) {
  PfnFuncGetModule fgm;
  PfnModCount mcount;
  PfnModEnum menum;
  PfnFuncLoad fload;
  if (!entry("cuFuncGetModule", &fgm) || !entry("cuModuleGetFunctionCount", &mcount) ||
      !entry("cuModuleEnumerateFunctions", &menum) || !entry("cuFuncLoad", &fload)) {
    ctx->err = "tk_ctx_set_async: driver lacks the module enumeration entry points";
    return TK_ECUDA;
  }
  const void* anchors[] = {tk_anchor_k_apply(), tk_anchor_k_gemm(),  tk_anchor_k_jacobi(),
                           tk_anchor_k_qr(),    tk_anchor_k_chol(),  tk_anchor_k_small(),
                           tk_anchor_k_conv(),  tk_anchor_prec(),    tk_anchor_ttk_api(),
                           tk_anchor_k_gemm_tma()};
  for (const void* a : anchors) {
    cudaFunction_t f;
    TK_CUDA_TRY(ctx, cudaGetFuncBySymbol(&f, a));
    CUmodule mod;
    unsigned int n = 0;
    if (fgm(&mod, (CUfunction)f) != CUDA_SUCCESS || mcount(&n, mod) != CUDA_SUCCESS) {
      ctx->err = "tk_ctx_set_async: cannot enumerate a kernel module";
      return TK_ECUDA;
    }
    std::vector<CUfunction> fs(n);
    if (n && menum(fs.data(), n, mod) != CUDA_SUCCESS) {
      ctx->err = "tk_ctx_set_async: cuModuleEnumerateFunctions failed";
      return TK_ECUDA;
    }
    for (CUfunction fn : fs)
      if (fload(fn) != CUDA_SUCCESS) {
        ctx->err = "tk_ctx_set_async: cuFuncLoad failed";
        return TK_ECUDA;
      }
  }
  return TK_OK;
}

struct tk_async {
  tk_ctx* ctx = nullptr;
  cudaStream_t user = nullptr;   // the context's stream (gated)
  cudaStream_t wstream = nullptr;  // the worker's stream
  uint32_t* flag = nullptr;      // device: last completed job sequence number
  uint32_t seq = 0;              // last enqueued
  std::thread th;
  std::thread::id tid;
  std::mutex m;
  std::condition_variable cv, idle;
  std::deque<std::function<int()>> q;
  bool stop = false, busy = false;
  int err = TK_OK;
  std::string msg;
  std::vector<cudaEvent_t> ev_free;

  void loop() {
    std::unique_lock<std::mutex> lk(m);
    for (;;) {
      cv.wait(lk, [&] { return stop || !q.empty(); });
      if (q.empty()) return;
      auto job = std::move(q.front());
      q.pop_front();
      busy = true;
      lk.unlock();
      const int st = job();
      lk.lock();
      if (st != TK_OK && err == TK_OK) {
        err = st;
        msg = ctx->err;
      }
      busy = false;
      if (q.empty()) idle.notify_all();
    }
  }
};

bool tk_async_on_worker(const tk_ctx* ctx) {
  return ctx->async && std::this_thread::get_id() == ctx->async->tid;
}

int tk_async_drain(tk_ctx* ctx) {
  tk_async* A = ctx->async;
  if (!A || std::this_thread::get_id() == A->tid) return TK_OK;
  std::unique_lock<std::mutex> lk(A->m);
  A->idle.wait(lk, [&] { return A->q.empty() && !A->busy; });
  const int st = A->err;
  if (st != TK_OK) {
    ctx->err = A->msg;
    A->err = TK_OK;
  }
  return st;
}

// Run `body` on the worker: it sees ctx->stream = the worker's stream, ordered after everything
// enqueued so far on the caller's stream; the caller's stream waits for its completion.
int tk_async_submit(tk_ctx* ctx, std::function<int()> body) {
  tk_async* A = ctx->async;
  cudaEvent_t ev;
  {
    std::lock_guard<std::mutex> lk(A->m);
    if (!A->ev_free.empty()) {
      ev = A->ev_free.back();
      A->ev_free.pop_back();
    } else if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
      ctx->err = "tk_async_submit: cudaEventCreate";
      return TK_ECUDA;
    }
  }
  TK_CUDA_TRY(ctx, cudaEventRecord(ev, A->user));
  const uint32_t seq = ++A->seq;
  auto job = [A, ev, seq, body = std::move(body)]() -> int {
    tk_ctx* c = A->ctx;
    c->stream = A->wstream;
    int st = cudaStreamWaitEvent(A->wstream, ev, 0) == cudaSuccess ? TK_OK : TK_ECUDA;
    if (st == TK_OK) st = body();
    // always release the gate (an error must not deadlock the caller's stream)
    if (g_write((CUstream)A->wstream, (CUdeviceptr)A->flag, seq, 0) != CUDA_SUCCESS &&
        st == TK_OK) {
      c->err = "cuStreamWriteValue32 failed";
      st = TK_ECUDA;
    }
    c->stream = A->user;
    {
      std::lock_guard<std::mutex> lk(A->m);
      A->ev_free.push_back(ev);
    }
    return st;
  };
  {
    std::lock_guard<std::mutex> lk(A->m);
    A->q.push_back(std::move(job));
  }
  A->cv.notify_one();
  if (g_wait((CUstream)A->user, (CUdeviceptr)A->flag, seq, CU_STREAM_WAIT_VALUE_GEQ) !=
      CUDA_SUCCESS) {
    ctx->err = "cuStreamWaitValue32 failed";
    tk_async_drain(ctx);
    return TK_ECUDA;
  }
  return TK_OK;
}

static void async_stop(tk_ctx* ctx) {
  tk_async* A = ctx->async;
  if (!A) return;
  {
    std::lock_guard<std::mutex> lk(A->m);
    A->stop = true;
  }
  A->cv.notify_all();
  if (A->th.joinable()) A->th.join();
  cudaStreamSynchronize(A->wstream);
  cudaStreamSynchronize(A->user);
  cudaStreamDestroy(A->wstream);
  cudaFree(A->flag);
  for (auto e : A->ev_free) cudaEventDestroy(e);
  ctx->async = nullptr;
  delete A;
}

extern "C" int tk_ctx_set_async(tk_ctx* ctx, int on) {
  if (!ctx) return TK_EARG;
  if (!on) {
    const int st = tk_async_drain(ctx);
    async_stop(ctx);
    return st;
  }
  if (ctx->async) return 1;
  if (!memops_available()) return 0;  // stays synchronous (still correct)
  TK_TRY(preload_kernels(ctx));
  auto* A = new tk_async();
  A->ctx = ctx;
  A->user = ctx->stream;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&A->wstream, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaMalloc(&A->flag, sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(A->flag, 0, sizeof(uint32_t)) != cudaSuccess) {
    cudaGetLastError();
    delete A;
    ctx->err = "tk_ctx_set_async: stream / flag allocation failed";
    return TK_ECUDA;
  }
  ctx->async = A;
  A->th = std::thread([A] { A->loop(); });
  A->tid = A->th.get_id();
  return 1;
}

// ---------------------------------------------------------------------------- copy-window gate
// The latency-bound phases of a rounding (the small-core chain before the big Gram pass, and the
// pass-2 / bond-2 chain after it) launch ~1500 short kernels whose command fetches share the
// PCIe link with bulk host <-> device copies: a concurrent 7 ms H2D copy at the start of a c4 op
// costs the op 6.5 ms (profiles/r02/e2e_diag.txt).  The DMMA-bound phase in between (form_W,
// gram_W: 35 ms at c4) is insensitive to it.  tk_ctx_gate_stream makes a user stream wait (a
// device-side wait on a flag, no host synchronisation) until the most recently SUBMITTED
// rounding of the context has reached that phase, so pipelined transfers of the neighbouring
// steps land inside the window.  A gate only ever waits for work that is already queued, and
// every rounding publishes its number on all exit paths: no call order can leave a stream
// waiting forever.
extern "C" int tk_ctx_gate_stream(tk_ctx* ctx, void* cuda_stream) {
  if (!ctx) return TK_EARG;
  if (!memops_available()) return 0;  // no stream memory operations: the stream is not gated
  if (!ctx->gate_flag) {
    // A gated stream does not idle until the rounding publishes its number, and CUDA's lazy
    // loading of a not-yet-loaded kernel waits for the device to idle: load every kernel of
    // the library first (as tk_ctx_set_async does).  Roundings submitted before the flag
    // existed never publish: wait for them, then start the flag at the current number.
    TK_TRY(preload_kernels(ctx));
    if (ctx->async) TK_TRY(tk_async_drain(ctx));
    TK_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    uint32_t* f = nullptr;
    const uint32_t v = ctx->round_seq;
    if (cudaMalloc(&f, sizeof(uint32_t)) != cudaSuccess ||
        cudaMemcpy(f, &v, sizeof(v), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaGetLastError();
      ctx->err = "tk_ctx_gate_stream: flag allocation failed";
      return TK_ECUDA;
    }
    ctx->gate_flag = f;
  }
  if (g_wait((CUstream)cuda_stream, (CUdeviceptr)ctx->gate_flag, ctx->round_seq,
             CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
    ctx->err = "tk_ctx_gate_stream: cuStreamWaitValue32 failed";
    return TK_ECUDA;
  }
  return 1;
}

// number of the rounding being submitted (caller thread)
uint32_t tk_gate_claim(tk_ctx* ctx) { return ++ctx->round_seq; }

void tk_gate_open(tk_ctx* ctx) {
  if (!ctx->gate_job) return;
  if (ctx->gate_flag)
    g_write((CUstream)ctx->stream, (CUdeviceptr)ctx->gate_flag, ctx->gate_job, 0);
  ctx->gate_job = 0;
}

void tk_gate_destroy(tk_ctx* ctx) {  // (after the queue was drained: every gate is open)
  if (!ctx->gate_flag) return;
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->gate_flag);
  ctx->gate_flag = nullptr;
}

void tk_async_destroy(tk_ctx* ctx) {
  tk_async_drain(ctx);
  async_stop(ctx);
}

extern "C" int tk_sync_ranks(tk_ctx* ctx, tk_tt* x) {
  (void)x;  // the worker publishes every job's ranks; draining the queue makes them valid
  if (!ctx) return TK_EARG;
  return tk_async_drain(ctx);
}
