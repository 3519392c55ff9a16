// Context handle + workspace (host side).
#pragma once

#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace sqb {
// Optional per-column callbacks of the left-looking sweep, used by the
// host-buffer entry points (host_pipe.cu) to overlap PCIe transfers with the
// factorization.  Both run on the host at enqueue time.
struct SweepHooks {
  // columns of W arrive in groups: make ctx->stream wait until columns
  // [0, upto) are resident; returns the end of the group that holds column
  // upto-1 (>= upto).  A null hooks pointer / streamed_input == false means
  // W is fully resident before the sweep starts.
  bool streamed_input = false;
  virtual int64_t wait_cols(sqb_ctx* ctx, int64_t upto) = 0;
  // called after the launch that finalises U[:, c] has been enqueued
  virtual int col_final(sqb_ctx* ctx, int64_t c) = 0;
  virtual ~SweepHooks() {}
};
}  // namespace sqb

struct sqb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  char err[512] = {0};
  void* ws = nullptr;          // grow-only scratch (partials, sketches, coefficients)
  size_t ws_bytes = 0;
  sqb::Status* d_status = nullptr;
  sqb::Status* h_status = nullptr;  // pinned mirror
  int64_t launches = 0;        // kernel launches issued (instrumentation for bench)
  int sm_count = 148;
  // per-launch CUDA-event timing of the dominant kernel (rhqr_col_kernel), on
  // the stream it is launched on; enabled by sqb_ctx_profile()
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;   // pairs (begin, end)
  std::vector<double> prof_bytes;     // algorithmic bytes of each timed launch
  size_t prof_used = 0;
  // NCCL communicator for the row-partitioned path (sqb_ctx_init_comm)
  void* nccl = nullptr;
  long long* dbg_ts = nullptr;  // instrumentation: step-kernel phase stamps for column dbg_col
  int dbg_col = -1;
  // stream trace (sqb_ctx_trace): an event after every launch, so consecutive
  // deltas give each kernel's time in the stream as issued (gap + run)
  bool trace = false;
  std::vector<cudaEvent_t> trace_ev;
  std::vector<const char*> trace_name;
  size_t trace_used = 0;
  // a copy of the identity-block rows (copy_top) waiting to ride on the next single-vector SRHT tree
  // launch (defer_copy_top / flush_copy_top, sketch.cu): one launch less per sketch of an Arnoldi vector
  bool top_pending = false;
  const void* top_X = nullptr;
  int64_t top_ldx = 0, top_m = 0, top_k = 0, top_ldy = 0;
  double* top_Y = nullptr;
  int top_dtype = 0;
  long long* dbg_cts = nullptr;  // instrumentation: column-pass block timeline of column dbg_ccol
  int dbg_ccol = -1;
  int nranks = 1;
  int rank = 0;
  // halo ranges of the row-partitioned SpMV (sqb_ctx_set_halo): [P][P][2]
  std::vector<int64_t> halo;
  // host-buffer entry points (host_pipe.cu): device copies of the caller's
  // host operands and transfer staging live in a second grow-only arena;
  // copy-engine streams run the H2D / D2H pipelines beside ctx->stream
  sqb::SweepHooks* hooks = nullptr;
  void* big = nullptr;
  size_t big_bytes = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaStream_t s_aux[4] = {nullptr, nullptr, nullptr, nullptr};  // streamed-sketch compute streams
  // in-kernel peer-memory exchange of the row-partitioned sweep (sqb_p2p_*):
  // every rank's mailbox is mapped into every peer (CUDA IPC over NVLink), a
  // rank's partials are stored straight into the peers' mailboxes and
  // published with a release flag the consuming kernel acquires
  int p2p_on = 0;
  int p2p_nranks = 0;
  int64_t p2p_count = 0;                // doubles per (parity, rank) slot
  std::vector<void*> p2p_local;         // own mailbox(es): 1, or nranks for virtual ranks
  std::vector<void*> p2p_opened;        // IPC-opened peer mailboxes
  std::vector<void*> p2p_absent;        // stand-ins for peers that never answer (fault injection)
  void** p2p_table = nullptr;           // device [n_local][nranks] mailbox bases
  unsigned long long p2p_seq = 0;       // exchanges so far (identical on every rank)
  // page-locked staging ring for PAGEABLE host operands (host_pipe.cu: staged_h2d)
  void* pg_slot[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t pg_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t pg_bytes = 0;
  unsigned pg_next = 0;
};

namespace sqb {

// Opt-in dynamic shared memory of a kernel.  The limit is a property of the
// kernel on the device, shared by every host thread and context: setting it to
// each call's own size races (thread A raises it, thread B lowers it, A's
// launch then fails with cudaErrorCooperativeLaunchTooLarge / invalid value).
// It is therefore set ONCE per (device, kernel) to the opt-in maximum less the
// kernel's static shared memory, and never lowered.
template <typename K>
inline cudaError_t allow_dyn_smem(K kern, size_t needed) {
  static std::mutex mu;
  static std::unordered_map<unsigned long long, int> limit;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long key = (unsigned long long)reinterpret_cast<uintptr_t>(reinterpret_cast<const void*>(kern)) ^
                                 ((unsigned long long)dev << 56);
  std::lock_guard<std::mutex> g(mu);
  auto it = limit.find(key);
  if (it == limit.end()) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int lim = optin - (int)fa.sharedSizeBytes;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
    if (e != cudaSuccess) return e;
    it = limit.emplace(key, lim).first;
  }
  return needed <= (size_t)it->second ? cudaSuccess : cudaErrorInvalidValue;
}

inline int set_error(sqb_ctx* ctx, int code, const char* fmt, ...) {
  if (ctx) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
    va_end(ap);
  }
  return code;
}

inline int set_cuda_error(sqb_ctx* ctx, cudaError_t e, const char* what, const char* file, int line) {
  return set_error(ctx, SQB_ERR_CUDA, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                   cudaGetErrorString(e), file, line, what);
}

// Bump allocator over the context workspace.  All requests of one call are
// made up front (plan), then the workspace grows once if needed.
struct WsPlan {
  std::vector<size_t> offs;
  size_t total = 0;
  size_t add(size_t bytes) {
    size_t o = (total + 255) & ~size_t(255);
    offs.push_back(o);
    total = o + bytes;
    return offs.size() - 1;
  }
};

inline int ws_reserve(sqb_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return SQB_OK;
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ctx->ws) SQB_CUDA_TRY(cudaFree(ctx->ws));
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  size_t want = bytes + (bytes >> 3);
  SQB_CUDA_TRY(cudaMalloc(&ctx->ws, want));
  ctx->ws_bytes = want;
  return SQB_OK;
}

template <typename P>
inline P* ws_ptr(sqb_ctx* ctx, const WsPlan& plan, size_t id) {
  return reinterpret_cast<P*>(static_cast<char*>(ctx->ws) + plan.offs[id]);
}

// bracket one launch of the profiled kernel with events (no-op when off)
inline void prof_begin(sqb_ctx* ctx) {
  if (!ctx->prof) return;
  if (ctx->prof_used + 2 > ctx->prof_ev.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->prof_ev.push_back(e);
    }
  }
  cudaEventRecord(ctx->prof_ev[ctx->prof_used], ctx->stream);
}
inline void prof_end(sqb_ctx* ctx, double alg_bytes) {
  if (!ctx->prof) return;
  cudaEventRecord(ctx->prof_ev[ctx->prof_used + 1], ctx->stream);
  ctx->prof_used += 2;
  ctx->prof_bytes.push_back(alg_bytes);
}

inline void trace_mark(sqb_ctx* ctx, const char* what) {
  if (ctx->trace_used >= ctx->trace_ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ctx->trace_ev.push_back(e);
    }
  }
  cudaEventRecord(ctx->trace_ev[ctx->trace_used++], ctx->stream);
  ctx->trace_name.push_back(what);
}

inline int check_launch(sqb_ctx* ctx, const char* what) {
  ctx->launches++;
  if (ctx->trace) trace_mark(ctx, what);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(ctx, e, what, __FILE__, __LINE__);
  return SQB_OK;
}

// Start of a computing entry point: clear the error text and the device
// status word on ctx->stream, so a failure left by an earlier unchecked call
// cannot turn this call's kernels into early-returning no-ops.
inline int begin_entry(sqb_ctx* ctx) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  ctx->top_pending = false;  // a deferred copy_top never outlives the call that deferred it
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  SQB_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(Status), ctx->stream));
  return SQB_OK;
}

// host-side rounding of a double to a storage format, matching numpy:
// float32/float16 round directly from double; ml_dtypes' bfloat16 goes
// through float32 (two round-to-nearest-even steps).
double round_scalar(int dtype, double x);

}  // namespace sqb

#define SQB_TRY(expr)              \
  do {                             \
    int r__ = (expr);              \
    if (r__ != SQB_OK) return r__; \
  } while (0)
