// Host-buffer entry points: the reference's call shape (numpy W in, numpy
// factors out, rhqr.py:254-267) with the PCIe transfers overlapped with the
// device factorization.
//
//   H2D   W arrives on the copy stream s_in.  A column-major host W streams in
//         column groups: the sweep (rhqr_left.cu, ensure_y0) waits for a
//         group only when pass c first needs y0_{c+1}, so the upload of
//         later columns overlaps the factorization of earlier ones.  A
//         row-major (C-order) host W can only be complete after its last row
//         block, so it streams in row blocks through two device staging slots
//         (transpose + rounding kernel per block) ahead of the whole sweep.
//   D2H   U[:, c] is final once pass c+1 has rewritten it (lazy scaling,
//         rhqr_kernels.cuh); the sweep calls col_final(c) after enqueuing that
//         pass and every group of columns is copied back on s_out while later
//         columns are still being factored.  S, T, R and the scalars follow
//         the finish kernel.
//
// The device copies of W and U are context scratch (a grow-only arena),
// never caller memory.  Host buffers should be page-locked for full PCIe
// bandwidth (the facade allocates its outputs that way); pageable buffers
// work but the driver stages them synchronously.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "sketch.cuh"

#include "dense.cuh"

namespace sqb {

int rec_rhqr_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t, void*,
                      int64_t, double*, int64_t, double*, int64_t, double*, int64_t, double*, double*, double*);
template <typename T>
int rec_finish_t(sqb_ctx* ctx, int scaling, const double* Z, int64_t od, int64_t m, const T* W2, int64_t n2,
                 int64_t ldw, T* U2, int64_t ldu, T* Utop, int64_t ldutop, double* S, int64_t lds, double* Tm,
                 int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* M,
                 double* X);

int rhqr_left_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t,
                       void*, int64_t, double*, int64_t, double*, int64_t, double*, int64_t, double*,
                       double*, double*);

// ---------------------------------------------------------------------------
// conversion kernels: fp64 host layout -> column-major storage dtype (the
// round_to of rhqr.py:264, precision.py:34-51: a finite value that overflows
// the storage format is a PrecisionRangeError, reported through the status
// word with the largest offending magnitude).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T round_store(double x, Status* st) {
  const auto r = Lo<T>::from_double(x);
  if (isfinite(x) && !isfinite((double)r)) {
    fail(st, SQB_ERR_RANGE, 0, 0.0);
    atomicMax(reinterpret_cast<unsigned long long*>(&st->val),
              (unsigned long long)__double_as_longlong(fabs(x)));
  }
  return Lo<T>::store(r);
}

// rows [0, R) of a row-major block (ld lds) -> dst[i + j*ldd], 32x32 tiles
template <typename T>
__global__ void __launch_bounds__(256) rowblock_to_colmajor(const double* __restrict__ src, int64_t lds,
                                                            int64_t R, int64_t m, T* __restrict__ dst,
                                                            int64_t ldd, Status* st) {
  __shared__ double tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + tx;
    tile[r][tx] = (i < R && j < m) ? src[i * lds + j] : 0.0;
  }
  __syncthreads();
  for (int c = ty; c < 32; c += 8) {
    const int64_t i = i0 + tx, j = j0 + c;
    if (i < R && j < m) dst[i + j * ldd] = round_store<T>(tile[tx][c], st);
  }
}

// column-major fp64 block (ld lds) -> column-major storage dtype
template <typename T>
__global__ void colblock_convert(const double* __restrict__ src, int64_t lds, int64_t R, int64_t k,
                                 T* __restrict__ dst, int64_t ldd, Status* st) {
  const int64_t tot = R * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % R, j = e / R;
    dst[i + j * ldd] = round_store<T>(src[i + j * lds], st);
  }
}

// column-major storage dtype -> fp64 (the float64 arrays the reference returns)
template <typename T>
__global__ void colblock_widen(const T* __restrict__ src, int64_t lds, int64_t R, int64_t k,
                               double* __restrict__ dst, int64_t ldd) {
  const int64_t tot = R * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % R, j = e / R;
    dst[i + j * ldd] = (double)Lo<T>::load(src[i + j * lds]);
  }
}

static size_t esize(int code) { return code == SQB_F64 ? 8 : code == SQB_F32 ? 4 : 2; }

template <typename F>
static int by_dtype(int code, F&& f) {
  switch (code) {
    case SQB_F64: return f(double());
    case SQB_F32: return f(float());
    case SQB_F16: return f(__half());
    case SQB_BF16: return f(__nv_bfloat16());
  }
  return SQB_ERR_ARG;
}

static int ensure_streams(sqb_ctx* ctx) {
  if (!ctx->s_in) SQB_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
  if (!ctx->s_out) SQB_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
  return SQB_OK;
}

static int big_reserve(sqb_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->big_bytes) return SQB_OK;
  SQB_CUDA_TRY(cudaDeviceSynchronize());
  if (ctx->big) SQB_CUDA_TRY(cudaFree(ctx->big));
  ctx->big = nullptr;
  ctx->big_bytes = 0;
  SQB_CUDA_TRY(cudaMalloc(&ctx->big, bytes));
  ctx->big_bytes = bytes;
  return SQB_OK;
}

struct EventPool {
  std::vector<cudaEvent_t> ev;
  cudaEvent_t get() {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ev.push_back(e);
    return e;
  }
  ~EventPool() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// leading dimension / base shift of a device column-major buffer so that row
// `align_row` of every column is 16-byte aligned (devarray.empty_colmajor)
struct DevLayout {
  int64_t ld, shift;  // elements
  size_t bytes;
};
static DevLayout dev_layout(int64_t rows, int64_t cols, int code, int64_t align_row) {
  const int64_t vn = 16 / (int64_t)esize(code);
  DevLayout L;
  L.ld = std::max<int64_t>(16, (rows + 15) / 16 * 16);
  L.shift = ((-align_row) % vn + vn) % vn;
  L.bytes = (size_t)(L.ld * std::max<int64_t>(cols, 1) + L.shift + vn) * esize(code);
  return L;
}

// ---------------------------------------------------------------------------
// Host -> device copy of a contiguous range that may live in PAGEABLE memory
// (the ndarray a caller of the reference passes).  cudaMemcpyAsync from
// pageable memory is staged by the driver through one bounce buffer,
// synchronously, at a fraction of the PCIe rate; here the range goes through
// a ring of four page-locked slots filled by a few host threads, so the CPU
// copy of slot k+1 runs under the DMA of slot k.  Page-locked sources take the
// plain asynchronous copy.
// ---------------------------------------------------------------------------
static bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

// A small pool of host threads that lives for the process (leaked on purpose:
// no static-destruction order to get wrong); one memcpy job at a time, split in
// page-aligned parts.  Spawning threads per 16 MB slot cost ~10 ms per GiB.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();
    return *p;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (4u << 20) || workers_ == 0) {
      memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);  // one job at a time (contexts on several threads share the pool)
    const unsigned parts = workers_ + 1;
    const size_t part = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
    {
      std::lock_guard<std::mutex> g(mu_);
      dst_ = (char*)dst; src_ = (const char*)src; bytes_ = bytes; part_ = part;
      pending_ = workers_;
      ++gen_;
    }
    cv_.notify_all();
    memcpy(dst, src, std::min(part, bytes));  // part 0 on the calling thread
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    const unsigned hc = std::thread::hardware_concurrency();
    workers_ = std::max(1u, std::min(8u, hc ? hc / 2 : 4u)) - 1;
    for (unsigned t = 0; t < workers_; ++t) std::thread([this, t] { run(t + 1); }).detach();
  }
  void run(unsigned idx) {
    unsigned long long seen = 0;
    for (;;) {
      char* d; const char* sp; size_t n, part;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        d = dst_; sp = src_; n = bytes_; part = part_;
      }
      const size_t o = (size_t)idx * part;
      if (o < n) memcpy(d + o, sp + o, std::min(part, n - o));
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  unsigned workers_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, part_ = 0;
};

static void parallel_memcpy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

static int staged_h2d(sqb_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s, bool pinned) {
  if (pinned || bytes < (1u << 20)) {
    SQB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return SQB_OK;
  }
  if (!ctx->pg_bytes) {
    const size_t slot = 16u << 20;
    for (int k = 0; k < 4; ++k) {
      SQB_CUDA_TRY(cudaHostAlloc(&ctx->pg_slot[k], slot, cudaHostAllocDefault));
      SQB_CUDA_TRY(cudaEventCreateWithFlags(&ctx->pg_ev[k], cudaEventDisableTiming));
    }
    ctx->pg_bytes = slot;
  }
  for (size_t o = 0; o < bytes; o += ctx->pg_bytes) {
    const unsigned k = ctx->pg_next++ & 3u;
    const size_t nb = std::min(ctx->pg_bytes, bytes - o);
    SQB_CUDA_TRY(cudaEventSynchronize(ctx->pg_ev[k]));  // the slot's previous DMA has drained (no-op when unused)
    parallel_memcpy(ctx->pg_slot[k], (const char*)src + o, nb);
    SQB_CUDA_TRY(cudaMemcpyAsync((char*)dst + o, ctx->pg_slot[k], nb, cudaMemcpyHostToDevice, s));
    SQB_CUDA_TRY(cudaEventRecord(ctx->pg_ev[k], s));
  }
  return SQB_OK;
}

struct HostPipe : SweepHooks {
  sqb_ctx* ctx = nullptr;
  EventPool* evp = nullptr;
  int code = SQB_F64;
  int64_t N = 0, m = 0;
  // input
  const double* Wh = nullptr;
  int64_t ldwh = 0;
  bool w_pinned = true;           // false: W is pageable, uploads go through the staging ring (staged_h2d)
  void* Wd = nullptr;
  int64_t ldwd = 0;
  double* stage_in[2] = {nullptr, nullptr};
  int64_t stage_in_elems = 0;
  int64_t gin = 8;               // columns per input group (column-major input)
  std::vector<cudaEvent_t> ev_in;  // per input group, recorded after the group is resident
  // output
  double* Uh = nullptr;
  int64_t lduh = 0;
  const void* Ud = nullptr;
  int64_t ldud = 0;
  double* stage_out[2] = {nullptr, nullptr};
  int64_t gout = 8;
  int64_t out_done = 0;
  int out_slot = 0;

  int issue_input_colmajor() {
    // column groups: a direct 2D copy for fp64 storage, staging + rounding otherwise
    const size_t es = esize(code);
    const int64_t ngrp = (m + gin - 1) / gin;
    ev_in.resize(ngrp);
    for (int64_t g = 0; g < ngrp; ++g) {
      const int64_t c0 = g * gin, k = std::min(gin, m - c0);
      if (code == SQB_F64) {
        if (w_pinned) {
          SQB_CUDA_TRY(cudaMemcpy2DAsync((char*)Wd + c0 * ldwd * es, ldwd * es, Wh + c0 * ldwh,
                                         ldwh * sizeof(double), N * sizeof(double), k, cudaMemcpyHostToDevice,
                                         ctx->s_in));
        } else {
          for (int64_t c = c0; c < c0 + k; ++c)
            SQB_TRY(staged_h2d(ctx, (char*)Wd + c * ldwd * es, Wh + c * ldwh, N * sizeof(double), ctx->s_in, false));
        }
      } else {
        double* sbuf = stage_in[g & 1];
        if (w_pinned) {
          SQB_CUDA_TRY(cudaMemcpy2DAsync(sbuf, N * sizeof(double), Wh + c0 * ldwh, ldwh * sizeof(double),
                                         N * sizeof(double), k, cudaMemcpyHostToDevice, ctx->s_in));
        } else {
          for (int64_t c = 0; c < k; ++c)
            SQB_TRY(staged_h2d(ctx, sbuf + c * N, Wh + (c0 + c) * ldwh, N * sizeof(double), ctx->s_in, false));
        }
        const unsigned gb = (unsigned)std::min<int64_t>((N * k + 255) / 256, 4 * ctx->sm_count);
        SQB_TRY(by_dtype(code, [&](auto t) {
          using T = decltype(t);
          colblock_convert<T><<<gb, 256, 0, ctx->s_in>>>(sbuf, N, N, k, (T*)Wd + c0 * ldwd, ldwd, ctx->d_status);
          return check_launch(ctx, "colblock_convert");
        }));
      }
      ev_in[g] = evp->get();
      SQB_CUDA_TRY(cudaEventRecord(ev_in[g], ctx->s_in));
    }
    streamed_input = true;
    return SQB_OK;
  }

  int issue_input_rowmajor() {
    // row blocks through two staging slots; copy and transpose share s_in,
    // so slot reuse is ordered without extra events
    const int64_t rb = std::max<int64_t>(1, stage_in_elems / std::max<int64_t>(ldwh, 1));
    int slot = 0;
    for (int64_t r0 = 0; r0 < N; r0 += rb, slot ^= 1) {
      const int64_t R = std::min(rb, N - r0);
      SQB_TRY(staged_h2d(ctx, stage_in[slot], Wh + r0 * ldwh, (size_t)R * ldwh * sizeof(double), ctx->s_in, w_pinned));
      dim3 grid((unsigned)((R + 31) / 32), (unsigned)((m + 31) / 32));
      SQB_TRY(by_dtype(code, [&](auto t) {
        using T = decltype(t);
        rowblock_to_colmajor<T><<<grid, 256, 0, ctx->s_in>>>(stage_in[slot], ldwh, R, m, (T*)Wd + r0, ldwd,
                                                             ctx->d_status);
        return check_launch(ctx, "rowblock_to_colmajor");
      }));
    }
    cudaEvent_t e = evp->get();
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->s_in));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, e, 0));
    streamed_input = false;
    return SQB_OK;
  }

  int64_t wait_cols(sqb_ctx* c, int64_t upto) override {
    const int64_t g = (upto - 1) / gin;
    cudaStreamWaitEvent(c->stream, ev_in[g], 0);
    return std::min(m, (g + 1) * gin);
  }

  int flush_out(int64_t end) {
    // U[:, out_done:end] are final on ctx->stream
    if (end <= out_done) return SQB_OK;
    cudaEvent_t e = evp->get();
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->stream));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, e, 0));
    const int64_t c0 = out_done, k = end - out_done;
    if (code == SQB_F64) {
      SQB_CUDA_TRY(cudaMemcpy2DAsync(Uh + c0 * lduh, lduh * sizeof(double), (const double*)Ud + c0 * ldud,
                                     ldud * sizeof(double), N * sizeof(double), k, cudaMemcpyDeviceToHost,
                                     ctx->s_out));
    } else {
      double* sbuf = stage_out[out_slot];
      out_slot ^= 1;
      const unsigned gb = (unsigned)std::min<int64_t>((N * k + 255) / 256, 4 * ctx->sm_count);
      SQB_TRY(by_dtype(code, [&](auto t) {
        using T = decltype(t);
        colblock_widen<T><<<gb, 256, 0, ctx->s_out>>>((const T*)Ud + c0 * ldud, ldud, N, k, sbuf, N);
        return check_launch(ctx, "colblock_widen");
      }));
      SQB_CUDA_TRY(cudaMemcpy2DAsync(Uh + c0 * lduh, lduh * sizeof(double), sbuf, N * sizeof(double),
                                     N * sizeof(double), k, cudaMemcpyDeviceToHost, ctx->s_out));
    }
    out_done = end;
    return SQB_OK;
  }

  int col_final(sqb_ctx*, int64_t c) override {
    if (c + 1 - out_done >= gout || c + 1 == m) return flush_out(c + 1);
    return SQB_OK;
  }
};

}  // namespace sqb

using namespace sqb;

extern "C" int sqb_rhqr_left_host(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                                  const double* W, int64_t N, int64_t m, int64_t ldw, int w_layout,
                                  double* U, int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt,
                                  double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  if (lo_dtype < SQB_F64 || lo_dtype > SQB_BF16) return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
  // the same argument checks as sqb_rhqr_left, before sk is dereferenced
  SQB_TRY(validate_left_args(ctx, sk, scaling, N, m));
  if (!W || !U || !S || !T || !R || !sigmas || !rhos || !betas)
    return set_error(ctx, SQB_ERR_ARG, "null host buffer");
  if (N < 1 || m < 1) return set_error(ctx, SQB_ERR_ARG, "empty matrix");
  const bool rowmajor = w_layout == 0;
  if (w_layout != 0 && w_layout != 1) return set_error(ctx, SQB_ERR_ARG, "unknown layout %d", w_layout);
  if ((rowmajor && ldw < m) || (!rowmajor && ldw < N) || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  SQB_TRY(ensure_streams(ctx));

  // device scratch: W, U (column-major, row m 16-byte aligned), S, T, R,
  // scalars, input/output staging
  const DevLayout LW = dev_layout(N, m, lo_dtype, m), LU = LW;
  const int64_t od = m + sk->ell;
  const int64_t stage_in_elems =
      lo_dtype == SQB_F64 && !rowmajor ? 0 : std::max<int64_t>(rowmajor ? 4 * ldw : 8 * N, (int64_t)(32ll << 20) / 8);
  const int64_t gout = 8;
  const int64_t stage_out_elems = lo_dtype == SQB_F64 ? 0 : gout * N;
  WsPlan plan;
  const size_t iW = plan.add(LW.bytes), iU = plan.add(LU.bytes);
  const size_t iS = plan.add(sizeof(double) * od * m), iT = plan.add(sizeof(double) * m * m),
               iR = plan.add(sizeof(double) * m * m), iX = plan.add(sizeof(double) * 3 * m);
  const size_t iI0 = plan.add(sizeof(double) * stage_in_elems), iI1 = plan.add(sizeof(double) * stage_in_elems);
  const size_t iO0 = plan.add(sizeof(double) * stage_out_elems), iO1 = plan.add(sizeof(double) * stage_out_elems);
  SQB_TRY(big_reserve(ctx, plan.total + 256));
  char* base = static_cast<char*>(ctx->big);
  const size_t es = esize(lo_dtype);
  void* Wd = base + plan.offs[iW] + LW.shift * es;
  void* Ud = base + plan.offs[iU] + LU.shift * es;
  double* Sd = reinterpret_cast<double*>(base + plan.offs[iS]);
  double* Td = reinterpret_cast<double*>(base + plan.offs[iT]);
  double* Rd = reinterpret_cast<double*>(base + plan.offs[iR]);
  double* Xd = reinterpret_cast<double*>(base + plan.offs[iX]);

  // the s_in / s_out streams must not run ahead of earlier work on ctx->stream
  // (a previous call may still be reading the arena)
  EventPool evp;
  {
    cudaEvent_t e = evp.get();
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->stream));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, e, 0));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, e, 0));
  }
  SQB_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(Status), ctx->stream));
  {
    cudaEvent_t e = evp.get();  // status cleared before the conversion kernels may set it
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->stream));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, e, 0));
  }

  HostPipe hp;
  hp.ctx = ctx;
  hp.evp = &evp;
  hp.code = lo_dtype;
  hp.N = N;
  hp.m = m;
  hp.Wh = W;
  hp.ldwh = ldw;
  hp.w_pinned = host_is_pinned(W);
  hp.Wd = Wd;
  hp.ldwd = LW.ld;
  hp.stage_in[0] = reinterpret_cast<double*>(base + plan.offs[iI0]);
  hp.stage_in[1] = reinterpret_cast<double*>(base + plan.offs[iI1]);
  hp.stage_in_elems = stage_in_elems;
  hp.gin = std::max<int64_t>(1, std::min<int64_t>(8, stage_in_elems > 0 ? stage_in_elems / N : 8));
  hp.Uh = U;
  hp.lduh = ldu;
  hp.Ud = Ud;
  hp.ldud = LU.ld;
  hp.stage_out[0] = reinterpret_cast<double*>(base + plan.offs[iO0]);
  hp.stage_out[1] = reinterpret_cast<double*>(base + plan.offs[iO1]);
  hp.gout = gout;
  SQB_TRY(rowmajor ? hp.issue_input_rowmajor() : hp.issue_input_colmajor());

  ctx->hooks = &hp;
  int rc = rhqr_left_dispatch(ctx, sk, scaling, lo_dtype, Wd, N, m, LW.ld, Ud, LU.ld, Sd, od, Td, m, Rd, m,
                              Xd, Xd + m, Xd + 2 * m);
  ctx->hooks = nullptr;
  if (rc != SQB_OK) {
    cudaDeviceSynchronize();
    return rc;
  }
  // small factors after the finish kernel
  SQB_CUDA_TRY(cudaMemcpy2DAsync(S, lds * sizeof(double), Sd, od * sizeof(double), od * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpy2DAsync(T, ldt * sizeof(double), Td, m * sizeof(double), m * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpy2DAsync(R, ldr * sizeof(double), Rd, m * sizeof(double), m * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(sigmas, Xd, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(rhos, Xd + m, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(betas, Xd + 2 * m, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->s_out));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SQB_OK;
}

// ---------------------------------------------------------------------------
// rec_rhqr with host operands (rhqr.py:368-395: numpy W in, numpy factors out).
//
//   H2D   W arrives on s_in in row blocks aligned to the split-K slabs of the
//         Gaussian sketch GEMM (K2): each block's slabs start on an auxiliary
//         stream as soon as the block is resident, so the 137 GFLOP sketch
//         runs under the upload; the slab-order reduction then gives Z
//         bitwise as the one-shot launch does.  (SRHT / low-precision
//         sketches: the blocks are uploaded, then the device path runs.)
//   D2H   U streams back after the reconstruction solve (every row of U2
//         depends on Mfac, i.e. on all of W: the two directions cannot overlap).
// ---------------------------------------------------------------------------
extern "C" int sqb_rec_rhqr_host(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const double* W,
                                 int64_t N, int64_t m, int64_t ldw, int w_layout, double* U, int64_t ldu, double* S,
                                 int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas,
                                 double* rhos, double* betas) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  if (lo_dtype < SQB_F64 || lo_dtype > SQB_BF16) return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (!W || !U || !S || !T || !R || !sigmas || !rhos || !betas)
    return set_error(ctx, SQB_ERR_ARG, "null host buffer");
  if (N < 1 || m < 1) return set_error(ctx, SQB_ERR_ARG, "empty matrix");
  if (sk->n != N - m)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld", (long long)sk->n,
                     (long long)(N - m));
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  const bool rowmajor = w_layout == 0;
  if (w_layout != 0 && w_layout != 1) return set_error(ctx, SQB_ERR_ARG, "unknown layout %d", w_layout);
  if ((rowmajor && ldw < m) || (!rowmajor && ldw < N) || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  SQB_TRY(ensure_streams(ctx));
  for (auto& a : ctx->s_aux)
    if (!a) SQB_CUDA_TRY(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));

  const int64_t n = N - m, od = m + sk->ell;
  const bool streamed = sk->kind == SQB_SKETCH_DENSE && lo_dtype == SQB_F64;
  const DevLayout LW = dev_layout(N, m, lo_dtype, m), LU = LW;
  const size_t es = esize(lo_dtype);
  int64_t ks = 0;
  const int nslab = streamed ? dense_slab_plan(sk, m, &ks) : 0;
  // input blocks: whole slab groups (streamed) or ~32 MB row blocks
  const int64_t blk_rows = streamed ? ks * std::max<int64_t>(1, ((int64_t)(48ll << 20) / (8 * m)) / ks)
                                    : std::max<int64_t>(1024, (int64_t)(32ll << 20) / (8 * m));
  const bool staged_in = rowmajor || lo_dtype != SQB_F64;
  const int64_t stage_in_elems = staged_in ? (blk_rows + m) * (rowmajor ? std::max(ldw, m) : m) : 0;
  const int64_t stage_out_elems = lo_dtype == SQB_F64 ? 0 : N * std::min<int64_t>(m, 8);
  WsPlan plan;
  const size_t iW = plan.add(LW.bytes), iU = plan.add(LU.bytes);
  const size_t iS = plan.add(sizeof(double) * od * m), iT = plan.add(sizeof(double) * m * m),
               iR = plan.add(sizeof(double) * m * m), iX = plan.add(sizeof(double) * 3 * m);
  const size_t iZ = plan.add(sizeof(double) * od * m), iM = plan.add(sizeof(double) * m * m);
  const size_t iP = plan.add(streamed ? sizeof(double) * (size_t)nslab * sk->ell * m : 8);
  const size_t iXs = plan.add(m > 64 ? sizeof(double) * n * m : 8);
  const size_t iI0 = plan.add(sizeof(double) * stage_in_elems), iI1 = plan.add(sizeof(double) * stage_in_elems);
  const size_t iO = plan.add(sizeof(double) * stage_out_elems);
  SQB_TRY(big_reserve(ctx, plan.total + 256));
  char* base = static_cast<char*>(ctx->big);
  void* Wd = base + plan.offs[iW] + LW.shift * es;
  void* Ud = base + plan.offs[iU] + LU.shift * es;
  double* Sd = reinterpret_cast<double*>(base + plan.offs[iS]);
  double* Td = reinterpret_cast<double*>(base + plan.offs[iT]);
  double* Rd = reinterpret_cast<double*>(base + plan.offs[iR]);
  double* Xd = reinterpret_cast<double*>(base + plan.offs[iX]);
  double* Zd = reinterpret_cast<double*>(base + plan.offs[iZ]);
  double* Md = reinterpret_cast<double*>(base + plan.offs[iM]);
  void* Pd = base + plan.offs[iP];
  double* stage_in[2] = {reinterpret_cast<double*>(base + plan.offs[iI0]),
                         reinterpret_cast<double*>(base + plan.offs[iI1])};
  double* stage_out = reinterpret_cast<double*>(base + plan.offs[iO]);
  Status* st = ctx->d_status;

  EventPool evp;
  {  // side streams must not run ahead of earlier work on ctx->stream (arena reuse)
    cudaEvent_t e = evp.get();
    SQB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(Status), ctx->stream));
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->stream));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_in, e, 0));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, e, 0));
    for (auto a : ctx->s_aux) SQB_CUDA_TRY(cudaStreamWaitEvent(a, e, 0));
  }
  // ---- upload in row blocks [r0, r1) of W (block 0 also carries the m identity rows)
  const bool w_pinned = host_is_pinned(W);  // a pageable row-major W goes through the staging ring
  std::vector<cudaEvent_t> done;
  int slot = 0, z = 0;
  for (int64_t r0 = 0, b = 0; r0 < N; ++b, slot ^= 1) {
    const int64_t r1 = std::min(N, (b == 0 ? m : r0) + blk_rows);
    const int64_t R = r1 - r0;
    if (rowmajor) {
      SQB_TRY(staged_h2d(ctx, stage_in[slot], W + r0 * ldw, (size_t)R * ldw * sizeof(double), ctx->s_in, w_pinned));
      dim3 grid((unsigned)((R + 31) / 32), (unsigned)((m + 31) / 32));
      SQB_TRY(by_dtype(lo_dtype, [&](auto t) {
        using TT = decltype(t);
        rowblock_to_colmajor<TT><<<grid, 256, 0, ctx->s_in>>>(stage_in[slot], ldw, R, m, (TT*)Wd + r0, LW.ld, st);
        return check_launch(ctx, "rowblock_to_colmajor");
      }));
    } else if (lo_dtype == SQB_F64) {
      SQB_CUDA_TRY(cudaMemcpy2DAsync((double*)Wd + r0, LW.ld * sizeof(double), W + r0, ldw * sizeof(double),
                                     R * sizeof(double), m, cudaMemcpyHostToDevice, ctx->s_in));
    } else {
      SQB_CUDA_TRY(cudaMemcpy2DAsync(stage_in[slot], R * sizeof(double), W + r0, ldw * sizeof(double),
                                     R * sizeof(double), m, cudaMemcpyHostToDevice, ctx->s_in));
      const unsigned gb = (unsigned)std::min<int64_t>((R * m + 255) / 256, 4 * ctx->sm_count);
      SQB_TRY(by_dtype(lo_dtype, [&](auto t) {
        using TT = decltype(t);
        colblock_convert<TT><<<gb, 256, 0, ctx->s_in>>>(stage_in[slot], R, R, m, (TT*)Wd + r0, LW.ld, st);
        return check_launch(ctx, "colblock_convert");
      }));
    }
    cudaEvent_t e = evp.get();
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->s_in));
    if (streamed) {
      // slabs whose Omega rows [z ks, (z+1) ks) are now resident
      const int zend = r1 >= N ? nslab : (int)std::min<int64_t>(nslab, (r1 - m) / ks);
      if (zend > z) {
        cudaStream_t cs = ctx->s_aux[b % 4];
        SQB_CUDA_TRY(cudaStreamWaitEvent(cs, e, 0));
        SQB_TRY(launch_dense_slabs(ctx, cs, sk, (const double*)Wd + m, LW.ld, m, z, zend, ks, Pd, st));
        cudaEvent_t e2 = evp.get();
        SQB_CUDA_TRY(cudaEventRecord(e2, cs));
        done.push_back(e2);
        z = zend;
      }
    }
    done.push_back(e);
    r0 = r1;
  }
  for (cudaEvent_t e : done) SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, e, 0));
  // ---- sketch-space work and the reconstruction on ctx->stream
  int rc = SQB_OK;
  if (streamed) {
    rc = launch_copy_top(ctx, SQB_F64, Wd, LW.ld, m, m, Zd, od, st);
    if (rc == SQB_OK) rc = launch_dense_reduce(ctx, sk, m, nslab, Pd, Zd, od, m, st);
    if (rc == SQB_OK)
      rc = rec_finish_t<double>(ctx, scaling, Zd, od, m, (const double*)Wd + m, n, LW.ld, (double*)Ud + m, LU.ld,
                                (double*)Ud, LU.ld, Sd, od, Td, m, Rd, m, Xd, Xd + m, Xd + 2 * m, Md,
                                reinterpret_cast<double*>(base + plan.offs[iXs]));
  } else {
    rc = rec_rhqr_dispatch(ctx, sk, scaling, lo_dtype, Wd, N, m, LW.ld, Ud, LU.ld, Sd, od, Td, m, Rd, m, Xd, Xd + m,
                           Xd + 2 * m);
  }
  if (rc != SQB_OK) {
    cudaDeviceSynchronize();
    return rc;
  }
  // ---- download U (float64, column-major host) on s_out, small factors on ctx->stream
  {
    cudaEvent_t e = evp.get();
    SQB_CUDA_TRY(cudaEventRecord(e, ctx->stream));
    SQB_CUDA_TRY(cudaStreamWaitEvent(ctx->s_out, e, 0));
    if (lo_dtype == SQB_F64) {
      SQB_CUDA_TRY(cudaMemcpy2DAsync(U, ldu * sizeof(double), Ud, LU.ld * sizeof(double), N * sizeof(double), m,
                                     cudaMemcpyDeviceToHost, ctx->s_out));
    } else {
      const int64_t g = std::min<int64_t>(m, 8);
      for (int64_t c0 = 0; c0 < m; c0 += g) {
        const int64_t k = std::min(g, m - c0);
        const unsigned gb = (unsigned)std::min<int64_t>((N * k + 255) / 256, 4 * ctx->sm_count);
        SQB_TRY(by_dtype(lo_dtype, [&](auto t) {
          using TT = decltype(t);
          colblock_widen<TT><<<gb, 256, 0, ctx->s_out>>>((const TT*)Ud + c0 * LU.ld, LU.ld, N, k, stage_out, N);
          return check_launch(ctx, "colblock_widen");
        }));
        SQB_CUDA_TRY(cudaMemcpy2DAsync(U + c0 * ldu, ldu * sizeof(double), stage_out, N * sizeof(double),
                                       N * sizeof(double), k, cudaMemcpyDeviceToHost, ctx->s_out));
      }
    }
  }
  SQB_CUDA_TRY(cudaMemcpy2DAsync(S, lds * sizeof(double), Sd, od * sizeof(double), od * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpy2DAsync(T, ldt * sizeof(double), Td, m * sizeof(double), m * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpy2DAsync(R, ldr * sizeof(double), Rd, m * sizeof(double), m * sizeof(double), m,
                                 cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(sigmas, Xd, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(rhos, Xd + m, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaMemcpyAsync(betas, Xd + 2 * m, m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->s_out));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return SQB_OK;
}
