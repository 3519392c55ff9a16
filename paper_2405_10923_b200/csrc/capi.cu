// extern "C" entry points (include/sketchqr_b200.h).
#include <cstring>

#include "sketch.cuh"

namespace sqb {
int rhqr_left_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t,
                       void*, int64_t, double*, int64_t, double*, int64_t, double*, int64_t, double*,
                       double*, double*);
int apply_reflectors_dispatch(sqb_ctx*, const sqb_sketch*, int64_t, int, const void*, int64_t, int64_t,
                              int64_t, const double*, int64_t, const double*, int64_t, int, const void*,
                              int64_t, int64_t, void*, int64_t, void*);
int thin_q_dispatch(sqb_ctx*, int, const void*, int64_t, int64_t, int64_t, const double*, int64_t,
                    double*, int64_t);
int gram_run(sqb_ctx*, const double*, int64_t, int64_t, int64_t, double*, int64_t);
int residual_norms_run(sqb_ctx*, const double*, int64_t, const double*, int64_t, const double*, int64_t,
                       int64_t, int64_t, int64_t, double*);
int sketch_q_run(sqb_ctx*, int, const void*, int64_t, int64_t, const double*, int64_t, const double*,
                 int64_t, int64_t, double*, int64_t);
int rhqr_block_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t, int64_t,
                        void*, int64_t, double*, int64_t, double*, int64_t, double*, int64_t, double*, double*,
                        double*);
int trim_left_dispatch(sqb_ctx*, const sqb_sketch*, const double*, int64_t, const double*, int64_t, int, int, const void*,
                       int64_t, int64_t, int64_t, void*, int64_t, double*, int64_t, double*, int64_t, double*,
                       int64_t, double*, int64_t, double*, int64_t, double*, double*, double*);
int trim_right_dispatch(sqb_ctx*, const sqb_sketch*, const double*, int64_t, const double*, int64_t, int, int, const void*,
                        int64_t, int64_t, int64_t, void*, int64_t, double*, int64_t, double*, int64_t, double*,
                        int64_t, double*, int64_t, double*, int64_t, double*, double*, double*);
int colscaled_apply_dispatch(sqb_ctx*, const sqb_sketch*, const double*, int64_t, int, const void*, int64_t,
                             int64_t, double*, int64_t);
int trim_thin_q_impl(sqb_ctx*, int, const void*, int64_t, int64_t, int64_t, const double*, int64_t,
                     const double*, int64_t, const double*, int64_t, int64_t, double*, int64_t);
int t_factor_impl(sqb_ctx*, const double*, int64_t, int64_t, int64_t, double*, int64_t);
int upper_tri_solve_impl(sqb_ctx*, const double*, int64_t, int64_t, const double*, int64_t, int64_t, double*, int64_t);
int rhqr_right_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t, void*,
                        int64_t, double*, int64_t, double*, int64_t, double*, double*, double*);
int rec_rhqr_dispatch(sqb_ctx*, const sqb_sketch*, int, int, const void*, int64_t, int64_t, int64_t, void*,
                      int64_t, double*, int64_t, double*, int64_t, double*, int64_t, double*, double*, double*);
int rh_vector_dispatch(sqb_ctx*, int, int, const void*, int64_t, const double*, int64_t, int64_t, void*,
                       double*, double*);
}  // namespace sqb

using namespace sqb;

static int check_dtype(sqb_ctx* ctx, int dtype) {
  if (dtype < SQB_F64 || dtype > SQB_BF16) return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", dtype);
  return SQB_OK;
}

static int prep(sqb_ctx* ctx) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  return SQB_OK;
}

extern "C" {

int sqb_version(void) { return 1; }

int sqb_ctx_create(int device, void* stream, sqb_ctx** out) {
  if (!out) return SQB_ERR_ARG;
  *out = nullptr;
  sqb_ctx* ctx = new sqb_ctx();
  ctx->device = device;
  ctx->stream = (cudaStream_t)stream;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->d_status, sizeof(Status));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_status, sizeof(Status));
  if (e == cudaSuccess) e = cudaMemset(ctx->d_status, 0, sizeof(Status));
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) {
    int r = set_cuda_error(ctx, e, "sqb_ctx_create", __FILE__, __LINE__);
    sqb_ctx_destroy(ctx);
    return r;
  }
  *out = ctx;
  return SQB_OK;
}

int sqb_ctx_trim(sqb_ctx* ctx) {
  SQB_TRY(prep(ctx));
  SQB_CUDA_TRY(cudaDeviceSynchronize());
  if (ctx->ws) SQB_CUDA_TRY(cudaFree(ctx->ws));
  if (ctx->big) SQB_CUDA_TRY(cudaFree(ctx->big));
  ctx->ws = ctx->big = nullptr;
  ctx->ws_bytes = ctx->big_bytes = 0;
  return SQB_OK;
}

int sqb_p2p_close(sqb_ctx* ctx);

int sqb_ctx_destroy(sqb_ctx* ctx) {
  if (!ctx) return SQB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->p2p_table || !ctx->p2p_local.empty()) sqb_p2p_close(ctx);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->s_in) cudaStreamSynchronize(ctx->s_in);
  if (ctx->s_out) cudaStreamSynchronize(ctx->s_out);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->big) cudaFree(ctx->big);
  for (cudaStream_t a : ctx->s_aux)
    if (a) {
      cudaStreamSynchronize(a);
      cudaStreamDestroy(a);
    }
  if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
  if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
  for (int k = 0; k < 4; ++k) {
    if (ctx->pg_slot[k]) cudaFreeHost(ctx->pg_slot[k]);
    if (ctx->pg_ev[k]) cudaEventDestroy(ctx->pg_ev[k]);
  }
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  for (cudaEvent_t e : ctx->prof_ev) cudaEventDestroy(e);
  delete ctx;
  return SQB_OK;
}

int sqb_ctx_set_stream(sqb_ctx* ctx, void* stream) {
  if (!ctx) return SQB_ERR_ARG;
  cudaStream_t next = (cudaStream_t)stream;
  if (next != ctx->stream) {
    // the workspace, arena and status word are shared by every stream the
    // context is used on: work enqueued on the new stream must not overtake
    // what the old stream may still be doing with them
    SQB_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaEvent_t e;
    SQB_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaError_t r = cudaEventRecord(e, ctx->stream);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(next, e, 0);
    cudaEventDestroy(e);
    if (r != cudaSuccess) return set_cuda_error(ctx, r, "sqb_ctx_set_stream", __FILE__, __LINE__);
    ctx->stream = next;
  }
  return SQB_OK;
}

const char* sqb_ctx_last_error(sqb_ctx* ctx) { return ctx ? ctx->err : "null context"; }

int64_t sqb_ctx_launches(sqb_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sqb_ctx_profile(sqb_ctx* ctx, int enable) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->prof = enable != 0;
  ctx->prof_used = 0;
  ctx->prof_bytes.clear();
  return SQB_OK;
}

int sqb_ctx_profile_read(sqb_ctx* ctx, double* total_ms, double* total_bytes, int64_t* launches) {
  SQB_TRY(prep(ctx));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  double ms = 0.0, by = 0.0;
  for (size_t i = 0; i < ctx->prof_bytes.size(); ++i) {
    float t = 0.f;
    SQB_CUDA_TRY(cudaEventElapsedTime(&t, ctx->prof_ev[2 * i], ctx->prof_ev[2 * i + 1]));
    ms += t;
    by += ctx->prof_bytes[i];
  }
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = by;
  if (launches) *launches = (int64_t)ctx->prof_bytes.size();
  ctx->prof_used = 0;
  ctx->prof_bytes.clear();
  return SQB_OK;
}

double sqb_round_scalar(int dtype, double x) { return round_scalar(dtype, x); }

int sqb_debug_step_stamps(sqb_ctx* ctx, long long* dev_buf, int column) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->dbg_ts = dev_buf;
  ctx->dbg_col = column;
  return SQB_OK;
}

int sqb_ctx_trace(sqb_ctx* ctx, int enable) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->trace = enable != 0;
  if (enable) {
    ctx->trace_used = 0;
    ctx->trace_name.clear();
    trace_mark(ctx, "(start)");
  }
  return SQB_OK;
}

int sqb_ctx_trace_read(sqb_ctx* ctx, char* buf, int64_t size) {
  SQB_TRY(prep(ctx));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  // per kernel name: launches, summed in-stream time (ms)
  std::vector<const char*> names;
  std::vector<double> ms;
  std::vector<int64_t> cnt;
  for (size_t i = 1; i < ctx->trace_used; ++i) {
    float t = 0.f;
    SQB_CUDA_TRY(cudaEventElapsedTime(&t, ctx->trace_ev[i - 1], ctx->trace_ev[i]));
    size_t k = 0;
    for (; k < names.size(); ++k)
      if (strcmp(names[k], ctx->trace_name[i]) == 0) break;
    if (k == names.size()) { names.push_back(ctx->trace_name[i]); ms.push_back(0.0); cnt.push_back(0); }
    ms[k] += t;
    cnt[k]++;
  }
  int64_t off = 0;
  for (size_t k = 0; k < names.size() && off < size - 1; ++k)
    off += snprintf(buf + off, (size_t)(size - off), "%s %lld %.6f\n", names[k], (long long)cnt[k], ms[k]);
  if (size > 0) buf[std::min<int64_t>(off, size - 1)] = 0;
  return SQB_OK;
}

int sqb_debug_col_stamps(sqb_ctx* ctx, long long* dev_buf, int column) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->dbg_cts = dev_buf;
  ctx->dbg_ccol = column;
  return SQB_OK;
}

int sqb_ctx_status(sqb_ctx* ctx, int* code, int* col, double* val) {
  SQB_TRY(prep(ctx));
  SQB_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(Status), cudaMemcpyDeviceToHost,
                               ctx->stream));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  SQB_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(Status), ctx->stream));
  if (code) *code = ctx->h_status->code;
  if (col) *col = ctx->h_status->col;
  if (val) *val = ctx->h_status->val;
  return SQB_OK;
}

int sqb_sketch_apply(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* X, int64_t ldx,
                     int64_t k, double* Y, int64_t ldy) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (k < 0 || ldx < sk->n || ldy < sk->ell) return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  WsPlan plan;
  const size_t iP = plan.add(sketch_partials_bytes(sk, dtype, k));
  SQB_TRY(ws_reserve(ctx, plan.total));
  return launch_sketch(ctx, sk, dtype, X, ldx, k, Y, ldy, 0, ws_ptr<void>(ctx, plan, iP), ctx->d_status);
}

int sqb_embedded_apply(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, int dtype, const void* X,
                       int64_t ldx, int64_t k, double* Y, int64_t ldy) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (m < 0 || k < 0 || ldx < m + sk->n || ldy < m + sk->ell)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  WsPlan plan;
  const size_t iP = plan.add(sketch_partials_bytes(sk, dtype, k));
  SQB_TRY(ws_reserve(ctx, plan.total));
  SQB_TRY(launch_copy_top(ctx, dtype, X, ldx, m, k, Y, ldy, ctx->d_status));
  return launch_sketch(ctx, sk, dtype, (const char*)X + m * elem_bytes(dtype), ldx, k, Y, ldy, m,
                       ws_ptr<void>(ctx, plan, iP), ctx->d_status);
}

int sqb_rhqr_left(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                  int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                  double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                  double* betas) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_left_args(ctx, sk, scaling, N, m));
  if (ldw < N || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  return rhqr_left_dispatch(ctx, sk, scaling, lo_dtype, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr,
                            sigmas, rhos, betas);
}

int sqb_rhqr_block(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                   int64_t N, int64_t m, int64_t ldw, int64_t block_size, void* U, int64_t ldu, double* S,
                   int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                   double* betas) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (block_size < 1) return set_error(ctx, SQB_ERR_ARG, "block_size must be positive");
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (m > 1024) return set_error(ctx, SQB_ERR_ARG, "m=%lld: the device sweep supports up to 1024 columns", (long long)m);
  if (sk->n != N - m)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld",
                     (long long)sk->n, (long long)(N - m));
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (ldw < N || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  return rhqr_block_dispatch(ctx, sk, scaling, lo_dtype, W, N, m, ldw, block_size, U, ldu, S, lds, T, ldt, R,
                             ldr, sigmas, rhos, betas);
}

int sqb_trim_rhqr_left(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t mscale, const double* E,
                       int64_t lde,
                       int scaling, int lo_dtype, const void* W, int64_t N, int64_t m, int64_t ldw, void* U,
                       int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt, double* Tt, int64_t ldtt,
                       double* R, int64_t ldr, double* L, int64_t ldl, double* sigmas, double* rhos,
                       double* betas) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (sk->n != N)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, W has %lld rows", (long long)sk->n,
                     (long long)N);
  if (m > N) return set_error(ctx, SQB_ERR_ARG, "cannot normalize %lld leading columns of %lld inputs",
                              (long long)m, (long long)N);
  if (!scales || !E || lde < sk->ell) return set_error(ctx, SQB_ERR_ARG, "column-scaled operator without scales/E");
  if (mscale < m || mscale > N)
    return set_error(ctx, SQB_ERR_ARG, "operator normalised over %lld leading columns, W has %lld", (long long)mscale,
                     (long long)m);
  if (ldw < N || ldu < N || lds < sk->ell || ldt < m || ldtt < m || ldr < m || ldl < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  const int64_t esz = lo_dtype == SQB_F64 ? 8 : lo_dtype == SQB_F32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(U) & 15) || (ldu * esz) % 16)
    return set_error(ctx, SQB_ERR_ARG, "U must be 16-byte aligned with a 16-byte multiple leading dimension");
  SQB_TRY(trim_left_dispatch(ctx, sk, scales, mscale, E, lde, scaling, lo_dtype, W, N, m, ldw, U, ldu, S, lds, T, ldt, Tt,
                             ldtt, R, ldr, L, ldl, sigmas, rhos, betas));
  return SQB_OK;
}

int sqb_trim_rhqr_right(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t mscale, const double* E,
                       int64_t lde,
                        int scaling, int lo_dtype, const void* W, int64_t N, int64_t m, int64_t ldw, void* U,
                        int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt, double* Tt, int64_t ldtt,
                        double* R, int64_t ldr, double* L, int64_t ldl, double* sigmas, double* rhos,
                        double* betas) {
  // the same argument contract as sqb_trim_rhqr_left (validated there with a
  // dry run of the checks only)
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (sk->n != N)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, W has %lld rows", (long long)sk->n,
                     (long long)N);
  if (m > N) return set_error(ctx, SQB_ERR_ARG, "cannot normalize %lld leading columns of %lld inputs",
                              (long long)m, (long long)N);
  if (!scales || !E || lde < sk->ell) return set_error(ctx, SQB_ERR_ARG, "column-scaled operator without scales/E");
  if (mscale < m || mscale > N)
    return set_error(ctx, SQB_ERR_ARG, "operator normalised over %lld leading columns, W has %lld", (long long)mscale,
                     (long long)m);
  if (ldw < N || ldu < N || lds < sk->ell || ldt < m || ldtt < m || ldr < m || ldl < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  SQB_TRY(trim_right_dispatch(ctx, sk, scales, mscale, E, lde, scaling, lo_dtype, W, N, m, ldw, U, ldu, S, lds, T, ldt, Tt,
                              ldtt, R, ldr, L, ldl, sigmas, rhos, betas));
  return SQB_OK;
}

int sqb_colscaled_apply(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t m, int dtype,
                        const void* X, int64_t ldx, int64_t k, double* Y, int64_t ldy) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (m < 0 || m > sk->n || !scales) return set_error(ctx, SQB_ERR_ARG, "bad column-scaled operator");
  if (ldx < sk->n || ldy < sk->ell) return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  return colscaled_apply_dispatch(ctx, sk, scales, m, dtype, X, ldx, k, Y, ldy);
}

int sqb_trim_thin_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
                    const double* T, int64_t ldt, const double* S, int64_t lds, const double* E, int64_t lde,
                    int64_t ell, double* Q, int64_t ldq) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  if (k < 0 || k > N || ldu < N || ldq < N || ldt < k || lds < ell || lde < ell)
    return set_error(ctx, SQB_ERR_ARG, "bad trimmed thin-Q arguments");
  return trim_thin_q_impl(ctx, lo_dtype, U, ldu, N, k, T, ldt, S, lds, E, lde, ell, Q, ldq);
}

int sqb_rhqr_right(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                   int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                   double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                   double* betas) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (sk->n != N - m)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld",
                     (long long)sk->n, (long long)(N - m));
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (ldw < N || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  SQB_TRY(rhqr_right_dispatch(ctx, sk, scaling, lo_dtype, W, N, m, ldw, U, ldu, S, lds, R, ldr, sigmas, rhos,
                              betas));
  return t_factor_impl(ctx, S, lds, m + sk->ell, m, T, ldt);
}

int sqb_apply_reflectors(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, int lo_dtype, const void* U,
                         int64_t ldu, int64_t N, int64_t r, const double* S, int64_t lds,
                         const double* T, int64_t ldt, int transpose_t, const void* X, int64_t ldx,
                         int64_t k, void* Out, int64_t ldo) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (sk->n != N - m) return set_error(ctx, SQB_ERR_ARG, "embedding is %lld x %lld, operand has %lld rows",
                                       (long long)(m + sk->ell), (long long)(m + sk->n), (long long)N);
  return apply_reflectors_dispatch(ctx, sk, m, lo_dtype, U, ldu, N, r, S, lds, T, ldt, transpose_t, X,
                                   ldx, k, Out, ldo, nullptr);
}

int sqb_thin_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
               const double* T, int64_t ldt, double* Q, int64_t ldq) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  if (k > N) return set_error(ctx, SQB_ERR_ARG, "more reflectors than rows");
  return thin_q_dispatch(ctx, lo_dtype, U, ldu, N, k, T, ldt, Q, ldq);
}

int sqb_gram(sqb_ctx* ctx, const double* A, int64_t lda, int64_t N, int64_t k, double* G, int64_t ldg) {
  SQB_TRY(begin_entry(ctx));
  return gram_run(ctx, A, lda, N, k, G, ldg);
}

int sqb_residual_norms(sqb_ctx* ctx, const double* W, int64_t ldw, const double* Q, int64_t ldq,
                       const double* R, int64_t ldr, int64_t N, int64_t k, int64_t kc, double* out) {
  SQB_TRY(begin_entry(ctx));
  return residual_norms_run(ctx, W, ldw, Q, ldq, R, ldr, N, k, kc, out);
}

int sqb_sketch_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t k, const double* T,
                 int64_t ldt, const double* S, int64_t lds, int64_t od, double* Q, int64_t ldq) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  return sketch_q_run(ctx, lo_dtype, U, ldu, k, T, ldt, S, lds, od, Q, ldq);
}

int sqb_rh_vector(sqb_ctx* ctx, int scaling, int lo_dtype, const void* w, int64_t n, const double* y,
                  int64_t od, int64_t j, void* u, double* s, double* scalars) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  if (j < 1 || j > od)
    return set_error(ctx, SQB_ERR_ARG, "elimination index %lld outside sketch of length %lld", (long long)j,
                     (long long)od);
  return rh_vector_dispatch(ctx, scaling, lo_dtype, w, n, y, od, j, u, s, scalars);
}

int sqb_rec_rhqr(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                 int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                 double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                 double* betas) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_dtype(ctx, lo_dtype));
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (sk->n != N - m)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld",
                     (long long)sk->n, (long long)(N - m));
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (ldw < N || ldu < N || lds < m + sk->ell || ldt < m || ldr < m)
    return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  return rec_rhqr_dispatch(ctx, sk, scaling, lo_dtype, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr,
                           sigmas, rhos, betas);
}

}  // extern "C"
