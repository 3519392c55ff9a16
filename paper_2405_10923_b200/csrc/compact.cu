// Compact-form application and Q materialisation (rhqr.py:100-119, 171-188),
// Gram matrices for the diagnostics (linalg.py:151-160, 193-197).
#include <algorithm>
#include <cooperative_groups.h>

#include "sketch.cuh"
#include "vec.cuh"
#include "gemv.cuh"

namespace cg = cooperative_groups;

namespace sqb {

// C[:, col] = op(T) (S^t Y[:, col]) ; one CTA per column of Y.  Warp per
// output with the lanes over the reduction index (warp_dot): every dot is a
// few L2 round trips, not a chain of dependent loads per thread.
constexpr int COEF_NT = 512;
__global__ void __launch_bounds__(COEF_NT)
coef_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ Tm, int64_t ldt,
            int transpose_t, const double* __restrict__ Y, int64_t ldy, int od, int r,
            double* __restrict__ C, int64_t ldc, const Status* st) {
  extern __shared__ double g[];  // [r]
  if (st && failed(st)) return;
  const int col = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* y = Y + (int64_t)col * ldy;
  for (int k = warp; k < r; k += nw) {
    const double d = warp_dot(S + (int64_t)k * lds, y, 0, od);
    if (lane == 0) g[k] = d;
  }
  __syncthreads();
  for (int i = warp; i < r; i += nw) {
    // (T^t g)[i] = T[:i+1, i] . g[:i+1] (a column of T);  (T g)[i] = T[i, i:] . g[i:]
    const double d = transpose_t ? warp_dot(Tm + (int64_t)i * ldt, g, 0, i + 1)
                                 : warp_dot_strided(Tm + i, ldt, g, i, r);
    if (lane == 0) C[i + (int64_t)col * ldc] = d;
  }
}

// One column on an 8-CTA cluster: partial S^t y over each CTA's block of the
// od rows, combined through DSMEM in rank order (every CTA holds all of g),
// then op(T) g with the outputs spread over the cluster's 64 warps.  The
// per-step coefficients of the Arnoldi compact update (krylov.py:141) were
// one L2-latency-bound CTA (44 us per step at m = 200).
constexpr int CCL = 8, CCL_NT = 256;
__global__ void __cluster_dims__(CCL, 1, 1) __launch_bounds__(CCL_NT)
coef_cl_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ Tm, int64_t ldt,
               int transpose_t, const double* __restrict__ y, int od, int r, double* __restrict__ C,
               const Status* st) {
  extern __shared__ double sm[];
  double* gp = sm;      // [r] partial
  double* g = sm + r;   // [r]
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const bool dead = st && failed(st);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = CCL_NT / 32;
  const int B = (od + CCL - 1) / CCL, r0 = rank * B, r1 = min(od, r0 + B);
  for (int k = warp; k < r; k += nw) {
    const double d = dead ? 0.0 : warp_dot(S + (int64_t)k * lds, y, r0, max(r0, r1));
    if (lane == 0) gp[k] = d;
  }
  cluster.sync();
  for (int k = threadIdx.x; k < r; k += CCL_NT) {
    double d = 0.0;
    for (int q = 0; q < CCL; ++q) d += cluster.map_shared_rank(gp, q)[k];
    g[k] = d;
  }
  cluster.sync();
  if (dead) return;
  const int gw = rank * nw + warp, ngw = CCL * nw;
  for (int i = gw; i < r; i += ngw) {
    const double d = transpose_t ? warp_dot(Tm + (int64_t)i * ldt, g, 0, i + 1)
                                 : warp_dot_strided(Tm + i, ldt, g, i, r);
    if (lane == 0) C[i] = d;
  }
}

static int launch_coef_col(sqb_ctx* ctx, const double* S, int64_t lds, const double* Tm, int64_t ldt,
                           int transpose_t, const double* y, int od, int r, double* C) {
  coef_cl_kernel<<<CCL, CCL_NT, sizeof(double) * 2 * r, ctx->stream>>>(S, lds, Tm, ldt, transpose_t, y, od, r, C,
                                                                      ctx->d_status);
  return check_launch(ctx, "coef_cl_kernel");
}

int launch_coef(sqb_ctx* ctx, const double* S, int64_t lds, const double* Tm, int64_t ldt, int transpose_t,
                const double* Y, int64_t ldy, int od, int r, double* C, int64_t ldc, int k) {
  coef_kernel<<<(unsigned)k, COEF_NT, sizeof(double) * r, ctx->stream>>>(S, lds, Tm, ldt, transpose_t, Y, ldy, od, r,
                                                                         C, ldc, ctx->d_status);
  return check_launch(ctx, "coef_kernel");
}

// Out[:, col] = fl(X[:, col] - fl(U C_lo[:, col]))  (rhqr.py:118); persistent
// row blocks, streaming GEMV core (gemv.cuh)
template <typename T>
__global__ void __launch_bounds__(GEMV_NT, 2)
update_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int r, const double* __restrict__ C,
              int64_t ldc, const T* X, int64_t ldx, T* Out, int64_t ldo, const Status* st) {
  using A = typename Lo<T>::acc;
  constexpr int VN = VecN<T>::n, NV = 4;
  extern __shared__ unsigned char smraw[];
  A* c = reinterpret_cast<A*>(smraw);
  if (st && failed(st)) return;
  const int col = blockIdx.y;
  for (int k = threadIdx.x; k < r; k += blockDim.x) c[k] = Lo<T>::from_double(C[k + (int64_t)col * ldc]);
  __syncthreads();
  const int64_t rows_per = (int64_t)GEMV_NT * NV * VN;
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per; r0 < N; r0 += (int64_t)gridDim.x * rows_per) {
    A acc[NV][VN];
    gemv_rows<T, NV>(U, ldu, r0, N, r, c, acc);
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < VN; ++j) {
        const int64_t i = r0 + (v * GEMV_NT + threadIdx.x) * VN + j;
        if (i < N)
          Out[i + (int64_t)col * ldo] =
              Lo<T>::store(Lo<T>::sub(Lo<T>::load(X[i + (int64_t)col * ldx]), Lo<T>::rnd(acc[v][j])));
      }
  }
}

// unaligned fallback
template <typename T>
__global__ void __launch_bounds__(256)
update_scalar_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int r, const double* __restrict__ C,
                     int64_t ldc, const T* X, int64_t ldx, T* Out, int64_t ldo, const Status* st) {
  using A = typename Lo<T>::acc;
  extern __shared__ unsigned char smraw[];
  A* c = reinterpret_cast<A*>(smraw);
  if (st && failed(st)) return;
  const int col = blockIdx.y;
  for (int k = threadIdx.x; k < r; k += blockDim.x) c[k] = Lo<T>::from_double(C[k + (int64_t)col * ldc]);
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    A d = 0;
    for (int k = 0; k < r; ++k) d = fma(Lo<T>::load(U[i + (int64_t)k * ldu]), c[k], d);
    Out[i + (int64_t)col * ldo] = Lo<T>::store(Lo<T>::sub(Lo<T>::load(X[i + (int64_t)col * ldx]), Lo<T>::rnd(d)));
  }
}

template <typename T>
static int apply_reflectors_t(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, const void* U,
                              int64_t ldu, int64_t N, int64_t r, const double* S, int64_t lds,
                              const double* Tm, int64_t ldt, int transpose_t, const void* X,
                              int64_t ldx, int64_t k, void* Out, int64_t ldo, void* ws_base) {
  const int64_t od = m + sk->ell;
  WsPlan plan;
  const size_t iY = plan.add(sizeof(double) * od * k);
  const size_t iC = plan.add(sizeof(double) * std::max<int64_t>(r, 1) * k);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, k));
  if (!ws_base) {
    SQB_TRY(ws_reserve(ctx, plan.total));
    ws_base = ctx->ws;
  }
  double* Y = reinterpret_cast<double*>(static_cast<char*>(ws_base) + plan.offs[iY]);
  double* C = reinterpret_cast<double*>(static_cast<char*>(ws_base) + plan.offs[iC]);
  const Status* st = ctx->d_status;
  if (r == 0) {  // no reflectors: Out = X
    if (Out != X)
      SQB_CUDA_TRY(cudaMemcpy2DAsync(Out, ldo * sizeof(T), X, ldx * sizeof(T), N * sizeof(T), k,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
    return SQB_OK;
  }
  SQB_TRY(launch_copy_top(ctx, Lo<T>::code, X, ldx, m, k, Y, od, st));
  SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const T*)X + m, ldx, k, Y, od, m,
                        static_cast<char*>(ws_base) + plan.offs[iP], st));
  if (k == 1) {
    SQB_TRY(launch_coef_col(ctx, S, lds, Tm, ldt, transpose_t, Y, (int)od, (int)r, C));
  } else {
    coef_kernel<<<(unsigned)k, COEF_NT, sizeof(double) * r, ctx->stream>>>(S, lds, Tm, ldt, transpose_t, Y, od,
                                                                       (int)od, (int)r, C, r, st);
    SQB_TRY(check_launch(ctx, "coef_kernel"));
  }
  constexpr int VN = VecN<T>::n;
  const bool vec = ((reinterpret_cast<uintptr_t>(U) & 15) == 0) && (ldu % VN == 0);
  if (vec) {
    const int64_t blocks = (N + (int64_t)GEMV_NT * 4 * VN - 1) / ((int64_t)GEMV_NT * 4 * VN);
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, 2 * (int64_t)ctx->sm_count)), (unsigned)k);
    update_kernel<T><<<grid, GEMV_NT, sizeof(typename Lo<T>::acc) * r, ctx->stream>>>(
        (const T*)U, ldu, N, (int)r, C, r, (const T*)X, ldx, (T*)Out, ldo, st);
  } else {
    dim3 grid((unsigned)std::min<int64_t>((N + 255) / 256, 4 * 148), (unsigned)k);
    update_scalar_kernel<T><<<grid, 256, sizeof(typename Lo<T>::acc) * r, ctx->stream>>>(
        (const T*)U, ldu, N, (int)r, C, r, (const T*)X, ldx, (T*)Out, ldo, st);
  }
  return check_launch(ctx, "update_kernel");
}

// Out = X - U op(T) S^t Y for a given sketch Y = Psi X (od x 1): the
// coefficient and update halves of apply_reflectors_t, used by the
// row-partitioned Arnoldi (krylov.cu) on each rank's rows after the sketch
// has been combined across ranks.  C: r doubles of scratch.
int compact_update_dispatch(sqb_ctx* ctx, int lo_dtype, const double* Y, int64_t od, const double* S, int64_t lds,
                            const double* Tm, int64_t ldt, int transpose_t, int64_t r, const void* U, int64_t ldu,
                            int64_t N, const void* X, void* Out, double* C) {
  const Status* st = ctx->d_status;
  SQB_TRY(launch_coef_col(ctx, S, lds, Tm, ldt, transpose_t, Y, (int)od, (int)r, C));
  auto run = [&](auto t) -> int {
    using T = decltype(t);
    constexpr int VN = VecN<T>::n;
    const bool vec = ((reinterpret_cast<uintptr_t>(U) & 15) == 0) && (ldu % VN == 0);
    if (vec) {
      const int64_t blocks = (N + (int64_t)GEMV_NT * 4 * VN - 1) / ((int64_t)GEMV_NT * 4 * VN);
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, 2 * (int64_t)ctx->sm_count)), 1);
      update_kernel<T><<<grid, GEMV_NT, sizeof(typename Lo<T>::acc) * r, ctx->stream>>>(
          (const T*)U, ldu, N, (int)r, C, r, (const T*)X, N, (T*)Out, N, st);
    } else {
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 4 * 148)), 1);
      update_scalar_kernel<T><<<grid, 256, sizeof(typename Lo<T>::acc) * r, ctx->stream>>>(
          (const T*)U, ldu, N, (int)r, C, r, (const T*)X, N, (T*)Out, N, st);
    }
    return check_launch(ctx, "update_kernel");
  };
  switch (lo_dtype) {
    case SQB_F64: return run(double());
    case SQB_F32: return run(float());
    case SQB_F16: return run(__half());
    case SQB_BF16: return run(__nv_bfloat16());
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

size_t apply_reflectors_ws_bytes(const sqb_sketch* sk, int dtype, int64_t m, int64_t r, int64_t k) {
  WsPlan plan;
  plan.add(sizeof(double) * (m + sk->ell) * k);
  plan.add(sizeof(double) * std::max<int64_t>(r, 1) * k);
  plan.add(sketch_partials_bytes(sk, dtype, k));
  return plan.total + 256;
}

int apply_reflectors_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, int lo_dtype,
                              const void* U, int64_t ldu, int64_t N, int64_t r, const double* S,
                              int64_t lds, const double* Tm, int64_t ldt, int transpose_t,
                              const void* X, int64_t ldx, int64_t k, void* Out, int64_t ldo,
                              void* ws_base) {
  switch (lo_dtype) {
    case SQB_F64: return apply_reflectors_t<double>(ctx, sk, m, U, ldu, N, r, S, lds, Tm, ldt, transpose_t, X, ldx, k, Out, ldo, ws_base);
    case SQB_F32: return apply_reflectors_t<float>(ctx, sk, m, U, ldu, N, r, S, lds, Tm, ldt, transpose_t, X, ldx, k, Out, ldo, ws_base);
    case SQB_F16: return apply_reflectors_t<__half>(ctx, sk, m, U, ldu, N, r, S, lds, Tm, ldt, transpose_t, X, ldx, k, Out, ldo, ws_base);
    case SQB_BF16: return apply_reflectors_t<__nv_bfloat16>(ctx, sk, m, U, ldu, N, r, S, lds, Tm, ldt, transpose_t, X, ldx, k, Out, ldo, ws_base);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

// ---------------------------------------------------------------------------
// thin Q = [I;0] - U (T U1^t), fp64 (rhqr.py:171-178)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void tu1t_kernel(const T* __restrict__ U, int64_t ldu, int k, const double* __restrict__ Tm,
                            int64_t ldt, double* __restrict__ M) {
  // M[i, j] = sum_l T[i, l] U[j, l]   (T upper: l >= i)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int i = e % k, j = e / k;
    double d = 0.0;
    for (int l = i; l < k; ++l) d = fma(Tm[i + (int64_t)l * ldt], (double)Lo<T>::load(U[j + (int64_t)l * ldu]), d);
    M[i + (int64_t)j * k] = d;
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
thin_q_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int k, const double* __restrict__ M,
              double* __restrict__ Q, int64_t ldq) {
  // blockIdx.y selects a block of (up to) 64 output columns: shared memory
  // holds M[:, j0:j0+64] only, so any k <= 400 fits
  extern __shared__ double sM[];  // k x jn
  const int j0 = blockIdx.y * 64;
  const int jn = min(64, k - j0);
  for (int e = threadIdx.x; e < k * jn; e += blockDim.x) sM[e] = M[(e % k) + (int64_t)(j0 + e / k) * k];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double u[64];
    for (int jj = 0; jj < jn; ++jj) u[jj] = 0.0;
    for (int l = 0; l < k; ++l) {
      const double ul = (double)Lo<T>::load(U[i + (int64_t)l * ldu]);
      for (int jj = 0; jj < jn; ++jj) u[jj] = fma(ul, sM[l + jj * k], u[jj]);
    }
    for (int jj = 0; jj < jn; ++jj) {
      const int j = j0 + jj;
      Q[i + (int64_t)j * ldq] = (i == j ? 1.0 : 0.0) - u[jj];
    }
  }
}

template <typename T>
static int launch_thin_q(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t N, int64_t k, const double* M,
                         double* Q, int64_t ldq) {
  if (k > 400) return set_error(ctx, SQB_ERR_ARG, "thin_q: k=%lld above 400", (long long)k);
  const size_t smem = sizeof(double) * k * std::min<int64_t>(64, k);
  cudaFuncSetAttribute(thin_q_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::max<size_t>(smem, 48 * 1024));
  const unsigned nb = (unsigned)((k + 63) / 64);
  thin_q_kernel<T><<<dim3((unsigned)std::min<int64_t>((N + 255) / 256, 2 * 148), nb), 256, smem, ctx->stream>>>(
      (const T*)U, ldu, N, (int)k, M, Q, ldq);
  return check_launch(ctx, "thin_q_kernel");
}

template <typename T>
static int thin_q_t(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t N, int64_t k, const double* Tm,
                    int64_t ldt, double* Q, int64_t ldq) {
  WsPlan plan;
  const size_t iM = plan.add(sizeof(double) * std::max<int64_t>(1, k * k));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* M = ws_ptr<double>(ctx, plan, iM);
  tu1t_kernel<T><<<(unsigned)std::max<int64_t>(1, (k * k + 255) / 256), 256, 0, ctx->stream>>>(
      (const T*)U, ldu, (int)k, Tm, ldt, M);
  SQB_TRY(check_launch(ctx, "tu1t_kernel"));
  return launch_thin_q<T>(ctx, U, ldu, N, k, M, Q, ldq);
}

// Q = [I;0] - U M for a given k x k fp64 M (ld k) — the trimmed thin Q
// (trim.py:211-225) passes M = T triu(S^t E)
template <typename T>
static int thin_q_m_t(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t N, int64_t k, const double* M, double* Q,
                      int64_t ldq) {
  return launch_thin_q<T>(ctx, U, ldu, N, k, M, Q, ldq);
}

int thin_q_m_dispatch(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
                      const double* M, double* Q, int64_t ldq) {
  switch (lo_dtype) {
    case SQB_F64: return thin_q_m_t<double>(ctx, U, ldu, N, k, M, Q, ldq);
    case SQB_F32: return thin_q_m_t<float>(ctx, U, ldu, N, k, M, Q, ldq);
    case SQB_F16: return thin_q_m_t<__half>(ctx, U, ldu, N, k, M, Q, ldq);
    case SQB_BF16: return thin_q_m_t<__nv_bfloat16>(ctx, U, ldu, N, k, M, Q, ldq);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

int thin_q_dispatch(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
                    const double* Tm, int64_t ldt, double* Q, int64_t ldq) {
  switch (lo_dtype) {
    case SQB_F64: return thin_q_t<double>(ctx, U, ldu, N, k, Tm, ldt, Q, ldq);
    case SQB_F32: return thin_q_t<float>(ctx, U, ldu, N, k, Tm, ldt, Q, ldq);
    case SQB_F16: return thin_q_t<__half>(ctx, U, ldu, N, k, Tm, ldt, Q, ldq);
    case SQB_BF16: return thin_q_t<__nv_bfloat16>(ctx, U, ldu, N, k, Tm, ldt, Q, ldq);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

// ---------------------------------------------------------------------------
// Gram G = A^t A (k x k) of fp64 A (N x k): split over row blocks, fixed-order sum
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
gram_partial_kernel(const double* __restrict__ A, int64_t lda, int64_t N, int k, int64_t rows_per,
                    double* __restrict__ P) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = min(N, r0 + rows_per);
  const int kk = k * k;
  for (int e = threadIdx.x; e < kk; e += blockDim.x) {
    const int i = e % k, j = e / k;
    if (i > j) continue;
    double d = 0.0;
    for (int64_t r = r0; r < r1; ++r) d = fma(A[r + i * lda], A[r + j * lda], d);
    P[(int64_t)blockIdx.x * kk + e] = d;
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ P, int nb, int k, double* __restrict__ G,
                                   int64_t ldg) {
  const int kk = k * k;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kk; e += gridDim.x * blockDim.x) {
    const int i = e % k, j = e / k;
    const int src = i <= j ? e : (j + i * k);
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += P[(int64_t)b * kk + src];
    G[i + (int64_t)j * ldg] = s;
  }
}

int gram_run(sqb_ctx* ctx, const double* A, int64_t lda, int64_t N, int64_t k, double* G, int64_t ldg) {
  if (k == 0) return SQB_OK;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(4 * 148, (N + 1023) / 1024));
  const int64_t rows_per = (N + nb - 1) / nb;
  WsPlan plan;
  const size_t iP = plan.add(sizeof(double) * nb * k * k);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* P = ws_ptr<double>(ctx, plan, iP);
  gram_partial_kernel<<<nb, 256, 0, ctx->stream>>>(A, lda, N, (int)k, rows_per, P);
  SQB_TRY(check_launch(ctx, "gram_partial_kernel"));
  gram_reduce_kernel<<<(unsigned)std::max<int64_t>(1, (k * k + 255) / 256), 256, 0, ctx->stream>>>(P, nb, (int)k, G, ldg);
  return check_launch(ctx, "gram_reduce_kernel");
}

}  // namespace sqb

namespace sqb {

// per-column sums of (W - Q R)^2 and W^2 (factorization_errors, linalg.py:169-190)
__global__ void __launch_bounds__(256)
residual_partial_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ Q,
                        int64_t ldq, const double* __restrict__ R, int64_t ldr, int64_t N, int k,
                        double* __restrict__ P, int nb) {
  __shared__ double red[32];
  const int j = blockIdx.y;
  double sd = 0.0, sw = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    double q = 0.0;
    for (int l = 0; l < k; ++l) q = fma(Q[i + l * ldq], R[l + (int64_t)j * ldr], q);
    const double w = W[i + (int64_t)j * ldw];
    const double d = w - q;
    sd = fma(d, d, sd);
    sw = fma(w, w, sw);
  }
  sd = block_sum(sd, red);
  sw = block_sum(sw, red);
  if (threadIdx.x == 0) {
    P[(int64_t)j * nb + blockIdx.x] = sd;
    P[(int64_t)(gridDim.y + j) * nb + blockIdx.x] = sw;
  }
}

__global__ void rowsum_kernel(const double* __restrict__ P, int rows, int nb, double* __restrict__ out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += P[(int64_t)r * nb + b];
    out[r] = s;
  }
}

int residual_norms_run(sqb_ctx* ctx, const double* W, int64_t ldw, const double* Q, int64_t ldq,
                       const double* R, int64_t ldr, int64_t N, int64_t k, int64_t kc, double* out) {
  if (kc == 0) return SQB_OK;
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(2 * 148, (N + 255) / 256));
  WsPlan plan;
  const size_t iP = plan.add(sizeof(double) * 2 * kc * nb);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* P = ws_ptr<double>(ctx, plan, iP);
  residual_partial_kernel<<<dim3(nb, (unsigned)kc), 256, 0, ctx->stream>>>(W, ldw, Q, ldq, R, ldr, N, (int)k, P, nb);
  SQB_TRY(check_launch(ctx, "residual_partial_kernel"));
  rowsum_kernel<<<(unsigned)((2 * kc + 255) / 256), 256, 0, ctx->stream>>>(P, (int)(2 * kc), nb, out);
  return check_launch(ctx, "rowsum_kernel");
}

}  // namespace sqb

namespace sqb {

template <typename T>
static int sketch_q_t(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t k, const double* Tm, int64_t ldt,
                      const double* S, int64_t lds, int64_t od, double* Q, int64_t ldq) {
  WsPlan plan;
  const size_t iM = plan.add(sizeof(double) * std::max<int64_t>(1, k * k));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* M = ws_ptr<double>(ctx, plan, iM);
  tu1t_kernel<T><<<(unsigned)std::max<int64_t>(1, (k * k + 255) / 256), 256, 0, ctx->stream>>>(
      (const T*)U, ldu, (int)k, Tm, ldt, M);
  SQB_TRY(check_launch(ctx, "tu1t_kernel"));
  return launch_thin_q<double>(ctx, S, lds, od, k, M, Q, ldq);
}

int sketch_q_run(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t k, const double* Tm,
                 int64_t ldt, const double* S, int64_t lds, int64_t od, double* Q, int64_t ldq) {
  switch (lo_dtype) {
    case SQB_F64: return sketch_q_t<double>(ctx, U, ldu, k, Tm, ldt, S, lds, od, Q, ldq);
    case SQB_F32: return sketch_q_t<float>(ctx, U, ldu, k, Tm, ldt, S, lds, od, Q, ldq);
    case SQB_F16: return sketch_q_t<__half>(ctx, U, ldu, k, Tm, ldt, S, lds, od, Q, ldq);
    case SQB_BF16: return sketch_q_t<__nv_bfloat16>(ctx, U, ldu, k, Tm, ldt, S, lds, od, Q, ldq);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb

namespace sqb {

// M[i, j] = sum_{l >= i} T[i, l] S[j, l]  (r x c), i.e. T S[:c, :]^t (arnoldi_q, krylov.py:77)
__global__ void ts_kernel(const double* __restrict__ Tm, int64_t ldt, const double* __restrict__ S,
                          int64_t lds, int r, int c, double* __restrict__ M) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < r * c; e += gridDim.x * blockDim.x) {
    const int i = e % r, j = e / r;
    double d = 0.0;
    for (int l = i; l < r; ++l) d = fma(Tm[i + (int64_t)l * ldt], S[j + (int64_t)l * lds], d);
    M[i + (int64_t)j * r] = d;
  }
}

// Q = [I;0] - U M with U (N x r, lo) and M (r x c): one thread per row, M in smem
template <typename T>
__global__ void __launch_bounds__(256)
compact_q_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int r, int c, const double* __restrict__ M,
                 double* __restrict__ Q, int64_t ldq) {
  extern __shared__ double sM[];
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) sM[e] = M[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < c; ++j) {
      double d = 0.0;
      for (int l = 0; l < r; ++l) d = fma((double)Lo<T>::load(U[i + (int64_t)l * ldu]), sM[l + j * r], d);
      Q[i + (int64_t)j * ldq] = (i == j ? 1.0 : 0.0) - d;
    }
  }
}

template <typename T>
static int arnoldi_q_t(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t N, int64_t r, const double* Tm,
                       int64_t ldt, const double* S, int64_t lds, int64_t c, double* Q, int64_t ldq) {
  WsPlan plan;
  const size_t iM = plan.add(sizeof(double) * std::max<int64_t>(1, r * c));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* M = ws_ptr<double>(ctx, plan, iM);
  ts_kernel<<<(unsigned)std::max<int64_t>(1, (r * c + 255) / 256), 256, 0, ctx->stream>>>(Tm, ldt, S, lds,
                                                                                          (int)r, (int)c, M);
  SQB_TRY(check_launch(ctx, "ts_kernel"));
  const size_t smem = sizeof(double) * std::max<int64_t>(1, r * c);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(compact_q_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  compact_q_kernel<T><<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 4 * 148)), 256, smem,
                        ctx->stream>>>((const T*)U, ldu, N, (int)r, (int)c, M, Q, ldq);
  return check_launch(ctx, "compact_q_kernel");
}

}  // namespace sqb

extern "C" int sqb_arnoldi_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t r,
                             const double* T, int64_t ldt, const double* S, int64_t lds, int64_t c, double* Q,
                             int64_t ldq) {
  using namespace sqb;
  SQB_TRY(begin_entry(ctx));
  if (c < 0 || c > r) return set_error(ctx, SQB_ERR_ARG, "have %lld reflectors, cannot build %lld columns",
                                       (long long)r, (long long)c);
  if ((int64_t)r * c * 8 > 200 * 1024) return set_error(ctx, SQB_ERR_ARG, "arnoldi_q: r*c too large");
  switch (lo_dtype) {
    case SQB_F64: return arnoldi_q_t<double>(ctx, U, ldu, N, r, T, ldt, S, lds, c, Q, ldq);
    case SQB_F32: return arnoldi_q_t<float>(ctx, U, ldu, N, r, T, ldt, S, lds, c, Q, ldq);
    case SQB_F16: return arnoldi_q_t<__half>(ctx, U, ldu, N, r, T, ldt, S, lds, c, Q, ldq);
    case SQB_BF16: return arnoldi_q_t<__nv_bfloat16>(ctx, U, ldu, N, r, T, ldt, S, lds, c, Q, ldq);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

// Out = X - U op(T) S^t Y with the sketch Y = Psi X given (od fp64): the
// compact-form update of apply_reflectors_compact (rhqr.py:100-119) without
// its sketch, for callers that hold Psi X already (the row-partitioned GMRES
// solution, whose padded coefficient vector has Psi pad = [pad[:m+1]; 0]).
extern "C" int sqb_compact_update(sqb_ctx* ctx, int lo_dtype, const double* Y, int64_t od, const double* S,
                                  int64_t lds, const double* T, int64_t ldt, int transpose_t, int64_t r,
                                  const void* U, int64_t ldu, int64_t N, const void* X, void* Out) {
  using namespace sqb;
  SQB_TRY(begin_entry(ctx));
  if (r < 1 || N < 1) return SQB_OK;
  WsPlan plan;
  const size_t iC = plan.add(sizeof(double) * r);
  SQB_TRY(ws_reserve(ctx, plan.total));
  return compact_update_dispatch(ctx, lo_dtype, Y, od, S, lds, T, ldt, transpose_t, r, U, ldu, N, X, Out,
                                 ws_ptr<double>(ctx, plan, iC));
}
