// Compact-form application and Q materialisation (rhqr.py:100-119, 171-188),
// Gram matrices for the diagnostics (linalg.py:151-160, 193-197).
#include <algorithm>
#include <cooperative_groups.h>

#include "sketch.cuh"
#include "vec.cuh"
#include "gemv.cuh"
#include "mma.cuh"

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

// fp64, several columns: Out = X - U C as one tall-skinny DMMA GEMM (defined
// below, next to the thin-Q kernel whose main loop it shares)
int launch_update_dmma(sqb_ctx* ctx, const double* U, int64_t ldu, int64_t N, int64_t r, const double* C,
                       const double* X, int64_t ldx, int64_t k, double* Out, int64_t ldo);

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
  defer_copy_top(ctx, Lo<T>::code, X, ldx, m, k, Y, od);
  SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const T*)X + m, ldx, k, Y, od, m,
                        static_cast<char*>(ws_base) + plan.offs[iP], st));
  SQB_TRY(flush_copy_top(ctx, st));
  if (k == 1) {
    SQB_TRY(launch_coef_col(ctx, S, lds, Tm, ldt, transpose_t, Y, (int)od, (int)r, C));
  } else {
    coef_kernel<<<(unsigned)k, COEF_NT, sizeof(double) * r, ctx->stream>>>(S, lds, Tm, ldt, transpose_t, Y, od,
                                                                       (int)od, (int)r, C, r, st);
    SQB_TRY(check_launch(ctx, "coef_kernel"));
  }
  constexpr int VN = VecN<T>::n;
  const bool vec = ((reinterpret_cast<uintptr_t>(U) & 15) == 0) && (ldu % VN == 0);
  if constexpr (std::is_same<T, double>::value) {
    // the per-column GEMV below re-reads U for every column of X (16 columns
    // on config 2's factors: 16 GB, 2.46 ms); from 4 columns on, one DMMA
    // GEMM reads U once
    static const bool no_dmma = [] { const char* e = getenv("SQB_UPDATE_GEMV"); return e && e[0] == '1'; }();
    if (k >= 4 && !no_dmma)
      return launch_update_dmma(ctx, (const double*)U, ldu, N, r, C, (const double*)X, ldx, k, (double*)Out, ldo);
  }
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

// thin Q on the FP64 tensor pipe: Q = [I;0] - U M is a tall-skinny GEMM
// (N x K times K x nc; config 2: 2^20 x 128 x 128 = 34 GFLOP, compute-bound
// at 37 TFLOP/s).  One CTA owns a 128-row x 64-column tile of Q; K runs in
// 32-deep chunks, U chunk (k-major, rows contiguous as in HBM) and M chunk
// (n-major, k contiguous) double-buffered in shared memory — cp.async for
// fp64 storage, load + widen for the low formats — and 8 warps of 32 x 32
// accumulate with DMMA m16n8k16.  Column blocks of the same row tile are
// adjacent in the grid, so the second read of the U tile hits L2.  The
// row-per-thread kernel above it replaced took 29.4 ms on config 2's factors
// (registers spilled around u[64], broadcast shared reads): this one 1.2 ms.
constexpr int TQ_BM = 128, TQ_BN = 64, TQ_BK = 32, TQ_AS = TQ_BM + 4, TQ_BS = TQ_BK + 4, TQ_NT = 256;
constexpr size_t TQ_SMEM = sizeof(double) * 2 * (size_t)(TQ_BK * TQ_AS + TQ_BN * TQ_BS);

__device__ __forceinline__ void cp_async8_ca(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}

// acc (the 32 x 32 warp tile of a 128 x 64 CTA tile) = A[r0 : r0+128, :K] M[:K, c0 : c0+64]
// A: N x K of T, column-major (lda); M: K x nc fp64, ld ldm
template <typename T>
__device__ __forceinline__ void tq_mainloop(double (&acc)[2][4][4], const T* __restrict__ A, int64_t lda, int64_t N,
                                            int K, const double* __restrict__ M, int64_t ldm, int nc, int64_t r0,
                                            int c0, double* sA, double* sB) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nk = (K + TQ_BK - 1) / TQ_BK;
  const bool a16 = std::is_same<T, double>::value && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0) &&
                   (r0 + TQ_BM <= N);
  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * TQ_BK;
    double* a = sA + st * TQ_BK * TQ_AS;
    double* b = sB + st * TQ_BN * TQ_BS;
    if (a16) {
      for (int e = tid; e < TQ_BK * TQ_BM / 2; e += TQ_NT) {
        const int k = e / (TQ_BM / 2), r = 2 * (e % (TQ_BM / 2));
        double* d = a + k * TQ_AS + r;
        if (k0 + k < K) cp_async16(d, reinterpret_cast<const double*>(A) + r0 + r + (int64_t)(k0 + k) * lda, 16);
        else { d[0] = 0.0; d[1] = 0.0; }
      }
    } else {
      for (int e = tid; e < TQ_BK * TQ_BM; e += TQ_NT) {
        const int k = e / TQ_BM, r = e % TQ_BM;
        double* d = a + k * TQ_AS + r;
        const bool in = k0 + k < K && r0 + r < N;
        if constexpr (std::is_same<T, double>::value) {
          if (in) cp_async8_ca(d, reinterpret_cast<const double*>(A) + r0 + r + (int64_t)(k0 + k) * lda);
          else *d = 0.0;
        } else {
          *d = in ? (double)Lo<T>::load(A[r0 + r + (int64_t)(k0 + k) * lda]) : 0.0;
        }
      }
    }
    for (int e = tid; e < TQ_BN * TQ_BK; e += TQ_NT) {
      const int n = e / TQ_BK, k = e % TQ_BK;
      b[n * TQ_BS + k] = (c0 + n < nc && k0 + k < K) ? __ldg(M + (k0 + k) + (int64_t)(c0 + n) * ldm) : 0.0;
    }
  };
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 4; ++z) acc[x][y][z] = 0.0;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  load_stage(0, 0);
  cp_async_commit_group();
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) load_stage((kt + 1) & 1, kt + 1);
    cp_async_commit_group();
    cp_async_wait_group<1>();
    __syncthreads();
    const double* as = sA + (kt & 1) * TQ_BK * TQ_AS + wm * 32;
    const double* bs = sB + (kt & 1) * TQ_BN * TQ_BS + (wn * 32) * TQ_BS;
#pragma unroll
    for (int k16 = 0; k16 < TQ_BK / 16; ++k16) {
      double a[2][8], b[4][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v = 0; v < 8; ++v) a[mt][v] = as[(k16 * 16 + t + 4 * (v >> 1)) * TQ_AS + mt * 16 + g + 8 * (v & 1)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) b[nt][v] = bs[(nt * 8 + g) * TQ_BS + k16 * 16 + t + 4 * v];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x16(acc[mt][nt], a[mt], b[nt]);
    }
    __syncthreads();  // the stage is refilled two iterations on
  }
  cp_async_wait_group<0>();
}

template <typename T>
__global__ void __launch_bounds__(TQ_NT, 2)
thin_q_dmma_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int K, const double* __restrict__ M, int nc,
                   int ncb, double* __restrict__ Q, int64_t ldq) {
  extern __shared__ __align__(16) unsigned char tq_raw[];
  double* sA = reinterpret_cast<double*>(tq_raw);   // [2][TQ_BK][TQ_AS]
  double* sB = sA + 2 * TQ_BK * TQ_AS;              // [2][TQ_BN][TQ_BS]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bid = blockIdx.x;
  const int64_t r0 = (bid / ncb) * TQ_BM;
  const int c0 = (int)(bid % ncb) * TQ_BN;
  double acc[2][4][4];
  tq_mainloop<T>(acc, U, ldu, N, K, M, K, nc, r0, c0, sA, sB);
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t r = r0 + wm * 32 + mt * 16 + g + h * 8;
          const int c = c0 + wn * 32 + nt * 8 + 2 * t + q;
          if (r < N && c < nc) Q[r + (int64_t)c * ldq] = (r == c ? 1.0 : 0.0) - acc[mt][nt][h * 2 + q];
        }
}

// Out = X - U C (fp64; U: N x r, C: r x k with ld r), the compact update
// (rhqr.py:118) for several columns at once: tq_mainloop, epilogue against X
__global__ void __launch_bounds__(TQ_NT, 2)
update_dmma_kernel(const double* __restrict__ U, int64_t ldu, int64_t N, int r, const double* __restrict__ C, int nc,
                   int ncb, const double* X, int64_t ldx, double* Out, int64_t ldo, const Status* st) {
  extern __shared__ __align__(16) unsigned char tq_raw[];
  double* sA = reinterpret_cast<double*>(tq_raw);
  double* sB = sA + 2 * TQ_BK * TQ_AS;
  if (st && failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bid = blockIdx.x;
  const int64_t r0 = (bid / ncb) * TQ_BM;
  const int c0 = (int)(bid % ncb) * TQ_BN;
  double acc[2][4][4];
  tq_mainloop<double>(acc, U, ldu, N, r, C, r, nc, r0, c0, sA, sB);
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t row = r0 + wm * 32 + mt * 16 + g + h * 8;
          const int c = c0 + wn * 32 + nt * 8 + 2 * t + q;
          if (row < N && c < nc) Out[row + (int64_t)c * ldo] = __dsub_rn(X[row + (int64_t)c * ldx], acc[mt][nt][h * 2 + q]);
        }
}

int launch_update_dmma(sqb_ctx* ctx, const double* U, int64_t ldu, int64_t N, int64_t r, const double* C,
                       const double* X, int64_t ldx, int64_t k, double* Out, int64_t ldo) {
  allow_dyn_smem(update_dmma_kernel, (size_t)(TQ_SMEM));
  const int ncb = (int)((k + TQ_BN - 1) / TQ_BN);
  const int64_t tiles = (N + TQ_BM - 1) / TQ_BM;
  update_dmma_kernel<<<(unsigned)(tiles * ncb), TQ_NT, TQ_SMEM, ctx->stream>>>(U, ldu, N, (int)r, C, (int)k, ncb, X, ldx,
                                                                              Out, ldo, ctx->d_status);
  return check_launch(ctx, "update_dmma_kernel");
}

template <typename T>
static int launch_thin_q(sqb_ctx* ctx, const void* U, int64_t ldu, int64_t N, int64_t k, const double* M,
                         double* Q, int64_t ldq) {
  if (k > 400) return set_error(ctx, SQB_ERR_ARG, "thin_q: k=%lld above 400", (long long)k);
  static const bool old_path = [] { const char* e = getenv("SQB_THINQ_OLD"); return e && e[0] == '1'; }();
  if (!old_path) {
    allow_dyn_smem(thin_q_dmma_kernel<T>, (size_t)(TQ_SMEM));
    const int ncb = (int)((k + TQ_BN - 1) / TQ_BN);
    const int64_t tiles = (N + TQ_BM - 1) / TQ_BM;
    thin_q_dmma_kernel<T><<<(unsigned)(tiles * ncb), TQ_NT, TQ_SMEM, ctx->stream>>>((const T*)U, ldu, N, (int)k, M,
                                                                                  (int)k, ncb, Q, ldq);
    return check_launch(ctx, "thin_q_dmma_kernel");
  }
  if (k > 400) return set_error(ctx, SQB_ERR_ARG, "thin_q: k=%lld above 400", (long long)k);
  const size_t smem = sizeof(double) * k * std::min<int64_t>(64, k);
  allow_dyn_smem(thin_q_kernel<T>, (size_t)(std::max<size_t>(smem, 48 * 1024)));
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

// Gram partials on the FP64 tensor pipe: CTA (b, pair) accumulates the 64 x 64
// block G[I, J] = A[rows_b, I]^t A[rows_b, J] (I <= J) over its row range in
// 32-row chunks.  Both operands are staged as [column][row] (rows contiguous,
// as in HBM; stride 36 = 4 mod 16 keeps both DMMA fragment loads
// conflict-free), double-buffered with cp.async.  The row-per-entry kernel
// above took 34 ms for config 2's Q (2^20 x 128); this one ~1 ms.
constexpr int GR_B = 64, GR_KC = 32, GR_ST = GR_KC + 4, GR_NT = 128;
constexpr size_t GR_SMEM = sizeof(double) * 2 * 2 * (size_t)GR_B * GR_ST;

__global__ void __launch_bounds__(GR_NT, 3)
gram_dmma_kernel(const double* __restrict__ A, int64_t lda, int64_t N, int k, int nblk, int64_t rows_per,
                 double* __restrict__ P) {
  extern __shared__ __align__(16) unsigned char gr_raw[];
  double* sI = reinterpret_cast<double*>(gr_raw);  // [2][GR_B][GR_ST]
  double* sJ = sI + 2 * GR_B * GR_ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // pair index -> (bi <= bj)
  int bi = 0, bj = 0;
  {
    int p = blockIdx.y;
    for (bj = 0; bj < nblk; ++bj) {
      if (p <= bj) { bi = p; break; }
      p -= bj + 1;
    }
  }
  const int i0 = bi * GR_B, j0 = bj * GR_B;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(N, r0 + rows_per);
  const int nch = r1 > r0 ? (int)((r1 - r0 + GR_KC - 1) / GR_KC) : 0;
  const bool a16 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0) && (r0 % 2 == 0);
  auto load_stage = [&](int st, int ch) {
    const int64_t rb = r0 + (int64_t)ch * GR_KC;
    double* di = sI + st * GR_B * GR_ST;
    double* dj = sJ + st * GR_B * GR_ST;
    for (int e = tid; e < 2 * GR_B * GR_KC / 2; e += GR_NT) {
      const int which = e / (GR_B * GR_KC / 2), f = e % (GR_B * GR_KC / 2);
      const int c = f / (GR_KC / 2), r = 2 * (f % (GR_KC / 2));
      const int col = (which ? j0 : i0) + c;
      double* d = (which ? dj : di) + c * GR_ST + r;
      const double* src = A + rb + r + (int64_t)col * lda;
      if (col < k && rb + r + 1 < r1 && a16) {
        cp_async16(d, src, 16);
      } else {
        d[0] = (col < k && rb + r < r1) ? src[0] : 0.0;
        d[1] = (col < k && rb + r + 1 < r1) ? src[1] : 0.0;
      }
    }
  };
  double acc[2][4][4];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int z = 0; z < 4; ++z) acc[x][y][z] = 0.0;
  const int wm = warp & 1, wn = warp >> 1, g = lane >> 2, t = lane & 3;
  if (nch > 0) load_stage(0, 0);
  cp_async_commit_group();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load_stage((ch + 1) & 1, ch + 1);
    cp_async_commit_group();
    cp_async_wait_group<1>();
    __syncthreads();
    const double* as = sI + (ch & 1) * GR_B * GR_ST + (wm * 32) * GR_ST;
    const double* bs = sJ + (ch & 1) * GR_B * GR_ST + (wn * 32) * GR_ST;
#pragma unroll
    for (int k16 = 0; k16 < GR_KC / 16; ++k16) {
      double a[2][8], b[4][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v = 0; v < 8; ++v) a[mt][v] = as[(mt * 16 + g + 8 * (v & 1)) * GR_ST + k16 * 16 + t + 4 * (v >> 1)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) b[nt][v] = bs[(nt * 8 + g) * GR_ST + k16 * 16 + t + 4 * v];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x16(acc[mt][nt], a[mt], b[nt]);
    }
    __syncthreads();
  }
  cp_async_wait_group<0>();
  double* p = P + (int64_t)blockIdx.x * k * k;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int i = i0 + wm * 32 + mt * 16 + g + h * 8;
          const int j = j0 + wn * 32 + nt * 8 + 2 * t + q;
          if (i <= j && j < k) p[i + (int64_t)j * k] = acc[mt][nt][h * 2 + q];
        }
}

int gram_run(sqb_ctx* ctx, const double* A, int64_t lda, int64_t N, int64_t k, double* G, int64_t ldg) {
  if (k == 0) return SQB_OK;
  static const bool old_path = [] { const char* e = getenv("SQB_GRAM_OLD"); return e && e[0] == '1'; }();
  if (!old_path) {
    const int nblk = (int)((k + GR_B - 1) / GR_B);
    const int npairs = nblk * (nblk + 1) / 2;
    int nb = (int)std::max<int64_t>(1, std::min<int64_t>((3 * (int64_t)ctx->sm_count + npairs - 1) / npairs,
                                                        (N + 4 * GR_KC - 1) / (4 * GR_KC)));
    int64_t rows_per = (N + nb - 1) / nb;
    rows_per = (rows_per + GR_KC - 1) / GR_KC * GR_KC;
    nb = (int)((N + rows_per - 1) / rows_per);
    WsPlan plan;
    const size_t iP = plan.add(sizeof(double) * nb * k * k);
    SQB_TRY(ws_reserve(ctx, plan.total));
    double* P = ws_ptr<double>(ctx, plan, iP);
    allow_dyn_smem(gram_dmma_kernel, (size_t)(GR_SMEM));
    gram_dmma_kernel<<<dim3((unsigned)nb, (unsigned)npairs), GR_NT, GR_SMEM, ctx->stream>>>(A, lda, N, (int)k, nblk,
                                                                                          rows_per, P);
    SQB_TRY(check_launch(ctx, "gram_dmma_kernel"));
    gram_reduce_kernel<<<(unsigned)std::max<int64_t>(1, (k * k + 255) / 256), 256, 0, ctx->stream>>>(P, nb, (int)k, G,
                                                                                                 ldg);
    return check_launch(ctx, "gram_reduce_kernel");
  }

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

// The same sums with the product Q R on the FP64 tensor pipe (tq_mainloop):
// CTA (b, column block) walks row tiles b, b + nb, ... of 128 rows, forms
// D = W - Q R for its 64 columns from the DMMA accumulators and keeps the
// per-column sums of D^2 and W^2 in registers; one fixed-order reduction
// (lane octets, then the four row warps) per CTA at the end.  The
// row-per-thread kernel above took 23 ms on config 2 (2^20 x 128); this ~1.3.
__global__ void __launch_bounds__(TQ_NT, 2)
residual_dmma_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ Q, int64_t ldq,
                     const double* __restrict__ R, int64_t ldr, int64_t N, int k, int kc, int ncb, int nb,
                     double* __restrict__ P) {
  extern __shared__ __align__(16) unsigned char tq_raw[];
  double* sA = reinterpret_cast<double*>(tq_raw);
  double* sB = sA + 2 * TQ_BK * TQ_AS;
  __shared__ double red[2][4][TQ_BN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp & 3, wn = warp >> 2, g = lane >> 2, t = lane & 3;
  const int cb = blockIdx.x % ncb, b = blockIdx.x / ncb;
  const int c0 = cb * TQ_BN;
  const int64_t tiles = (N + TQ_BM - 1) / TQ_BM;
  double sd[4][2], sw[4][2];
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int q = 0; q < 2; ++q) sd[nt][q] = sw[nt][q] = 0.0;
  for (int64_t tile = b; tile < tiles; tile += nb) {
    const int64_t r0 = tile * TQ_BM;
    double acc[2][4][4];
    tq_mainloop<double>(acc, Q, ldq, N, k, R, ldr, kc, r0, c0, sA, sB);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int64_t r = r0 + wm * 32 + mt * 16 + g + h * 8;
            const int c = c0 + wn * 32 + nt * 8 + 2 * t + q;
            if (r < N && c < kc) {
              const double w = W[r + (int64_t)c * ldw];
              const double d = w - acc[mt][nt][h * 2 + q];
              sd[nt][q] = fma(d, d, sd[nt][q]);
              sw[nt][q] = fma(w, w, sw[nt][q]);
            }
          }
  }
  // lanes sharing t hold the same columns: sum over g (lane bits 2..4), then over the row warps
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double x = sd[nt][q], y = sw[nt][q];
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, o);
        y += __shfl_xor_sync(0xffffffffu, y, o);
      }
      if (g == 0) {
        red[0][wm][wn * 32 + nt * 8 + 2 * t + q] = x;
        red[1][wm][wn * 32 + nt * 8 + 2 * t + q] = y;
      }
    }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * TQ_BN; e += TQ_NT) {
    const int which = e / TQ_BN, c = e % TQ_BN;
    if (c0 + c < kc)
      P[(int64_t)(which * kc + c0 + c) * nb + b] =
          ((red[which][0][c] + red[which][1][c]) + red[which][2][c]) + red[which][3][c];
  }
}

int residual_norms_run(sqb_ctx* ctx, const double* W, int64_t ldw, const double* Q, int64_t ldq,
                       const double* R, int64_t ldr, int64_t N, int64_t k, int64_t kc, double* out) {
  if (kc == 0) return SQB_OK;
  static const bool old_path = [] { const char* e = getenv("SQB_RESID_OLD"); return e && e[0] == '1'; }();
  if (!old_path) {
    const int ncb = (int)((kc + TQ_BN - 1) / TQ_BN);
    const int64_t tiles = (N + TQ_BM - 1) / TQ_BM;
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (2 * (int64_t)ctx->sm_count + ncb - 1) / ncb));
    WsPlan plan;
    const size_t iP = plan.add(sizeof(double) * 2 * kc * nb);
    SQB_TRY(ws_reserve(ctx, plan.total));
    double* P = ws_ptr<double>(ctx, plan, iP);
    allow_dyn_smem(residual_dmma_kernel, (size_t)(TQ_SMEM));
    residual_dmma_kernel<<<(unsigned)(nb * ncb), TQ_NT, TQ_SMEM, ctx->stream>>>(W, ldw, Q, ldq, R, ldr, N, (int)k,
                                                                               (int)kc, ncb, nb, P);
    SQB_TRY(check_launch(ctx, "residual_dmma_kernel"));
    rowsum_kernel<<<(unsigned)((2 * kc + 255) / 256), 256, 0, ctx->stream>>>(P, (int)(2 * kc), nb, out);
    return check_launch(ctx, "rowsum_kernel");
  }

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
  // Q = [I;0] - U M is thin Q's tall-skinny product with K = r, nc = c: the
  // same DMMA kernel (the row-per-thread compact_q_kernel above took 2.97 ms
  // for 2^20 x 51 and held M in shared memory, which capped r c at 25600)
  static const bool old_path = [] { const char* e = getenv("SQB_THINQ_OLD"); return e && e[0] == '1'; }();
  if (!old_path) {
    allow_dyn_smem(thin_q_dmma_kernel<T>, (size_t)(TQ_SMEM));
    const int ncb = (int)((c + TQ_BN - 1) / TQ_BN);
    const int64_t tiles = (N + TQ_BM - 1) / TQ_BM;
    thin_q_dmma_kernel<T><<<(unsigned)(tiles * std::max(ncb, 1)), TQ_NT, TQ_SMEM, ctx->stream>>>(
        (const T*)U, ldu, N, (int)r, M, (int)c, std::max(ncb, 1), Q, ldq);
    return check_launch(ctx, "thin_q_dmma_kernel");
  }
  if ((int64_t)r * c * 8 > 200 * 1024) return set_error(ctx, SQB_ERR_ARG, "arnoldi_q: r*c too large");
  const size_t smem = sizeof(double) * std::max<int64_t>(1, r * c);
  if (smem > 48 * 1024)
    allow_dyn_smem(compact_q_kernel<T>, (size_t)(smem));
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
