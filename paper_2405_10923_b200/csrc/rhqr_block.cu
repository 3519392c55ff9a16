// Blocked left-looking RHQR (rhqr_block, rhqr.py:334-365) and the compact-form
// T recovered from the sketches alone (t_factor_from_sketches, rhqr.py:122-132).
//
// Per panel [j0, j1):   X = W[:, j0:j1]
//   for every earlier panel p (in order, each one re-sketching X, rhqr.py:357-360):
//       Y = Psi X                      (K1, b columns at once)
//       C = T_p^t (S_p^t Y)            (coef_kernel, high precision)
//       X = fl(X - fl(U_p C))          (panel_update_kernel: one HBM pass, b_p x b FMAs per row)
//   the left-looking sweep over X with pivot offset j0 (left_sweep_t, the
//   rhqr_left machinery with StepArgs::off).
// The per-panel T blocks are returned on the diagonal of an m x m array
// (BlockRHQRFactors.panels[k].T); the stacked global T comes from
// t_factor_from_sketches(S).
#include <algorithm>

#include "rhqr_kernels.cuh"

namespace sqb {

template <typename T>
int left_sweep_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                 int64_t ldw, int64_t ncol, int64_t off, void* U, int64_t ldu, double* S, int64_t lds,
                 double* Tm, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                 double* betas, void* ws_base);
size_t left_sweep_ws_bytes(const sqb_sketch* sk, int code, int64_t m, int64_t ncol);
__global__ void coef_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ Tm, int64_t ldt,
                            int transpose_t, const double* __restrict__ Y, int64_t ldy, int od, int r,
                            double* __restrict__ C, int64_t ldc, const Status* st);
__global__ void upper_tri_solve_kernel(const double* __restrict__ R, int64_t ldr, int m,
                                       const double* __restrict__ B, int64_t ldb, double* __restrict__ X,
                                       int64_t ldx, Status* st);

// X[:, :b] = fl(X - fl(U[:, :bp] C)), C (bp x b) in the high precision rounded
// to low once (rhqr.py:360).  A CTA owns PU_RB rows; U rows are staged through
// shared memory KC columns at a time, the two thread halves own 16 output
// columns each.
constexpr int PU_RB = 128, PU_KC = 32, PU_JC = 16;

template <typename T>
__global__ void __launch_bounds__(256)
panel_update_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int bp, const double* __restrict__ C,
                    int64_t ldc, T* X, int64_t ldx, int b, const Status* st) {
  using A = typename Lo<T>::acc;
  __shared__ T Us[PU_KC][PU_RB];
  __shared__ A Cs[PU_KC][2 * PU_JC];
  if (failed(st)) return;
  const int row = threadIdx.x % PU_RB, h = threadIdx.x / PU_RB;
  for (int64_t r0 = (int64_t)blockIdx.x * PU_RB; r0 < N; r0 += (int64_t)gridDim.x * PU_RB) {
    const int64_t i = r0 + row;
    for (int jb = 0; jb < b; jb += 2 * PU_JC) {
      A acc[PU_JC];
#pragma unroll
      for (int j = 0; j < PU_JC; ++j) acc[j] = A(0);
      for (int kb = 0; kb < bp; kb += PU_KC) {
        __syncthreads();
        T v[PU_KC * PU_RB / 256];
#pragma unroll
        for (int q = 0; q < PU_KC * PU_RB / 256; ++q) {
          const int e = threadIdx.x + q * 256, k = e / PU_RB, r = e % PU_RB;
          v[q] = (kb + k < bp && r0 + r < N) ? U[(r0 + r) + (int64_t)(kb + k) * ldu] : Lo<T>::store(A(0));
        }
#pragma unroll
        for (int q = 0; q < PU_KC * PU_RB / 256; ++q) {
          const int e = threadIdx.x + q * 256;
          Us[e / PU_RB][e % PU_RB] = v[q];
        }
        for (int e = threadIdx.x; e < PU_KC * 2 * PU_JC; e += 256) {
          const int k = e / (2 * PU_JC), j = e % (2 * PU_JC);
          Cs[k][j] = (kb + k < bp && jb + j < b) ? Lo<T>::from_double(C[(kb + k) + (int64_t)(jb + j) * ldc]) : A(0);
        }
        __syncthreads();
        const int kn = min(PU_KC, bp - kb);
        for (int k = 0; k < kn; ++k) {
          const A u = Lo<T>::load(Us[k][row]);
#pragma unroll
          for (int j = 0; j < PU_JC; ++j) acc[j] = fma(u, Cs[k][h * PU_JC + j], acc[j]);
        }
      }
      if (i < N) {
#pragma unroll
        for (int j = 0; j < PU_JC; ++j) {
          const int col = jb + h * PU_JC + j;
          if (col < b) {
            T* x = X + i + (int64_t)col * ldx;
            *x = Lo<T>::store(Lo<T>::sub(Lo<T>::load(*x), Lo<T>::rnd(acc[j])));
          }
        }
      }
    }
  }
}

template <typename T>
static int panel_update(sqb_ctx* ctx, const T* U, int64_t ldu, int64_t N, int64_t bp, const double* C, int64_t ldc,
                        T* X, int64_t ldx, int64_t b) {
  const int64_t blocks = (N + PU_RB - 1) / PU_RB;
  const unsigned grid = (unsigned)std::min<int64_t>(blocks, 8 * (int64_t)ctx->sm_count);
  panel_update_kernel<T><<<grid, 256, 0, ctx->stream>>>(U, ldu, N, (int)bp, C, ldc, X, ldx, (int)b, ctx->d_status);
  return check_launch(ctx, "panel_update_kernel");
}

template <typename T>
static int rhqr_block_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                        int64_t ldw, int64_t bs, void* U, int64_t ldu, double* S, int64_t lds, double* Tm,
                        int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  const int64_t od = m + sk->ell;
  const int64_t b0 = std::min(bs, m);
  constexpr int VN = VecN<T>::n;
  // panel buffer: row m of every column 16-byte aligned (vector path of the sweep)
  const int64_t ldx = (N + VN - 1) / VN * VN;
  const int64_t shift = (VN - m % VN) % VN;
  WsPlan plan;
  const size_t iX = plan.add(sizeof(T) * (ldx * b0 + shift));
  const size_t iY = plan.add(sizeof(double) * od * b0);
  const size_t iC = plan.add(sizeof(double) * m * b0);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, b0));
  const size_t iSw = plan.add(left_sweep_ws_bytes(sk, Lo<T>::code, m, b0));
  SQB_TRY(ws_reserve(ctx, plan.total));
  T* X = ws_ptr<T>(ctx, plan, iX) + shift;
  double* Y = ws_ptr<double>(ctx, plan, iY);
  double* C = ws_ptr<double>(ctx, plan, iC);
  void* P = ws_ptr<void>(ctx, plan, iP);
  void* sw = ws_ptr<void>(ctx, plan, iSw);
  Status* st = ctx->d_status;
  const size_t esz = sizeof(T);
  // T holds the panel triangles on its diagonal blocks; the rest is zero
  SQB_CUDA_TRY(cudaMemset2DAsync(Tm, ldt * sizeof(double), 0, m * sizeof(double), m, ctx->stream));
  for (int64_t j0 = 0; j0 < m; j0 += bs) {
    const int64_t b = std::min(bs, m - j0);
    SQB_CUDA_TRY(cudaMemcpy2DAsync(X, ldx * esz, (const T*)W + j0 * ldw, ldw * esz, N * esz, b,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    for (int64_t p0 = 0; p0 < j0; p0 += bs) {
      const int64_t bp = std::min(bs, j0 - p0);
      SQB_TRY(launch_copy_top(ctx, Lo<T>::code, X, ldx, m, b, Y, od, st));
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, X + m, ldx, b, Y, od, m, P, st));
      coef_kernel<<<(unsigned)b, 256, sizeof(double) * bp, ctx->stream>>>(
          S + p0 * lds, lds, Tm + p0 + p0 * ldt, ldt, 1, Y, od, (int)od, (int)bp, C, bp, st);
      SQB_TRY(check_launch(ctx, "coef_kernel"));
      SQB_TRY(panel_update<T>(ctx, (const T*)U + p0 * ldu, ldu, N, bp, C, bp, X, ldx, b));
    }
    SQB_TRY(left_sweep_t<T>(ctx, sk, scaling, X, N, m, ldx, b, j0, (T*)U + j0 * ldu, ldu, S + j0 * lds, lds,
                            Tm + j0 + j0 * ldt, ldt, R + j0 * ldr, ldr, sigmas + j0, rhos + j0, betas + j0, sw));
  }
  return SQB_OK;
}

int rhqr_block_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W, int64_t N,
                        int64_t m, int64_t ldw, int64_t bs, void* U, int64_t ldu, double* S, int64_t lds,
                        double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                        double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rhqr_block_t<double>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rhqr_block_t<float>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rhqr_block_t<__half>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rhqr_block_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

// Tinv = strict upper triangle of S^t S plus half its diagonal, and B = I
// (rhqr.py:129-131); one warp per entry (i <= j)
__global__ void tinv_kernel(const double* __restrict__ S, int64_t lds, int od, int k, double* __restrict__ Tinv,
                            double* __restrict__ B) {
  const int i = blockIdx.x, j = blockIdx.y, lane = threadIdx.x;
  if (i > j) {
    if (lane == 0) { Tinv[i + (int64_t)j * k] = 0.0; B[i + (int64_t)j * k] = 0.0; }
    return;
  }
  double d = 0.0;
  for (int r = lane; r < od; r += 32) d = fma(S[r + (int64_t)i * lds], S[r + (int64_t)j * lds], d);
  d = warp_sum(d);
  if (lane == 0) {
    Tinv[i + (int64_t)j * k] = i == j ? d / 2.0 : d;
    B[i + (int64_t)j * k] = i == j ? 1.0 : 0.0;
  }
}

}  // namespace sqb

extern "C" int sqb_t_factor(sqb_ctx* ctx, const double* S, int64_t lds, int64_t od, int64_t k, double* T,
                            int64_t ldt) {
  using namespace sqb;
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  if (k < 1) return SQB_OK;
  if (lds < od || ldt < k) return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  WsPlan plan;
  const size_t iA = plan.add(sizeof(double) * k * k);
  const size_t iB = plan.add(sizeof(double) * k * k);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* Tinv = ws_ptr<double>(ctx, plan, iA);
  double* B = ws_ptr<double>(ctx, plan, iB);
  tinv_kernel<<<dim3((unsigned)k, (unsigned)k), 32, 0, ctx->stream>>>(S, lds, (int)od, (int)k, Tinv, B);
  SQB_TRY(check_launch(ctx, "tinv_kernel"));
  upper_tri_solve_kernel<<<(unsigned)k, 256, sizeof(double) * k, ctx->stream>>>(Tinv, k, (int)k, B, k, T, ldt,
                                                                               ctx->d_status);
  return check_launch(ctx, "upper_tri_solve_kernel");
}
