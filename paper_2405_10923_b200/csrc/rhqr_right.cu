// Right-looking RHQR (rhqr_right, rhqr.py:270-301).
//
// Per column c:  Y = Psi Wl[:, c:]               (K1 over the trailing block)
//                step = rh_vector(Wl[:, c], Y[:, 0], c + 1)
//                R[:c, c] = Wl[:c, c];  R[c, c] = -sigma rho
//                coef = beta (s^t Y[:, 1:])      (high precision)
//                Wl[:, c+1:] = fl(Wl[:, c+1:] - fl(u coef^t))   (rank-1, one HBM pass)
// then T = t_factor_from_sketches(S).  The trailing block is re-sketched every
// step, as in the reference — this variant exists for completeness and as the
// right-looking baseline; rhqr_left/rhqr_block are the fast paths.
#include <algorithm>

#include "sketch.cuh"

namespace sqb {

int rh_vector_dispatch(sqb_ctx*, int, int, const void*, int64_t, const double*, int64_t, int64_t, void*,
                       double*, double*);

// R column c and the per-column scalars from rh_scalars_kernel's scal[]
template <typename T>
__global__ void right_post_kernel(const T* __restrict__ wc, int c, const double* scal, double* R, int64_t ldr,
                                  double* sig, double* rho, double* bet, const Status* st) {
  if (failed(st)) return;
  for (int i = threadIdx.x; i < c; i += blockDim.x) R[i + (int64_t)c * ldr] = (double)Lo<T>::load(wc[i]);
  if (threadIdx.x == 0) {
    R[c + (int64_t)c * ldr] = -scal[0] * scal[1];
    sig[c] = scal[0];
    rho[c] = scal[1];
    bet[c] = scal[2];
  }
}

// coef[j] = beta * (s^t Y[:, 1 + j]) in fp64, rounded to low (rhqr.py:296)
__global__ void right_coef_kernel(const double* __restrict__ s, const double* __restrict__ Y, int64_t ldy, int od,
                                  const double* scal, double* coef, const Status* st) {
  __shared__ double red[32];
  if (failed(st)) return;
  const int j = blockIdx.x;
  const double* y = Y + (int64_t)(j + 1) * ldy;
  double d = 0.0;
  for (int i = threadIdx.x; i < od; i += blockDim.x) d = fma(s[i], y[i], d);
  d = block_sum(d, red);
  if (threadIdx.x == 0) coef[j] = __dmul_rn(scal[2], d);
}

// X[:, j] = fl(X[:, j] - fl(u * coef_lo[j])) for j < k  (rhqr.py:297-298: np.outer then subtract)
template <typename T>
__global__ void __launch_bounds__(256)
rank1_update_kernel(const T* __restrict__ u, const double* __restrict__ coef, T* X, int64_t ldx, int64_t N,
                    int k, const Status* st) {
  using A = typename Lo<T>::acc;
  if (failed(st)) return;
  const int j = blockIdx.y;
  const A cj = Lo<T>::from_double(coef[j]);
  T* x = X + (int64_t)j * ldx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = Lo<T>::store(Lo<T>::sub(Lo<T>::load(x[i]), Lo<T>::mul(Lo<T>::load(u[i]), cj)));
}

template <typename T>
static int rhqr_right_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                        int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds, double* R, int64_t ldr,
                        double* sigmas, double* rhos, double* betas) {
  const int64_t od = m + sk->ell;
  const size_t esz = sizeof(T);
  const int64_t ldx = (N + 7) / 8 * 8;
  WsPlan plan;
  const size_t iX = plan.add(esz * ldx * m);
  const size_t iY = plan.add(sizeof(double) * od * m);
  const size_t iC = plan.add(sizeof(double) * (m + 1));
  const size_t isc = plan.add(sizeof(double) * 8);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, m));
  SQB_TRY(ws_reserve(ctx, plan.total));
  T* X = ws_ptr<T>(ctx, plan, iX);
  double* Y = ws_ptr<double>(ctx, plan, iY);
  double* coef = ws_ptr<double>(ctx, plan, iC);
  double* scal = ws_ptr<double>(ctx, plan, isc);
  void* P = ws_ptr<void>(ctx, plan, iP);
  Status* st = ctx->d_status;
  SQB_CUDA_TRY(cudaMemcpy2DAsync(X, ldx * esz, W, ldw * esz, N * esz, m, cudaMemcpyDeviceToDevice, ctx->stream));
  SQB_CUDA_TRY(cudaMemset2DAsync(R, ldr * sizeof(double), 0, m * sizeof(double), m, ctx->stream));
  for (int64_t c = 0; c < m; ++c) {
    const int64_t k = m - c;
    T* Xc = X + c * ldx;
    SQB_TRY(launch_copy_top(ctx, Lo<T>::code, Xc, ldx, m, k, Y, od, st));
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, Xc + m, ldx, k, Y, od, m, P, st));
    SQB_TRY(rh_vector_dispatch(ctx, scaling, Lo<T>::code, Xc, N, Y, od, c + 1, (T*)U + c * ldu, S + c * lds, scal));
    right_post_kernel<T><<<1, 256, 0, ctx->stream>>>(Xc, (int)c, scal, R, ldr, sigmas, rhos, betas, st);
    SQB_TRY(check_launch(ctx, "right_post_kernel"));
    if (k > 1) {
      right_coef_kernel<<<(unsigned)(k - 1), 256, 0, ctx->stream>>>(S + c * lds, Y, od, (int)od, scal, coef, st);
      SQB_TRY(check_launch(ctx, "right_coef_kernel"));
      const unsigned gx = (unsigned)std::min<int64_t>((N + 255) / 256, std::max<int64_t>(1, 4 * 148 / (k - 1) + 1));
      rank1_update_kernel<T><<<dim3(gx, (unsigned)(k - 1)), 256, 0, ctx->stream>>>(
          (const T*)U + c * ldu, coef, Xc + ldx, ldx, N, (int)(k - 1), st);
      SQB_TRY(check_launch(ctx, "rank1_update_kernel"));
    }
  }
  return SQB_OK;
}

int rhqr_right_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W, int64_t N,
                        int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds, double* R,
                        int64_t ldr, double* sigmas, double* rhos, double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rhqr_right_t<double>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rhqr_right_t<float>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rhqr_right_t<__half>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rhqr_right_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb
