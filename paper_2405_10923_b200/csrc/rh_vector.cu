// Single reflector for the public API (rh_vector, rhqr.py:51-97).
#include <algorithm>

#include "ctx.cuh"

namespace sqb {
template <typename T>
__device__ __forceinline__ typename Lo<T>::acc lazy_scale_rv(typename Lo<T>::acc w, double f, int scaling) {
  const double u = scaling == SQB_SCALE_SQRT2 ? __dmul_rn((double)w, f) : __ddiv_rn((double)w, f);
  return Lo<T>::from_double(u);
}
}  // namespace sqb

// ---------------------------------------------------------------------------
// single reflector (rh_vector, rhqr.py:51-97) for the public API
// ---------------------------------------------------------------------------
namespace sqb {

__global__ void rh_scalars_kernel(const double* __restrict__ y, int od, int jj, int scaling,
                                  double* scal, Status* st) {
  __shared__ double red[32];
  double part = 0.0;
  for (int r = jj + threadIdx.x; r < od; r += blockDim.x) part = fma(y[r], y[r], part);
  const double rho = sqrt(block_sum(part, red));
  if (threadIdx.x == 0) {
    const double sigma = y[jj] >= 0.0 ? 1.0 : -1.0;
    const double gamma = __dadd_rn(y[jj], sigma * rho);
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
    if (rho == 0.0) fail(st, SQB_ERR_BREAKDOWN, jj + 1, 0.0);
    else if (!isfinite(beta)) fail(st, SQB_ERR_BREAKDOWN, jj + 1, rho);
    double f, bo;
    if (scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
    else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    scal[0] = sigma; scal[1] = rho; scal[2] = bo; scal[3] = f; scal[4] = gamma;
  }
}

template <typename T>
__global__ void rh_vectors_kernel(const T* __restrict__ w, int64_t n, const double* __restrict__ y,
                                  int od, int jj, int scaling, const double* scal, T* __restrict__ u,
                                  double* __restrict__ s, const Status* st) {
  if (failed(st)) return;
  const double sigma = scal[0], rho = scal[1], f = scal[3], gamma = scal[4];
  const bool sq = scaling == SQB_SCALE_SQRT2;
  const int64_t tot = n > od ? n : od;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      double uh = i < jj ? 0.0 : (double)Lo<T>::load(w[i]);
      if (i == jj) uh = __dadd_rn(uh, sigma * rho);
      const double uv = sq ? __dmul_rn(uh, f) : __ddiv_rn(uh, f);
      u[i] = Lo<T>::store(Lo<T>::from_double(uv));
    }
    if (i < od) {
      const double yh = i < jj ? 0.0 : (i == jj ? gamma : y[i]);
      s[i] = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    }
  }
}

template <typename T>
static int rh_vector_t(sqb_ctx* ctx, int scaling, const void* w, int64_t n, const double* y, int64_t od,
                       int64_t j, void* u, double* s, double* scal) {
  rh_scalars_kernel<<<1, 256, 0, ctx->stream>>>(y, (int)od, (int)(j - 1), scaling, scal, ctx->d_status);
  SQB_TRY(check_launch(ctx, "rh_scalars_kernel"));
  const int64_t tot = std::max(n, od);
  rh_vectors_kernel<T><<<(unsigned)std::min<int64_t>((tot + 255) / 256, 4 * 148), 256, 0, ctx->stream>>>(
      (const T*)w, n, y, (int)od, (int)(j - 1), scaling, scal, (T*)u, s, ctx->d_status);
  return check_launch(ctx, "rh_vectors_kernel");
}

int rh_vector_dispatch(sqb_ctx* ctx, int scaling, int lo_dtype, const void* w, int64_t n, const double* y,
                       int64_t od, int64_t j, void* u, double* s, double* scal) {
  switch (lo_dtype) {
    case SQB_F64: return rh_vector_t<double>(ctx, scaling, w, n, y, od, j, u, s, scal);
    case SQB_F32: return rh_vector_t<float>(ctx, scaling, w, n, y, od, j, u, s, scal);
    case SQB_F16: return rh_vector_t<__half>(ctx, scaling, w, n, y, od, j, u, s, scal);
    case SQB_BF16: return rh_vector_t<__nv_bfloat16>(ctx, scaling, w, n, y, od, j, u, s, scal);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb
