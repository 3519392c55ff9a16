// recRHQR on the device (rec_rhqr, rhqr.py:368-395):
//   Z = Psi W (one sketch of all columns; K2 DMMA for a Gaussian Omega),
//   K5  householder_qr(Z) in the high precision (baselines.py:33-89), one CTA,
//   Mfac = triu(T^t S^t Z), zero-diagonal check (rhqr.py:387-391),
//   K6  U2 = W2 Mfac^{-1} by row-wise forward substitution (right_tri_solve,
//       linalg.py:119-129), streamed over the n-m rows,
//   U = [S[:m]; round_to(U2, low)].
#include <algorithm>
#include <cfloat>

#include "pdl.cuh"
#include "sketch.cuh"

namespace sqb {

constexpr int HQR_NT = 1024;

// K5: left-looking Householder QR with compact T of Z (od x m), fp64 throughout.
// Writes S = U_z (od x m), T, R (m x m), sigmas/rhos/betas.
__global__ void __launch_bounds__(HQR_NT)
hqr_kernel(const double* __restrict__ Z, int64_t ldz, int od, int m, int scaling, double* S,
           int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr, double* sig, double* rhos,
           double* bets, Status* st) {
  extern __shared__ double sm[];
  double* w = sm;          // [od]
  double* g = w + od;      // [m]
  double* cf = g + m;      // [m]
  double* red = cf + m;    // [32]
  __shared__ double scal[4];
  if (failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = HQR_NT / 32;
  for (int e = tid; e < m * m; e += HQR_NT) {
    T[(e % m) + (int64_t)(e / m) * ldt] = 0.0;
    R[(e % m) + (int64_t)(e / m) * ldr] = 0.0;
  }
  for (int c = 0; c < m; ++c) {
    for (int r = tid; r < od; r += HQR_NT) w[r] = Z[r + (int64_t)c * ldz];
    __syncthreads();
    if (c > 0) {
      // coef = T[:c,:c]^t (U[:, :c]^t w); w = w - U[:, :c] coef   (baselines.py:57-59)
      for (int k = warp; k < c; k += nw) {
        const double* uk = S + (int64_t)k * lds;
        double d = 0.0;
        for (int r = k + lane; r < od; r += 32) d = fma(uk[r], w[r], d);
        d = warp_sum(d);
        if (lane == 0) g[k] = d;
      }
      __syncthreads();
      for (int j = warp; j < c; j += nw) {
        double d = 0.0;
        for (int k = lane; k <= j; k += 32) d = fma(T[k + (int64_t)j * ldt], g[k], d);
        d = warp_sum(d);
        if (lane == 0) cf[j] = d;
      }
      __syncthreads();
      for (int r = tid; r < od; r += HQR_NT) {
        double d = 0.0;
        const int kmax = min(c, r + 1);  // U[r, k] = 0 for k > r
        for (int k = 0; k < kmax; ++k) d = fma(S[r + (int64_t)k * lds], cf[k], d);
        w[r] = w[r] - d;
      }
      __syncthreads();
    }
    double p = 0.0;
    for (int r = c + tid; r < od; r += HQR_NT) p = fma(w[r], w[r], p);
    const double rho = sqrt(block_sum(p, red));
    if (tid == 0) {
      const double sigma = w[c] >= 0.0 ? 1.0 : -1.0;
      const double gamma = __dadd_rn(w[c], sigma * rho);
      const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
      double f, bo;
      if (scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
      else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
      scal[0] = sigma; scal[1] = gamma; scal[2] = f; scal[3] = bo;
      if (rho == 0.0) fail(st, SQB_ERR_BREAKDOWN, c + 1, 0.0);
      sig[c] = sigma; rhos[c] = rho; bets[c] = bo;
      R[c + (int64_t)c * ldr] = -sigma * rho;
    }
    __syncthreads();
    if (rho == 0.0) return;
    const double gamma = scal[1], f = scal[2], bo = scal[3];
    const bool sq = scaling == SQB_SCALE_SQRT2;
    for (int r = tid; r < od; r += HQR_NT) {
      const double uh = r < c ? 0.0 : (r == c ? gamma : w[r]);
      S[r + (int64_t)c * lds] = sq ? __dmul_rn(uh, f) : __ddiv_rn(uh, f);
      if (r < c) R[r + (int64_t)c * ldr] = w[r];
    }
    __syncthreads();
    if (c > 0) {
      // T[:c, c] = -beta T[:c,:c] (U[:, :c]^t u)   (baselines.py:78-81)
      const double* uc = S + (int64_t)c * lds;
      for (int k = warp; k < c; k += nw) {
        const double* uk = S + (int64_t)k * lds;
        double d = 0.0;
        for (int r = c + lane; r < od; r += 32) d = fma(uk[r], uc[r], d);  // u[r] = 0 for r < c
        d = warp_sum(d);
        if (lane == 0) g[k] = d;
      }
      __syncthreads();
      for (int i = warp; i < c; i += nw) {
        double d = 0.0;
        for (int k = i + lane; k < c; k += 32) d = fma(T[i + (int64_t)k * ldt], g[k], d);
        d = warp_sum(d);
        if (lane == 0) T[i + (int64_t)c * ldt] = __dmul_rn(-bo, d);
      }
    }
    if (tid == 0) T[c + (int64_t)c * ldt] = bo;
    __syncthreads();
  }
}

// Mfac[:, j] = triu(T^t (S^t Z[:, j]))  — one CTA per column j
__global__ void __launch_bounds__(256)
mfac_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ T, int64_t ldt,
            const double* __restrict__ Z, int64_t ldz, int od, int m, double* M, const Status* st) {
  extern __shared__ double g[];  // [m]
  if (failed(st)) return;
  const int j = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* zj = Z + (int64_t)j * ldz;
  for (int k = warp; k < m; k += 8) {
    const double* sk = S + (int64_t)k * lds;
    double d = 0.0;
    for (int r = k + lane; r < od; r += 32) d = fma(sk[r], zj[r], d);
    d = warp_sum(d);
    if (lane == 0) g[k] = d;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += 256) {
    double d = 0.0;
    if (i <= j)
      for (int k = 0; k <= i; ++k) d = fma(T[k + (int64_t)i * ldt], g[k], d);
    M[i + (int64_t)j * m] = d;
  }
}

// zero-diagonal check (rhqr.py:388-391): argmin |diag| < DBL_MIN -> breakdown
__global__ void mfac_check_kernel(const double* M, int m, Status* st) {
  if (threadIdx.x != 0 || failed(st)) return;
  int k = 0;
  double dmin = fabs(M[0]);
  for (int j = 1; j < m; ++j) {
    const double d = fabs(M[j + (int64_t)j * m]);
    if (d < dmin) { dmin = d; k = j; }
  }
  if (dmin < DBL_MIN) fail(st, SQB_ERR_BREAKDOWN, k + 1, -1.0);
}

// K6: U2 = W2 Mfac^{-1}: per row x, x Mfac = w by forward substitution in fp64
// (x_j = (w_j - sum_{i<j} x_i M_ij) / M_jj), x kept in registers (m <= MAXM).
template <typename T, int MAXM>
__global__ void __launch_bounds__(128)
trsm_rows_kernel(const T* __restrict__ W2, int64_t ldw, int64_t n, int m, const double* __restrict__ M,
                 T* __restrict__ U2, int64_t ldu, const Status* st) {
  extern __shared__ double sM[];  // m x m, column-major
  if (failed(st)) return;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sM[e] = M[e];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double x[MAXM];
#pragma unroll
    for (int j = 0; j < MAXM; ++j)
      if (j < m) x[j] = (double)Lo<T>::load(W2[r + (int64_t)j * ldw]);
#pragma unroll
    for (int j = 0; j < MAXM; ++j) {
      if (j < m) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < j; ++i) s = fma(x[i], sM[i + j * m], s);
        x[j] = __ddiv_rn(x[j] - s, sM[j + j * m]);
      }
    }
#pragma unroll
    for (int j = 0; j < MAXM; ++j)
      if (j < m) U2[r + (int64_t)j * ldu] = Lo<T>::store(Lo<T>::from_double(x[j]));
  }
}

// generic fallback for wide m: x in global scratch (the output itself)
template <typename T>
__global__ void __launch_bounds__(128)
trsm_rows_generic_kernel(const T* __restrict__ W2, int64_t ldw, int64_t n, int m,
                         const double* __restrict__ M, T* __restrict__ U2, int64_t ldu, double* X,
                         const Status* st) {
  if (failed(st)) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int i = 0; i < j; ++i) s = fma(X[r + (int64_t)i * n], M[i + (int64_t)j * m], s);
      const double xj = __ddiv_rn((double)Lo<T>::load(W2[r + (int64_t)j * ldw]) - s, M[j + (int64_t)j * m]);
      X[r + (int64_t)j * n] = xj;
      U2[r + (int64_t)j * ldu] = Lo<T>::store(Lo<T>::from_double(xj));
    }
  }
}

template <typename T>
__global__ void top_from_s_kernel(const double* S, int64_t lds, int m, T* U, int64_t ldu, const Status* st) {
  if (failed(st)) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x)
    U[(e % m) + (int64_t)(e / m) * ldu] = Lo<T>::store(Lo<T>::from_double(S[(e % m) + (int64_t)(e / m) * lds]));
}

template <typename T>
static int rec_rhqr_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                      int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt,
                      double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  const int64_t n = N - m, od = m + sk->ell;
  WsPlan plan;
  const size_t iZ = plan.add(sizeof(double) * od * m);
  const size_t iM = plan.add(sizeof(double) * m * m);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, m));
  const size_t iX = plan.add(m > 64 ? sizeof(double) * n * m : 8);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* Z = ws_ptr<double>(ctx, plan, iZ);
  double* M = ws_ptr<double>(ctx, plan, iM);
  Status* st = ctx->d_status;
  const size_t esz = sizeof(T);
  // Z = Psi W  (rhqr.py:382)
  SQB_TRY(launch_copy_top(ctx, Lo<T>::code, W, ldw, m, m, Z, od, st));
  SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)W + m * esz, ldw, m, Z, od, m,
                        ws_ptr<void>(ctx, plan, iP), st));
  // K5: householder_qr(Z) (rhqr.py:383)
  const size_t hsm = sizeof(double) * (od + 2 * m + 32);
  cudaFuncSetAttribute(hqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(hsm, 48 << 10));
  hqr_kernel<<<1, HQR_NT, hsm, ctx->stream>>>(Z, od, (int)od, (int)m, scaling, S, lds, Tm, ldt, R, ldr,
                                              sigmas, rhos, betas, st);
  SQB_TRY(check_launch(ctx, "hqr_kernel"));
  // Mfac = triu(T^t S^t Z) and its diagonal check (rhqr.py:387-391)
  mfac_kernel<<<(unsigned)m, 256, sizeof(double) * m, ctx->stream>>>(S, lds, Tm, ldt, Z, od, (int)od, (int)m, M, st);
  SQB_TRY(check_launch(ctx, "mfac_kernel"));
  mfac_check_kernel<<<1, 32, 0, ctx->stream>>>(M, (int)m, st);
  SQB_TRY(check_launch(ctx, "mfac_check_kernel"));
  // K6: U2 = W2 Mfac^{-1}; U = [S[:m]; U2]
  const T* W2 = (const T*)W + m;
  T* U2 = (T*)U + m;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 8 * 148));
  const size_t msm = sizeof(double) * m * m;
  if (m <= 16) {
    trsm_rows_kernel<T, 16><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
  } else if (m <= 32) {
    trsm_rows_kernel<T, 32><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
  } else if (m <= 64) {
    trsm_rows_kernel<T, 64><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
  } else {
    trsm_rows_generic_kernel<T><<<grid, 128, 0, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu,
                                                                ws_ptr<double>(ctx, plan, iX), st);
  }
  SQB_TRY(check_launch(ctx, "trsm_rows_kernel"));
  top_from_s_kernel<T><<<(unsigned)std::max<int64_t>(1, (m * m + 255) / 256), 256, 0, ctx->stream>>>(
      S, lds, (int)m, (T*)U, ldu, st);
  return check_launch(ctx, "top_from_s_kernel");
}

int rec_rhqr_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                      int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                      double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                      double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rec_rhqr_t<double>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rec_rhqr_t<float>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rec_rhqr_t<__half>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rec_rhqr_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb
