// Householder QR of a TALL fp64 matrix (p x m, p beyond one CTA's shared
// memory) — the classic baseline the paper measures RHQR against
// (baselines.py:33-89: left-looking, compact T) and the QR behind the SVD
// condition number of an ill-conditioned W (linalg.py:151-160).
//
// Per column c the reference forms, in the high precision,
//   coef = T_c^t (U_c^t w),  w <- w - U_c coef,  rh_vector scalars from ||w[c:]||,
//   u = scaled (0, gamma, w[c+1:]),  T[:c, c] = -beta T_c (U_c^t u),  R[:, c]
// i.e. THREE streams over the c finished reflectors (two transposed GEMVs and
// one GEMV) — the p-dimensional inner products RHQR replaces by sketches.
// Here: persistent row-block kernels for the three streams (the GEMV is
// gemv.cuh's; the transposed GEMV keeps its block of x in registers and
// reduces four columns at a time), one-CTA kernels for the c x c algebra,
// partial sums combined in a fixed order.  ~1.5 m^2 p values of traffic
// (config 2's shape: 206 GB, 3x rhqr_left).
#include <algorithm>

#include "ctx.cuh"
#include "gemv.cuh"
#include "vec.cuh"

namespace sqb {

constexpr int HT_NV = 4;                                   // 16-byte runs per thread and column
constexpr int HT_ROWS = GEMV_NT * HT_NV * 2;               // rows per block step (2048)

struct HtScal {  // scalars of the current column (device)
  double rho, sigma, gamma, beta, f, wc;
};

// P[b][k] = sum over the rows >= r_lo of CTA b's row blocks of U[r, k] x[r], k < c
__global__ void __launch_bounds__(GEMV_NT, 2)
hqrt_dots_kernel(const double* __restrict__ U, int64_t ldu, int64_t p, int c, const double* __restrict__ x,
                 int64_t r_lo, double* __restrict__ P, int ldp, const Status* st) {
  extern __shared__ double ht_sm[];  // [8 warps][c] partials of this row block, then [c] running sums
  double* wpart = ht_sm;
  double* run = ht_sm + (GEMV_NT / 32) * c;
  if (failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < c; k += GEMV_NT) run[k] = 0.0;
  __syncthreads();
  for (int64_t r0 = (int64_t)blockIdx.x * HT_ROWS; r0 < p; r0 += (int64_t)gridDim.x * HT_ROWS) {
    // this thread's rows of x (zero outside [r_lo, p))
    double xv[HT_NV][2];
    const bool full = r0 + HT_ROWS <= p;
#pragma unroll
    for (int v = 0; v < HT_NV; ++v)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t i = r0 + (int64_t)(v * GEMV_NT + tid) * 2 + j;
        xv[v][j] = (i >= r_lo && i < p) ? x[i] : 0.0;
      }
    auto ld = [&](double (&u)[HT_NV][2], int k) {
      const double* col = U + r0 + (int64_t)k * ldu;
#pragma unroll
      for (int v = 0; v < HT_NV; ++v) {
        const int64_t o = (int64_t)(v * GEMV_NT + tid) * 2;
        if (full) vload_stream<double>(col + o, u[v]);
        else load_run<double, 2>(col, o, p - r0, u[v]);
      }
    };
    auto dot = [&](const double (&u)[HT_NV][2]) {
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int v = 0; v < HT_NV; ++v) {
        d0 = fma(u[v][0], xv[v][0], d0);
        d1 = fma(u[v][1], xv[v][1], d1);
      }
      return d0 + d1;
    };
    double u0[HT_NV][2], u1[HT_NV][2];
    if (c > 0) ld(u0, 0);
    int k = 0;
    for (; k + 2 <= c; k += 2) {
      ld(u1, k + 1);
      double a = dot(u0);
      if (k + 2 < c) ld(u0, k + 2);
      double b = dot(u1);
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == 0) { wpart[warp * c + k] = a; wpart[warp * c + k + 1] = b; }
    }
    if (k < c) {
      const double a = warp_sum(dot(u0));
      if (lane == 0) wpart[warp * c + k] = a;
    }
    __syncthreads();
    for (int kk = tid; kk < c; kk += GEMV_NT) {
      double s = 0.0;
#pragma unroll
      for (int w8 = 0; w8 < GEMV_NT / 32; ++w8) s += wpart[w8 * c + kk];
      run[kk] += s;
    }
    __syncthreads();
  }
  for (int k = tid; k < c; k += GEMV_NT) P[(int64_t)blockIdx.x * ldp + k] = run[k];
}

// coef = T_c^t (sum_b P[b]) (baselines.py:59)
__global__ void __launch_bounds__(256)
hqrt_coef_kernel(const double* __restrict__ P, int nb, int ldp, const double* __restrict__ T, int64_t ldt, int c,
                 double* __restrict__ coef, const Status* st) {
  extern __shared__ double d[];
  if (failed(st)) return;
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += P[(int64_t)b * ldp + k];
    d[k] = s;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i <= j; ++i) s = fma(T[i + (int64_t)j * ldt], d[i], s);
    coef[j] = s;
  }
}

// w = A[:, c] - U_c coef, stored unscaled in U[:, c]; Pn[b] = sum of w[r]^2 over CTA b's rows >= c
__global__ void __launch_bounds__(GEMV_NT, 2)
hqrt_update_kernel(const double* __restrict__ A, int64_t lda, double* U, int64_t ldu, int64_t p, int c,
                   const double* __restrict__ coef, double* __restrict__ Pn, const Status* st) {
  extern __shared__ double cs[];
  __shared__ double red[32];
  if (failed(st)) return;
  for (int k = threadIdx.x; k < c; k += blockDim.x) cs[k] = coef[k];
  __syncthreads();
  const double* a = A + (int64_t)c * lda;
  double* uc = U + (int64_t)c * ldu;
  double nrm = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * HT_ROWS; r0 < p; r0 += (int64_t)gridDim.x * HT_ROWS) {
    double acc[HT_NV][2];
    gemv_rows<double, HT_NV>(U, ldu, r0, p, c, cs, acc);
#pragma unroll
    for (int v = 0; v < HT_NV; ++v)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t i = r0 + (int64_t)(v * GEMV_NT + threadIdx.x) * 2 + j;
        if (i < p) {
          const double w = __dsub_rn(a[i], acc[v][j]);
          uc[i] = w;
          if (i >= c) nrm = fma(w, w, nrm);
        }
      }
  }
  nrm = block_sum(nrm, red);
  if (threadIdx.x == 0) Pn[blockIdx.x] = nrm;
}

// rh_vector's scalars (baselines.py:61-76), R's column (:85-86), breakdown (:63)
__global__ void __launch_bounds__(256)
hqrt_scalars_kernel(const double* __restrict__ Pn, int nb, const double* __restrict__ U, int64_t ldu, int c,
                    int scaling, double* __restrict__ R, int64_t ldr, double* sigmas, double* rhos, double* betas,
                    HtScal* sc, Status* st) {
  if (failed(st)) return;
  const double* uc = U + (int64_t)c * ldu;
  for (int r = threadIdx.x; r < c; r += blockDim.x) R[r + (int64_t)c * ldr] = uc[r];
  if (threadIdx.x == 0) {
    double r2 = 0.0;
    for (int b = 0; b < nb; ++b) r2 += Pn[b];
    const double rho = sqrt(r2);
    const double wc = uc[c];
    const double sigma = wc >= 0.0 ? 1.0 : -1.0;
    const double gamma = __dadd_rn(wc, sigma * rho);
    double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
    if (rho == 0.0) { fail(st, SQB_ERR_BREAKDOWN, c + 1, 0.0); return; }
    if (!isfinite(beta)) { fail(st, SQB_ERR_BREAKDOWN, c + 1, rho); return; }
    double f;
    if (scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); beta = 1.0; }
    else { f = gamma; beta = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    sc->rho = rho; sc->sigma = sigma; sc->gamma = gamma; sc->beta = beta; sc->f = f; sc->wc = wc;
    R[c + (int64_t)c * ldr] = -sigma * rho;
    sigmas[c] = sigma; rhos[c] = rho; betas[c] = beta;
  }
}

// U[:, c] = scaled (0, .., 0, gamma, w[c+1:]) (baselines.py:68-78)
__global__ void __launch_bounds__(256)
hqrt_scale_kernel(double* __restrict__ uc, int64_t p, int c, int scaling, const HtScal* __restrict__ sc,
                  const Status* st) {
  if (failed(st)) return;
  const double f = sc->f, gamma = sc->gamma;
  const bool sq = scaling == SQB_SCALE_SQRT2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += (int64_t)gridDim.x * blockDim.x) {
    const double y = i < c ? 0.0 : (i == c ? gamma : uc[i]);
    uc[i] = sq ? __dmul_rn(y, f) : __ddiv_rn(y, f);
  }
}

// T[:c, c] = -beta T_c (sum_b P[b]), T[c, c] = beta (baselines.py:80-84)
__global__ void __launch_bounds__(256)
hqrt_tcol_kernel(const double* __restrict__ P, int nb, int ldp, double* T, int64_t ldt, int c,
                 const HtScal* __restrict__ sc, const Status* st) {
  extern __shared__ double e[];
  if (failed(st)) return;
  const double beta = sc->beta;
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += P[(int64_t)b * ldp + k];
    e[k] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) {
    double s = 0.0;
    for (int k = i; k < c; ++k) s = fma(T[i + (int64_t)k * ldt], e[k], s);
    T[i + (int64_t)c * ldt] = __dmul_rn(-beta, s);
  }
  if (threadIdx.x == 0) T[c + (int64_t)c * ldt] = beta;
}

int hqr_tall(sqb_ctx* ctx, int scaling, const double* A, int64_t lda, int64_t p, int64_t m, double* U, int64_t ldu,
             double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  if (m > 1024) return set_error(ctx, SQB_ERR_ARG, "householder_qr: m=%lld above 1024", (long long)m);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>((p + HT_ROWS - 1) / HT_ROWS, 2 * (int64_t)ctx->sm_count));
  const int ldp = (int)m;
  WsPlan plan;
  const size_t iP = plan.add(sizeof(double) * (size_t)nb * ldp);
  const size_t iPn = plan.add(sizeof(double) * nb);
  const size_t iC = plan.add(sizeof(double) * m);
  const size_t iS = plan.add(sizeof(HtScal));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* P = ws_ptr<double>(ctx, plan, iP);
  double* Pn = ws_ptr<double>(ctx, plan, iPn);
  double* coef = ws_ptr<double>(ctx, plan, iC);
  HtScal* sc = ws_ptr<HtScal>(ctx, plan, iS);
  Status* st = ctx->d_status;
  SQB_CUDA_TRY(cudaMemset2DAsync(T, ldt * sizeof(double), 0, m * sizeof(double), m, ctx->stream));
  SQB_CUDA_TRY(cudaMemset2DAsync(R, ldr * sizeof(double), 0, m * sizeof(double), m, ctx->stream));
  const size_t dsm_max = sizeof(double) * (GEMV_NT / 32 + 1) * m;
  allow_dyn_smem(hqrt_dots_kernel, (size_t)(std::max<size_t>(dsm_max, 48 << 10)));
  const unsigned gs = (unsigned)std::max<int64_t>(1, std::min<int64_t>((p + 255) / 256, 4 * (int64_t)ctx->sm_count));
  for (int c = 0; c < (int)m; ++c) {
    const size_t dsm = sizeof(double) * (GEMV_NT / 32 + 1) * std::max(c, 1);
    if (c > 0) {
      hqrt_dots_kernel<<<nb, GEMV_NT, dsm, ctx->stream>>>(U, ldu, p, c, A + (int64_t)c * lda, 0, P, ldp, st);
      SQB_TRY(check_launch(ctx, "hqrt_dots_kernel"));
      hqrt_coef_kernel<<<1, 256, sizeof(double) * c, ctx->stream>>>(P, nb, ldp, T, ldt, c, coef, st);
      SQB_TRY(check_launch(ctx, "hqrt_coef_kernel"));
    }
    hqrt_update_kernel<<<nb, GEMV_NT, sizeof(double) * std::max(c, 1), ctx->stream>>>(A, lda, U, ldu, p, c, coef, Pn,
                                                                                    st);
    SQB_TRY(check_launch(ctx, "hqrt_update_kernel"));
    hqrt_scalars_kernel<<<1, 256, 0, ctx->stream>>>(Pn, nb, U, ldu, c, scaling, R, ldr, sigmas, rhos, betas, sc, st);
    SQB_TRY(check_launch(ctx, "hqrt_scalars_kernel"));
    hqrt_scale_kernel<<<gs, 256, 0, ctx->stream>>>(U + (int64_t)c * ldu, p, c, scaling, sc, st);
    SQB_TRY(check_launch(ctx, "hqrt_scale_kernel"));
    if (c > 0) {
      hqrt_dots_kernel<<<nb, GEMV_NT, dsm, ctx->stream>>>(U, ldu, p, c, U + (int64_t)c * ldu, c, P, ldp, st);
      SQB_TRY(check_launch(ctx, "hqrt_dots_kernel"));
    }
    hqrt_tcol_kernel<<<1, 256, sizeof(double) * std::max(c, 1), ctx->stream>>>(P, nb, ldp, T, ldt, c, sc, st);
    SQB_TRY(check_launch(ctx, "hqrt_tcol_kernel"));
  }
  return SQB_OK;
}

}  // namespace sqb
