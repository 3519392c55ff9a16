// Trimmed RHQR, left-looking (trim.py:272-325).
//
// The operator is the column-scaled wrapper of a base sketch over all N
// coordinates (sketching.py:216-235): coordinates < m are multiplied by
// scales[k] in the arithmetic dtype before the base sketch.  Per column c
// (1-based j = c + 1):
//   c > 0:  z = Om(W[:, c])                 (all columns in one batched K1)
//           h = S^t z - L w[:c];  coef = T~^t h          (trim_coef_kernel)
//           w = fl(w - fl(U[:, :c] coef))                (streaming GEMV)
//   trim_rh_vector (trim.py:80-146):
//           z = Om([0; w[c:]]);  rho = ||z||;  v0 = fl(w[c] + sigma rho)
//           vs = Om([0; v0, w[c+1:]])           (the prepared input with one
//                                                entry replaced, K1 again)
//           beta = 2 / ||vs||^2, sqrt2 / unit scaling, breakdown checks
//   S[:, c] = vs;  R[:c, c] = w[:c];  R[c, c] = -sigma rho
//   L[c, :c] = E^t vs;  T column (_extend_t);  T~ column (trim.py:312-316)
//   U[:, c] = [0; v] * f  (or / piv)
// Sketch-space work runs in single-CTA kernels on the device; nothing returns
// to the host until the sweep ends.  Breakdowns set the device status with
// col = j | kind << 24 (kind 0: tail annihilated, 1: reflector cancelled,
// 2: unit pivot vanished), which the facade maps to the reference's messages.
#include <algorithm>

#include "sketch.cuh"
#include "vec.cuh"
#include "gemv.cuh"
#include "pdl.cuh"

namespace sqb {

int t_factor_impl(sqb_ctx*, const double*, int64_t, int64_t, int64_t, double*, int64_t);
int upper_tri_solve_impl(sqb_ctx*, const double*, int64_t, int64_t, const double*, int64_t, int64_t, double*, int64_t);

constexpr int TRIM_NT = 256;
constexpr int TRIM_SNT = 1024;  // single-CTA sketch-space kernels

// x = Xs of the column-scaled wrapper applied to [0 (c0 entries); w[c0:]]
template <typename T>
__global__ void trim_prep_kernel(T* __restrict__ x, const T* __restrict__ w, int64_t N, int64_t c0, int64_t m,
                                 const double* __restrict__ scales, const Status* st) {
  if (failed(st)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    T v;
    if (i < c0) v = Lo<T>::store(typename Lo<T>::acc(0));
    else if (i < m) v = Lo<T>::store(Lo<T>::mul(Lo<T>::load(w[i]), Lo<T>::from_double(scales[i])));
    else v = w[i];  // x * 1.0 is exact
    x[i] = v;
  }
}

// the column-scaled copy of W[:, 1:] (blockIdx.y = column - 1)
template <typename T>
__global__ void trim_prep_batch_kernel(T* __restrict__ X, int64_t ldx, const T* __restrict__ W, int64_t ldw,
                                       int64_t N, int64_t m, const double* __restrict__ scales, const Status* st) {
  if (failed(st)) return;
  T* x = X + blockIdx.y * ldx;
  const T* w = W + (blockIdx.y + 1) * ldw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = i < m ? Lo<T>::store(Lo<T>::mul(Lo<T>::load(w[i]), Lo<T>::from_double(scales[i]))) : w[i];
}

// h = S[:, :c]^t z - L[:c, :c] w[:c];  coef = T~[:c, :c]^t h   (trim.py:296-299)
// Sketch-space kernels run one CTA of TRIM_SNT threads with one warp per
// output and the lanes over the reduction index (coalesced, 32 loads in
// flight per warp): a thread-per-output loop was a chain of c dependent
// strided loads per column (ncu: 33 us per launch, the finish kernel 53 us)
template <typename T>
__global__ void __launch_bounds__(TRIM_SNT)
trim_coef_kernel(const double* __restrict__ S, int64_t lds, int ell, const double* __restrict__ z,
                 const double* __restrict__ L, int64_t ldl, const T* __restrict__ w, const double* __restrict__ Tt,
                 int64_t ldtt, int c, double* __restrict__ coef, const Status* st) {
  extern __shared__ double h[];  // [c]
  pdl_trigger();  // PDL: the next column kernel may be scheduled now
  pdl_wait();     // ... and this one reads its predecessor's output only after this
  if (failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = TRIM_SNT / 32;
  for (int k = warp; k < c; k += NW) {
    double d = 0.0;
    for (int i = lane; i < ell; i += 32) d = fma(S[i + k * lds], z[i], d);
    d = warp_sum(d);
    double e = 0.0;
    for (int i = lane; i < k; i += 32) e = fma(L[k + i * ldl], (double)Lo<T>::load(w[i]), e);
    e = warp_sum(e);
    if (lane == 0) h[k] = d - e;
  }
  __syncthreads();
  for (int i = warp; i < c; i += NW) {  // coef[i] = T~[:i+1, i] . h[:i+1]
    const double* ti = Tt + (int64_t)i * ldtt;
    double d = 0.0;
    for (int k = lane; k <= i; k += 32) d = fma(ti[k], h[k], d);
    d = warp_sum(d);
    if (lane == 0) coef[i] = d;
  }
}

// w = fl(W[:, c] - fl(U[:, :c] coef_lo)) over all N rows (trim.py:300; w = W[:, c]
// for c = 0), fused with the column-scaled input of the next K1:
// x = [0 (c entries); w[c:m] * scales; w[m:]] (trim_prep_kernel's map)
template <typename T>
__global__ void __launch_bounds__(GEMV_NT, 2)
trim_update_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int c, const double* __restrict__ coef,
                   const T* __restrict__ Wc, T* __restrict__ w, T* __restrict__ x, int64_t m,
                   const double* __restrict__ scales, const Status* st) {
  using A = typename Lo<T>::acc;
  constexpr int VN = VecN<T>::n, NV = 4;
  extern __shared__ unsigned char smraw[];
  A* cl = reinterpret_cast<A*>(smraw);
  pdl_trigger();  // PDL: the next column kernel may be scheduled now
  pdl_wait();     // ... and this one reads its predecessor's output only after this
  if (failed(st)) return;
  for (int k = threadIdx.x; k < c; k += blockDim.x) cl[k] = Lo<T>::from_double(coef[k]);
  __syncthreads();
  const int64_t rows_per = (int64_t)GEMV_NT * NV * VN;
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per; r0 < N; r0 += (int64_t)gridDim.x * rows_per) {
    A acc[NV][VN];
    gemv_rows<T, NV>(U, ldu, r0, N, c, cl, acc);
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < VN; ++j) {
        const int64_t i = r0 + (v * GEMV_NT + threadIdx.x) * VN + j;
        if (i < N) {
          const T wv = c > 0 ? Lo<T>::store(Lo<T>::sub(Lo<T>::load(Wc[i]), Lo<T>::rnd(acc[v][j]))) : Wc[i];
          w[i] = wv;
          T xv;
          if (i < c) xv = Lo<T>::store(A(0));
          else if (i < m) xv = Lo<T>::store(Lo<T>::mul(Lo<T>::load(wv), Lo<T>::from_double(scales[i])));
          else xv = wv;  // x * 1.0 is exact
          x[i] = xv;
        }
      }
  }
}

// fp64 block sum of squares (all threads get the result)
__device__ __forceinline__ double block_sumsq(const double* __restrict__ y, int n, double* red) {
  double d = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) d = fma(y[i], y[i], d);
  return block_sum(d, red);
}

// after z = Om([0; w[c:]]): rho, sigma, v0; replace entry c of the prepared
// input by the scaled v0 so the next K1 sketches [0; v] (trim.py:103-114)
template <typename T>
__global__ void __launch_bounds__(TRIM_NT)
trim_tail_kernel(const double* __restrict__ z, int ell, const T* __restrict__ w, int c,
                 const double* __restrict__ scales, T* __restrict__ x, double* __restrict__ scal, Status* st) {
  __shared__ double red[32];
  pdl_trigger();  // PDL: the next column kernel may be scheduled now
  pdl_wait();     // ... and this one reads its predecessor's output only after this
  if (failed(st)) return;
  const double zn = __dsqrt_rn(block_sumsq(z, ell, red));
  if (threadIdx.x == 0) {
    const double rho = zn;  // round_to(., high) is the identity for fp64
    if (rho == 0.0) {
      fail(st, SQB_ERR_BREAKDOWN, (c + 1), 0.0);
      return;
    }
    const double wc = (double)Lo<T>::load(w[c]);
    const double sg = wc >= 0.0 ? 1.0 : -1.0;
    const double v0 = (double)Lo<T>::from_double(__dadd_rn(wc, sg * rho));
    x[c] = Lo<T>::store(Lo<T>::mul(Lo<T>::from_double(v0), Lo<T>::from_double(scales[c])));
    scal[0] = sg;
    scal[1] = rho;
    scal[2] = zn;
    scal[3] = v0;
  }
}

// after vs = Om([0; v]): scaling, breakdown checks, and every sketch-space
// column of the step (trim.py:115-146, 304-316)
template <typename T>
__global__ void __launch_bounds__(TRIM_SNT)
trim_finish_kernel(double* __restrict__ vs, int ell, int c, int scaling, double u_high, const T* __restrict__ w,
                   const T* __restrict__ U, int64_t ldu, const double* __restrict__ E, int64_t lde,
                   double* __restrict__ S, int64_t lds, double* __restrict__ Tm, int64_t ldt,
                   double* __restrict__ Tt, int64_t ldtt, double* __restrict__ R, int64_t ldr,
                   double* __restrict__ L, int64_t ldl, double* __restrict__ sig, double* __restrict__ rho_out,
                   double* __restrict__ bet, double* __restrict__ scal, Status* st) {
  extern __shared__ double sh[];  // [c] S^t vs, [c] lrow, [c] g, [1] flag
  __shared__ double red[32];
  pdl_trigger();  // PDL: the next column kernel may be scheduled now
  pdl_wait();     // ... and this one reads its predecessor's output only after this
  if (failed(st)) return;
  double* sv = sh;
  double* lrow = sh + c;
  double* g = sh + 2 * c;
  const double sg = scal[0], rho = scal[1], zn = scal[2];
  const double nv = __dsqrt_rn(block_sumsq(vs, ell, red));
  if (nv <= 8.0 * u_high * (zn + rho)) {
    if (threadIdx.x == 0) fail(st, SQB_ERR_BREAKDOWN, (c + 1) | (1 << 24), nv);
    return;
  }
  double beta = __ddiv_rn(2.0, __dmul_rn(nv, nv));
  double fac;  // v = v * fac (sqrt2) or v / fac (unit)
  if (scaling == SQB_SCALE_SQRT2) {
    fac = __dsqrt_rn(beta);
    beta = 1.0;
  } else {
    const double piv = vs[0];
    if (fabs(piv) <= 8.0 * u_high * nv) {
      if (threadIdx.x == 0) fail(st, SQB_ERR_BREAKDOWN, (c + 1) | (2 << 24), piv);
      return;
    }
    fac = piv;
    beta = __dmul_rn(__dmul_rn(beta, piv), piv);
  }
  __syncthreads();  // every thread has read vs[0] before it is rescaled
  for (int i = threadIdx.x; i < ell; i += TRIM_SNT) {
    const double s = scaling == SQB_SCALE_SQRT2 ? __dmul_rn(vs[i], fac) : __ddiv_rn(vs[i], fac);
    vs[i] = s;
    S[i + (int64_t)c * lds] = s;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = TRIM_SNT / 32;
  for (int k = warp; k < c; k += NW) {
    double a = 0.0, b = 0.0;
    for (int i = lane; i < ell; i += 32) {
      a = fma(S[i + (int64_t)k * lds], vs[i], a);
      b = fma(E[i + (int64_t)k * lde], vs[i], b);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      sv[k] = a;
      lrow[k] = b;
      L[c + (int64_t)k * ldl] = b;
    }
  }
  __syncthreads();
  for (int k = warp; k < c; k += NW) {  // g = S^t vs - U[:c, :c]^t lrow
    const T* uk = U + (int64_t)k * ldu;
    double d = 0.0;
    for (int i = k + lane; i < c; i += 32) d = fma((double)Lo<T>::load(uk[i]), lrow[i], d);
    d = warp_sum(d);
    if (lane == 0) g[k] = sv[k] - d;
  }
  __syncthreads();
  for (int i = warp; i < c; i += NW) {  // T[i, c], T~[i, c]: row i of T, T~ against sv, g
    double t = 0.0, tt = 0.0;
    for (int k = i + lane; k < c; k += 32) {
      t = fma(Tm[i + (int64_t)k * ldt], sv[k], t);
      tt = fma(Tt[i + (int64_t)k * ldtt], g[k], tt);
    }
    t = warp_sum(t);
    tt = warp_sum(tt);
    if (lane == 0) {
      Tm[i + (int64_t)c * ldt] = __dmul_rn(-beta, t);
      Tt[i + (int64_t)c * ldtt] = __dmul_rn(-beta, tt);
      R[i + (int64_t)c * ldr] = (double)Lo<T>::load(w[i]);
    }
  }
  if (threadIdx.x == 0) {
    Tm[c + (int64_t)c * ldt] = beta;
    Tt[c + (int64_t)c * ldtt] = beta;
    R[c + (int64_t)c * ldr] = -sg * rho;
    sig[c] = sg;
    rho_out[c] = rho;
    bet[c] = beta;
    scal[4] = fac;
  }
}

// U[:, c] = [0; v0, w[c+1:]] scaled (trim.py:131-144, then round_to low)
template <typename T>
__global__ void trim_ucol_kernel(T* __restrict__ Uc, const T* __restrict__ w, int64_t N, int c, int scaling,
                                 const double* __restrict__ scal, const Status* st) {
  pdl_trigger();  // PDL: the next column kernel may be scheduled now
  pdl_wait();     // ... and this one reads its predecessor's output only after this
  if (failed(st)) return;
  const double fac = scal[4], v0 = scal[3];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < c) {
      Uc[i] = Lo<T>::store(typename Lo<T>::acc(0));
      continue;
    }
    const double v = i == c ? v0 : (double)Lo<T>::load(w[i]);
    const double u = scaling == SQB_SCALE_SQRT2 ? __dmul_rn(v, fac) : __ddiv_rn(v, fac);
    Uc[i] = Lo<T>::store(Lo<T>::from_double(u));
  }
}

template <typename T>
static int trim_left_t(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t ms, const double* E, int64_t lde,
                       int scaling, const void* W, int64_t N, int64_t m, int64_t ldw, void* Uv, int64_t ldu,
                       double* S, int64_t lds, double* Tm, int64_t ldt, double* Tt, int64_t ldtt, double* R,
                       int64_t ldr, double* L, int64_t ldl, double* sig, double* rho, double* bet) {
  const int64_t ell = sk->ell;
  const size_t esz = sizeof(T);
  const int64_t ldx = (N + 15) / 16 * 16;
  WsPlan plan;
  const size_t ix = plan.add(esz * ldx);
  const size_t iw = plan.add(esz * ldx);
  const size_t iz = plan.add(sizeof(double) * ell);
  const size_t iv = plan.add(sizeof(double) * ell);
  const size_t ic = plan.add(sizeof(double) * (m + 1));
  const size_t is = plan.add(sizeof(double) * 8);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, m));
  // the update sketches z_c = Om(W[:, c]) of the ORIGINAL columns do not
  // depend on the sweep: one batched K1 over the column-scaled W up front
  const size_t iXa = plan.add(esz * ldx * (m > 1 ? m - 1 : 1));
  const size_t iZ0 = plan.add(sizeof(double) * ell * m);
  SQB_TRY(ws_reserve(ctx, plan.total));
  T* x = ws_ptr<T>(ctx, plan, ix);
  T* w = ws_ptr<T>(ctx, plan, iw);
  T* Xa = ws_ptr<T>(ctx, plan, iXa);
  double* Z0 = ws_ptr<double>(ctx, plan, iZ0);
  double* z = ws_ptr<double>(ctx, plan, iz);
  double* vs = ws_ptr<double>(ctx, plan, iv);
  double* coef = ws_ptr<double>(ctx, plan, ic);
  double* scal = ws_ptr<double>(ctx, plan, is);
  void* P = ws_ptr<void>(ctx, plan, iP);
  T* U = static_cast<T*>(Uv);
  Status* st = ctx->d_status;
  cudaStream_t s = ctx->stream;
  for (double* M : {Tm, Tt, R, L}) {
    const int64_t ld = M == Tm ? ldt : M == Tt ? ldtt : M == R ? ldr : ldl;
    SQB_CUDA_TRY(cudaMemset2DAsync(M, ld * sizeof(double), 0, m * sizeof(double), m, s));
  }
  const unsigned gv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 4 * ctx->sm_count));
  const double u_high = 1.0 / 9007199254740992.0;  // 2^-53: the device path computes high in fp64
  const int64_t rows_per = (int64_t)GEMV_NT * 4 * VecN<T>::n;
  const unsigned gu = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + rows_per - 1) / rows_per,
                                                                       2 * ctx->sm_count));
  if (m > 1) {
    const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 2 * ctx->sm_count));
    trim_prep_batch_kernel<T><<<dim3(gb, (unsigned)(m - 1)), 256, 0, s>>>(Xa, ldx, (const T*)W, ldw, N, ms,
                                                                          scales, st);
    SQB_TRY(check_launch(ctx, "trim_prep_batch_kernel"));
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, Xa, ldx, m - 1, Z0 + ell, ell, 0, P, st));
  }
  for (int64_t c = 0; c < m; ++c) {
    if (c > 0) {  // w[:c] (read by the coefficient kernel) is W[:c, c]: the original column
      SQB_TRY(launch_pdl(ctx, "trim_coef_kernel", trim_coef_kernel<T>, dim3(1), dim3(TRIM_SNT), sizeof(double) * c,
                         (const double*)S, lds, (int)ell, (const double*)(Z0 + c * ell), (const double*)L, ldl,
                         (const T*)W + c * ldw, (const double*)Tt, ldtt, (int)c, coef, (const Status*)st));
    }
    SQB_TRY(launch_pdl(ctx, "trim_update_kernel", trim_update_kernel<T>, dim3(gu), dim3(GEMV_NT),
                       sizeof(typename Lo<T>::acc) * std::max<int64_t>(c, 1), (const T*)U, ldu, N, (int)c,
                       (const double*)coef, (const T*)W + c * ldw, w, x, ms, scales, (const Status*)st));
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, x, ldx, 1, z, ell, 0, P, st));
    SQB_TRY(launch_pdl(ctx, "trim_tail_kernel", trim_tail_kernel<T>, dim3(1), dim3(TRIM_NT), 0, (const double*)z,
                       (int)ell, (const T*)w, (int)c, scales, x, scal, st));
    // x differs from the z sketch's input only at entry c: re-sketch the head tile
    SQB_TRY(launch_sketch_resketch_head(ctx, sk, Lo<T>::code, x, ldx, c + 1, vs, ell, 0, P, st));
    SQB_TRY(launch_pdl(ctx, "trim_finish_kernel", trim_finish_kernel<T>, dim3(1), dim3(TRIM_SNT),
                       sizeof(double) * (3 * c + 1), vs, (int)ell, (int)c, scaling, u_high, (const T*)w,
                       (const T*)U, ldu, E, lde, S, lds, Tm, ldt, Tt, ldtt, R, ldr, L, ldl, sig, rho, bet, scal, st));
    SQB_TRY(launch_pdl(ctx, "trim_ucol_kernel", trim_ucol_kernel<T>, dim3(gv), dim3(256), 0, U + c * ldu,
                       (const T*)w, N, (int)c, scaling, (const double*)scal, (const Status*)st));
  }
  return SQB_OK;
}

// ---------------------------------------------------------------------------
// the column-scaled operator alone (sketching.py:230-235) and the trimmed
// thin Q (trim.py:211-225)
// ---------------------------------------------------------------------------
template <typename T>
static int colscaled_apply_t(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t m, const void* X,
                             int64_t ldx, int64_t k, double* Y, int64_t ldy) {
  const int64_t N = sk->n, ldp = (N + 15) / 16 * 16;
  WsPlan plan;
  const size_t ix = plan.add(sizeof(T) * ldp);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, 1));
  SQB_TRY(ws_reserve(ctx, plan.total));
  T* x = ws_ptr<T>(ctx, plan, ix);
  void* P = ws_ptr<void>(ctx, plan, iP);
  const unsigned gv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 4 * ctx->sm_count));
  for (int64_t j = 0; j < k; ++j) {
    trim_prep_kernel<T><<<gv, 256, 0, ctx->stream>>>(x, (const T*)X + j * ldx, N, 0, m, scales, ctx->d_status);
    SQB_TRY(check_launch(ctx, "trim_prep_kernel"));
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, x, ldp, 1, Y + j * ldy, ldy, 0, P, ctx->d_status));
  }
  return SQB_OK;
}

int colscaled_apply_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t m, int dtype,
                             const void* X, int64_t ldx, int64_t k, double* Y, int64_t ldy) {
  switch (dtype) {
    case SQB_F64: return colscaled_apply_t<double>(ctx, sk, scales, m, X, ldx, k, Y, ldy);
    case SQB_F32: return colscaled_apply_t<float>(ctx, sk, scales, m, X, ldx, k, Y, ldy);
    case SQB_F16: return colscaled_apply_t<__half>(ctx, sk, scales, m, X, ldx, k, Y, ldy);
    case SQB_BF16: return colscaled_apply_t<__nv_bfloat16>(ctx, sk, scales, m, X, ldx, k, Y, ldy);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", dtype);
}

// G = triu(S^t E) (k x k, ld k), then M = T G (T upper, so M[i, j] = sum_{i <= l <= j} T[i, l] G[l, j]).
// One thread per entry with the sums in index order; G lives in the workspace (k is not bounded by
// shared memory: the acceptance runs of the reference use k = 300).
__global__ void trim_g_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ E, int64_t lde,
                              int ell, int k, double* __restrict__ G) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(e % k), j = (int)(e / k);
    double d = 0.0;
    if (l <= j)
      for (int i = 0; i < ell; ++i) d = fma(S[i + (int64_t)l * lds], E[i + (int64_t)j * lde], d);
    G[e] = d;
  }
}

__global__ void trim_tm_kernel(const double* __restrict__ Tm, int64_t ldt, const double* __restrict__ G, int k,
                               double* __restrict__ M) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)k * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e % k), j = (int)(e / k);
    double d = 0.0;
    for (int l = i; l <= j; ++l) d = fma(Tm[i + (int64_t)l * ldt], G[l + (int64_t)j * k], d);
    M[e] = d;
  }
}

int thin_q_m_dispatch(sqb_ctx*, int, const void*, int64_t, int64_t, int64_t, const double*, double*, int64_t);

int trim_thin_q_impl(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
                     const double* Tm, int64_t ldt, const double* S, int64_t lds, const double* E, int64_t lde,
                     int64_t ell, double* Q, int64_t ldq) {
  WsPlan plan;
  const size_t iM = plan.add(sizeof(double) * std::max<int64_t>(1, k * k));
  const size_t iG = plan.add(sizeof(double) * std::max<int64_t>(1, k * k));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* M = ws_ptr<double>(ctx, plan, iM);
  double* G = ws_ptr<double>(ctx, plan, iG);
  const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((k * k + 255) / 256, 4 * ctx->sm_count));
  trim_g_kernel<<<gb, 256, 0, ctx->stream>>>(S, lds, E, lde, (int)ell, (int)k, G);
  SQB_TRY(check_launch(ctx, "trim_g_kernel"));
  trim_tm_kernel<<<gb, 256, 0, ctx->stream>>>(Tm, ldt, G, (int)k, M);
  SQB_TRY(check_launch(ctx, "trim_tm_kernel"));
  return thin_q_m_dispatch(ctx, lo_dtype, U, ldu, N, k, M, Q, ldq);
}

// ---------------------------------------------------------------------------
// Right-looking trimmed RHQR (trim.py:238-269): per column the reflector of
// the tail (same kernels as the left sweep), then the trailing columns are
// updated through the masked sketch; T, T~ and L are assembled from S, E and
// U after the sweep (t_factor_from_sketches, t_tilde_from_factors).
// ---------------------------------------------------------------------------
// X[:, j] = column-scaled copy of Y[:, j] with rows < c0 zeroed (trim.py:256-258)
template <typename T>
__global__ void trim_mask_batch_kernel(T* __restrict__ X, int64_t ldx, const T* __restrict__ Y, int64_t ldy,
                                       int64_t N, int64_t c0, int64_t m, const double* __restrict__ scales,
                                       const Status* st) {
  if (failed(st)) return;
  T* x = X + blockIdx.y * ldx;
  const T* y = Y + blockIdx.y * ldy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = i < c0 ? Lo<T>::store(typename Lo<T>::acc(0))
                  : (i < m ? Lo<T>::store(Lo<T>::mul(Lo<T>::load(y[i]), Lo<T>::from_double(scales[i]))) : y[i]);
}

// coef[j] = beta (s^t X[:, j]) in fp64 (trim.py:260)
__global__ void trim_rcoef_kernel(const double* __restrict__ s, const double* __restrict__ Xs, int64_t ldx, int ell,
                                  const double* __restrict__ bet, int c, double* __restrict__ coef, const Status* st) {
  __shared__ double red[32];
  if (failed(st)) return;
  const int j = blockIdx.x;
  double d = 0.0;
  for (int i = threadIdx.x; i < ell; i += blockDim.x) d = fma(s[i], Xs[i + (int64_t)j * ldx], d);
  d = block_sum(d, red);
  if (threadIdx.x == 0) coef[j] = __dmul_rn(bet[c], d);
}

// Y[:, j] = fl(Y[:, j] - fl(u coef_lo[j]))  (trim.py:261-263: np.outer, then subtract)
template <typename T>
__global__ void trim_rank1_kernel(const T* __restrict__ u, const double* __restrict__ coef, T* __restrict__ Y,
                                  int64_t ldy, int64_t N, const Status* st) {
  using A = typename Lo<T>::acc;
  if (failed(st)) return;
  const A cj = Lo<T>::from_double(coef[blockIdx.y]);
  T* y = Y + blockIdx.y * ldy;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = Lo<T>::store(Lo<T>::sub(Lo<T>::load(y[i]), Lo<T>::mul(Lo<T>::load(u[i]), cj)));
}

// A^t (for T~^t = -A^{-1}, trim.py:189-208), the identity, and L = tril(S^t E, -1)
template <typename T>
__global__ void trim_tilde_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ E,
                                  int64_t lde, int ell, const T* __restrict__ U, int64_t ldu, int m,
                                  double* __restrict__ At, double* __restrict__ I, double* __restrict__ L,
                                  int64_t ldl, double* __restrict__ Lt) {
  // Lt[i, k] = <s_i, e_k> for k < i (scratch m x m, also written to L)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
    const int i = e % m, k = e / m;
    double d = 0.0;
    if (k < i)
      for (int r = 0; r < ell; ++r) d = fma(S[r + (int64_t)i * lds], E[r + (int64_t)k * lde], d);
    Lt[e] = d;
    L[i + (int64_t)k * ldl] = d;
  }
  __syncthreads();
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x) {
    const int i = e % m, k = e / m;
    double corr = 0.0;  // (Lt U[:m])[i, k] = sum_{k <= l < i} Lt[i, l] U[l, k]
    for (int l = k; l < i; ++l) corr = fma(Lt[i + l * m], (double)Lo<T>::load(U[l + (int64_t)k * ldu]), corr);
    double g = 0.0;
    if (k <= i)
      for (int r = 0; r < ell; ++r) g = fma(S[r + (int64_t)i * lds], S[r + (int64_t)k * lds], g);
    double a = corr;
    if (k < i) a = __dsub_rn(a, g);
    else if (k == i) a = __dsub_rn(a, g / 2.0);
    At[k + (int64_t)i * m] = a;  // A^t[k, i] = A[i, k]
    I[e] = i == k ? 1.0 : 0.0;
  }
}

__global__ void trim_negate_kernel(const double* __restrict__ X, int m, double* __restrict__ Tt, int64_t ldtt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x)
    Tt[e % m + (int64_t)(e / m) * ldtt] = -X[e];
}

template <typename T>
static int trim_right_t(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t ms, const double* E, int64_t lde,
                        int scaling, const void* W, int64_t N, int64_t m, int64_t ldw, void* Uv, int64_t ldu,
                        double* S, int64_t lds, double* Tm, int64_t ldt, double* Tt, int64_t ldtt, double* R,
                        int64_t ldr, double* L, int64_t ldl, double* sig, double* rho, double* bet) {
  const int64_t ell = sk->ell;
  const size_t esz = sizeof(T);
  const int64_t ldx = (N + 15) / 16 * 16;
  T* U = static_cast<T*>(Uv);
  cudaStream_t s = ctx->stream;
  Status* st = ctx->d_status;
  {
    WsPlan plan;
    const size_t iWl = plan.add(esz * ldx * m);                       // working copy of W
    const size_t iXm = plan.add(esz * ldx * (m > 1 ? m - 1 : 1));     // masked, scaled trailing block
    const size_t ix = plan.add(esz * ldx);
    const size_t iz = plan.add(sizeof(double) * ell);
    const size_t iv = plan.add(sizeof(double) * ell);
    const size_t iY = plan.add(sizeof(double) * ell * m);
    const size_t ic = plan.add(sizeof(double) * (m + 1));
    const size_t is = plan.add(sizeof(double) * 8);
    const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, m));
    SQB_TRY(ws_reserve(ctx, plan.total));
    T* Wl = ws_ptr<T>(ctx, plan, iWl);
    T* Xm = ws_ptr<T>(ctx, plan, iXm);
    T* x = ws_ptr<T>(ctx, plan, ix);
    double* z = ws_ptr<double>(ctx, plan, iz);
    double* vs = ws_ptr<double>(ctx, plan, iv);
    double* Yx = ws_ptr<double>(ctx, plan, iY);
    double* coef = ws_ptr<double>(ctx, plan, ic);
    double* scal = ws_ptr<double>(ctx, plan, is);
    void* P = ws_ptr<void>(ctx, plan, iP);
    SQB_CUDA_TRY(cudaMemcpy2DAsync(Wl, ldx * esz, W, ldw * esz, N * esz, m, cudaMemcpyDeviceToDevice, s));
    for (double* M : {Tm, Tt, R, L}) {
      const int64_t ld = M == Tm ? ldt : M == Tt ? ldtt : M == R ? ldr : ldl;
      SQB_CUDA_TRY(cudaMemset2DAsync(M, ld * sizeof(double), 0, m * sizeof(double), m, s));
    }
    const unsigned gv = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 4 * ctx->sm_count));
    const double u_high = 1.0 / 9007199254740992.0;
    for (int64_t c = 0; c < m; ++c) {
      T* w = Wl + c * ldx;
      trim_prep_kernel<T><<<gv, 256, 0, s>>>(x, w, N, c, ms, scales, st);
      SQB_TRY(check_launch(ctx, "trim_prep_kernel"));
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, x, ldx, 1, z, ell, 0, P, st));
      trim_tail_kernel<T><<<1, TRIM_NT, 0, s>>>(z, (int)ell, w, (int)c, scales, x, scal, st);
      SQB_TRY(check_launch(ctx, "trim_tail_kernel"));
      // x differs from the z sketch's input only at entry c: re-sketch the head tile
      SQB_TRY(launch_sketch_resketch_head(ctx, sk, Lo<T>::code, x, ldx, c + 1, vs, ell, 0, P, st));
      // the left sweep's finish kernel also grows T, T~ and L; the right
      // variant overwrites them below with the reference's assembled forms
      trim_finish_kernel<T><<<1, TRIM_SNT, sizeof(double) * (3 * c + 1), s>>>(
          vs, (int)ell, (int)c, scaling, u_high, w, U, ldu, E, lde, S, lds, Tm, ldt, Tt, ldtt, R, ldr, L, ldl, sig,
          rho, bet, scal, st);
      SQB_TRY(check_launch(ctx, "trim_finish_kernel"));
      trim_ucol_kernel<T><<<gv, 256, 0, s>>>(U + c * ldu, w, N, (int)c, scaling, scal, st);
      SQB_TRY(check_launch(ctx, "trim_ucol_kernel"));
      const int64_t k = m - c - 1;
      if (k > 0) {
        const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 2 * ctx->sm_count));
        trim_mask_batch_kernel<T><<<dim3(gb, (unsigned)k), 256, 0, s>>>(Xm, ldx, w + ldx, ldx, N, c, ms, scales, st);
        SQB_TRY(check_launch(ctx, "trim_mask_batch_kernel"));
        SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, Xm, ldx, k, Yx, ell, 0, P, st));
        trim_rcoef_kernel<<<(unsigned)k, 256, 0, s>>>(S + c * lds, Yx, ell, (int)ell, bet, (int)c, coef, st);
        SQB_TRY(check_launch(ctx, "trim_rcoef_kernel"));
        trim_rank1_kernel<T><<<dim3(gb, (unsigned)k), 256, 0, s>>>(U + c * ldu, coef, w + ldx, ldx, N, st);
        SQB_TRY(check_launch(ctx, "trim_rank1_kernel"));
      }
    }
  }
  // T = t_factor_from_sketches(S) (rhqr.py:122-132); may reuse the workspace
  SQB_TRY(t_factor_impl(ctx, S, lds, ell, m, Tm, ldt));
  WsPlan plan;
  const size_t iA = plan.add(sizeof(double) * m * m);
  const size_t iI = plan.add(sizeof(double) * m * m);
  const size_t iX = plan.add(sizeof(double) * m * m);
  const size_t iL = plan.add(sizeof(double) * m * m);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* At = ws_ptr<double>(ctx, plan, iA);
  double* I = ws_ptr<double>(ctx, plan, iI);
  double* X = ws_ptr<double>(ctx, plan, iX);
  double* Lt = ws_ptr<double>(ctx, plan, iL);
  trim_tilde_kernel<T><<<1, 256, 0, s>>>(S, lds, E, lde, (int)ell, U, ldu, (int)m, At, I, L, ldl, Lt);
  SQB_TRY(check_launch(ctx, "trim_tilde_kernel"));
  SQB_TRY(upper_tri_solve_impl(ctx, At, m, m, I, m, m, X, m));
  trim_negate_kernel<<<(unsigned)std::max<int64_t>(1, (m * m + 255) / 256), 256, 0, s>>>(X, (int)m, Tt, ldtt);
  return check_launch(ctx, "trim_negate_kernel");
}

int trim_right_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t ms, const double* E, int64_t lde,
                        int scaling, int lo_dtype, const void* W, int64_t N, int64_t m, int64_t ldw, void* U,
                        int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt, double* Tt, int64_t ldtt,
                        double* R, int64_t ldr, double* L, int64_t ldl, double* sig, double* rho, double* bet) {
#define SQB_TRIM_CALL(TY)                                                                                       \
  return trim_right_t<TY>(ctx, sk, scales, ms, E, lde, scaling, W, N, m, ldw, U, ldu, S, lds, Tm, ldt, Tt, ldtt, R, \
                          ldr, L, ldl, sig, rho, bet)
  switch (lo_dtype) {
    case SQB_F64: SQB_TRIM_CALL(double);
    case SQB_F32: SQB_TRIM_CALL(float);
    case SQB_F16: SQB_TRIM_CALL(__half);
    case SQB_BF16: SQB_TRIM_CALL(__nv_bfloat16);
  }
#undef SQB_TRIM_CALL
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

int trim_left_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t ms, const double* E, int64_t lde,
                       int scaling, int lo_dtype, const void* W, int64_t N, int64_t m, int64_t ldw, void* U,
                       int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt, double* Tt, int64_t ldtt,
                       double* R, int64_t ldr, double* L, int64_t ldl, double* sig, double* rho, double* bet) {
#define SQB_TRIM_CALL(TY)                                                                                      \
  return trim_left_t<TY>(ctx, sk, scales, ms, E, lde, scaling, W, N, m, ldw, U, ldu, S, lds, Tm, ldt, Tt, ldtt, R, \
                         ldr, L, ldl, sig, rho, bet)
  switch (lo_dtype) {
    case SQB_F64: SQB_TRIM_CALL(double);
    case SQB_F32: SQB_TRIM_CALL(float);
    case SQB_F16: SQB_TRIM_CALL(__half);
    case SQB_BF16: SQB_TRIM_CALL(__nv_bfloat16);
  }
#undef SQB_TRIM_CALL
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb
