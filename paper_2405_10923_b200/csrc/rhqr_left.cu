// Left-looking randomized Householder QR on the device (rhqr_left, rhqr.py:254-267;
// the hot loop _left_sweep, rhqr.py:219-251).
//
// Per column c:
//   K3+K1  rhqr_col_kernel  one HBM pass over rows >= m: lazily scale column
//          c-1 (u = fl(w * f)), w_c = fl(W[:,c] - fl(U[:, :c] coef)), store
//          w_c (unscaled) into U[:, c], and emit the in-tile SRHT leaves of
//          w_c.  An extra CTA does the m-row identity block.
//   tree   srht_tree_kernel      y[m:] = Omega w_c (bit-exact tree)
//   K4     rhqr_step_kernel      rh_vector (rhqr.py:51-97) on y, S/T/R column
//          (_extend_t :135-140), the next column's coefficients
//          T^t (S^t y0_{c+1}) (:241) — all fp64 in one CTA, no host trip.
// The raw sketches y0 = Psi W[:, c] of all columns are computed once up front
// (bitwise equal to the per-column psi.apply(w)).
#include <algorithm>

#include "sketch.cuh"
#include "vec.cuh"

namespace sqb {

constexpr int COL_NT = 256;
constexpr int STEP_NT = 512;

struct ColArgs {
  int c;            // current column (>= 1)
  int m;            // identity-block rows = columns of W
  int64_t n;        // Omega input length (N - m)
  int ell;
  int log_tb;
  int64_t n_tiles;
  int64_t n_eff;
  const void* W;    // column-major, ldw
  int64_t ldw;
  void* U;          // column-major, ldu
  int64_t ldu;
  const double* coef;   // [c] fp64 coefficients T^t S^t y0 (rhqr.py:241)
  const double* fscale; // [1] f (sqrt2) or gamma (unit) of column c-1
  int scaling;
  int srht;             // emit SRHT leaves (else the sketch runs separately)
  const uint32_t* bits;
  const int64_t* idx;
  double scale_lo;
  void* P;              // leaves [ell][n_tiles] (acc type)
  double* y;            // (m + ell) sketch of w_c; [0, m) written here
  const Status* st;
};

template <typename T>
__device__ __forceinline__ typename Lo<T>::acc lazy_scale(typename Lo<T>::acc w, double f, int scaling) {
  // rhqr.py:86-95 then round_to(u, low): u = fl64(w * f) or fl64(w / gamma)
  const double u = scaling == SQB_SCALE_SQRT2 ? __dmul_rn((double)w, f) : __ddiv_rn((double)w, f);
  return Lo<T>::from_double(u);
}

// identity block: y[r] = w_c[r] = fl(W[r,c] - fl(sum_k U[r,k] coef[k])), r < m
template <typename T>
__device__ void col_top_block(const ColArgs& a, const typename Lo<T>::acc* sc) {
  using A = typename Lo<T>::acc;
  const T* W = (const T*)a.W;
  const T* U = (const T*)a.U;
  for (int r = threadIdx.x; r < a.m; r += blockDim.x) {
    A acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    int k = 0;
    for (; k + 4 <= a.c; k += 4) {
      acc0 = fma(Lo<T>::load(U[r + (int64_t)k * a.ldu]), sc[k], acc0);
      acc1 = fma(Lo<T>::load(U[r + (int64_t)(k + 1) * a.ldu]), sc[k + 1], acc1);
      acc2 = fma(Lo<T>::load(U[r + (int64_t)(k + 2) * a.ldu]), sc[k + 2], acc2);
      acc3 = fma(Lo<T>::load(U[r + (int64_t)(k + 3) * a.ldu]), sc[k + 3], acc3);
    }
    for (; k < a.c; ++k) acc0 = fma(Lo<T>::load(U[r + (int64_t)k * a.ldu]), sc[k], acc0);
    const A dot = (acc0 + acc1) + (acc2 + acc3);
    const A w = Lo<T>::sub(Lo<T>::load(W[r + (int64_t)a.c * a.ldw]), Lo<T>::rnd(dot));
    a.y[r] = (double)w;
  }
}

template <typename T, int VN>
__global__ void __launch_bounds__(COL_NT, 2) rhqr_col_kernel(ColArgs a) {
  using A = typename Lo<T>::acc;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* sc = reinterpret_cast<A*>(smem_raw);                      // coef rounded to low [c]
  A* sm = sc + ((a.c + 3) & ~3);                              // tile buffer
  if (failed(a.st)) return;
  const int c = a.c;
  for (int k = threadIdx.x; k < c; k += COL_NT) sc[k] = Lo<T>::from_double(a.coef[k]);
  __syncthreads();
  if (blockIdx.x == a.n_eff) {
    col_top_block<T>(a, sc);
    return;
  }
  constexpr int TB = 1 << TileCfg<T>::LOG_TB;
  constexpr int NV = TB / (COL_NT * VN);  // runs of VN rows per thread
  const int tb = 1 << a.log_tb;
  const int64_t e0 = (int64_t)blockIdx.x << a.log_tb;  // first Omega coordinate of the tile
  const int64_t lim = a.n - e0;                       // valid rows in this tile (may exceed tb)
  const int64_t rows = lim < tb ? lim : tb;
  const int64_t ro = (int64_t)a.m + e0;                // first row of the tile in W / U
  T* U = (T*)a.U;
  const T* W = (const T*)a.W;

  A acc[NV][VN];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < VN; ++j) acc[v][j] = A(0);

  // final columns 0 .. c-2
  for (int k = 0; k < c - 1; ++k) {
    const T* col = U + ro + (int64_t)k * a.ldu;
    const A ck = sc[k];
    A v0[NV][VN];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if (i < tb) load_run<T, VN>(col, i, rows, v0[v]);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int j = 0; j < VN; ++j) acc[v][j] = fma(v0[v][j], ck, acc[v][j]);
  }
  // column c-1: lazy scaling of the stored w_{c-1}, write back u_{c-1}
  {
    const T* src = (c == 1 ? W : (const T*)U) + ro + (int64_t)(c - 1) * (c == 1 ? 0 : a.ldu);
    T* dst = U + ro + (int64_t)(c - 1) * a.ldu;
    const double f = *a.fscale;
    const A ck = sc[c - 1];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if (i < tb) {
        A x[VN];
        load_run<T, VN>(src, i, rows, x);
#pragma unroll
        for (int j = 0; j < VN; ++j) {
          x[j] = lazy_scale<T>(x[j], f, a.scaling);
          acc[v][j] = fma(x[j], ck, acc[v][j]);
        }
        store_run<T, VN>(dst, i, rows, x);
      }
    }
  }
  // w_c = fl(W[:, c] - fl(dot)); store unscaled into U[:, c]; SRHT input to smem
  {
    const T* wc = W + ro + (int64_t)c * a.ldw;
    T* uc = U + ro + (int64_t)c * a.ldu;
    const A s_lo = (A)a.scale_lo;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if (i < tb) {
        A x[VN];
        load_run<T, VN>(wc, i, rows, x);
#pragma unroll
        for (int j = 0; j < VN; ++j) x[j] = Lo<T>::sub(x[j], Lo<T>::rnd(acc[v][j]));
        store_run<T, VN>(uc, i, rows, x);
        if (a.srht) {
          const int64_t e = e0 + i;
          const uint32_t sb = __ldg(a.bits + (e >> 5)) >> (e & 31);
#pragma unroll
          for (int j = 0; j < VN; ++j)
            sm[pidx<A>(i + j)] = (i + j < rows) ? srht_in<T>(x[j], s_lo, (sb >> j) & 1u) : A(0);
        }
      }
    }
  }
  if (!a.srht) return;
  __syncthreads();
  tile_fwht<T>(sm, a.log_tb);
  tile_gather<T>(sm, a.idx, a.ell, a.log_tb, (A*)a.P + blockIdx.x, a.n_tiles);
}

// ---------------------------------------------------------------------------
// K4: one CTA, fp64 sketch-space step for column c (rhqr.py:51-97, 135-140,
// 241, 245-250)
// ---------------------------------------------------------------------------
struct StepArgs {
  int c, m, ell, od;          // od = m + ell (Psi output dim)
  int scaling;
  const double* y;            // sketch of w_c (od)
  const double* Y0;           // raw sketches (od x m, ld od)
  double* S; int64_t lds;
  double* T; int64_t ldt;
  double* R; int64_t ldr;
  void* U; int64_t ldu;       // identity-block rows of U[:, c] are written here
  double* sigmas; double* rhos; double* betas;
  double* coef_next;          // [c+1]
  double* fscale;             // [1]
  Status* st;
};

template <typename T>
__global__ void __launch_bounds__(STEP_NT) rhqr_step_kernel(StepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* s = reinterpret_cast<double*>(smem_raw);  // [od] new reflector sketch
  double* v = s + a.od;                            // [m] S^t s, then S^t y0
  double* red = v + a.m;                           // [32]
  __shared__ double sh_scal[4];
  if (failed(a.st)) return;
  const int c = a.c, od = a.od, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarp = STEP_NT / 32;
  // rho = ||y[c:]||_2 (rhqr.py:72)
  double part = 0.0;
  for (int r = c + tid; r < od; r += STEP_NT) part = fma(a.y[r], a.y[r], part);
  const double rho = sqrt(block_sum(part, red));
  if (tid == 0) {
    const double yc = a.y[c];
    const double sigma = yc >= 0.0 ? 1.0 : -1.0;                       // linalg.py:200-202
    const double gamma = __dadd_rn(yc, sigma * rho);                     // rhqr.py:76
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));  // :77
    int bad = 0;
    if (rho == 0.0) { fail(a.st, SQB_ERR_BREAKDOWN, c + 1, 0.0); bad = 1; }
    else if (!isfinite(beta)) { fail(a.st, SQB_ERR_BREAKDOWN, c + 1, rho); bad = 1; }
    double f, beta_out;
    if (a.scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); beta_out = 1.0; }
    else { f = gamma; beta_out = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    sh_scal[0] = sigma; sh_scal[1] = gamma; sh_scal[2] = f; sh_scal[3] = bad ? -1.0 : beta_out;
    a.sigmas[c] = sigma; a.rhos[c] = rho; a.betas[c] = beta_out;
    *a.fscale = f;
  }
  __syncthreads();
  const double sigma = sh_scal[0], gamma = sh_scal[1], f = sh_scal[2], beta_out = sh_scal[3];
  if (beta_out < 0.0) return;  // breakdown recorded
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  // s = Psi u (rhqr.py:83-96); u's identity-block rows; R column (:248-249)
  T* U = (T*)a.U;
  for (int r = tid; r < od; r += STEP_NT) {
    const double yh = r < c ? 0.0 : (r == c ? gamma : a.y[r]);
    const double sv = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s[r] = sv;
    a.S[r + (int64_t)c * a.lds] = sv;
    if (r < a.m) {
      U[r + (int64_t)c * a.ldu] = Lo<T>::store(Lo<T>::from_double(sv));
      a.R[r + (int64_t)c * a.ldr] = r < c ? a.y[r] : (r == c ? -sigma * rho : 0.0);
    }
  }
  __syncthreads();
  // v = S[:, :c]^t s  (warp per column, rows strided by lane)
  for (int k = warp; k < c; k += nwarp) {
    const double* sk = a.S + (int64_t)k * a.lds;
    double d = 0.0;
    for (int r = k + lane; r < od; r += 32) d = fma(sk[r], s[r], d);  // S[r,k] = 0 for r < k
    d = warp_sum(d);
    if (lane == 0) v[k] = d;
  }
  __syncthreads();
  // T[:c, c] = -beta * T[:c,:c] v ; T[c,c] = beta  (rhqr.py:135-140)
  for (int i = tid; i < c; i += STEP_NT) {
    double d = 0.0;
    for (int k = i; k < c; ++k) d = fma(a.T[i + (int64_t)k * a.ldt], v[k], d);
    a.T[i + (int64_t)c * a.ldt] = __dmul_rn(-beta_out, d);
  }
  if (tid == 0) a.T[c + (int64_t)c * a.ldt] = beta_out;
  if (c + 1 >= a.m) return;
  __syncthreads();
  // next coefficients: g = S[:, :c+1]^t y0_{c+1}; coef = T[:c+1,:c+1]^t g (rhqr.py:241)
  const double* y0 = a.Y0 + (int64_t)(c + 1) * od;
  for (int k = warp; k <= c; k += nwarp) {
    const double* sk = a.S + (int64_t)k * a.lds;
    double d = 0.0;
    for (int r = k + lane; r < od; r += 32) d = fma(k == c ? s[r] : sk[r], y0[r], d);
    d = warp_sum(d);
    if (lane == 0) v[k] = d;
  }
  __syncthreads();
  for (int k = warp; k <= c; k += nwarp) {
    const double* tk = a.T + (int64_t)k * a.ldt;  // column k of T, rows 0..k
    double d = 0.0;
    for (int i = lane; i <= k; i += 32) d = fma(tk[i], v[i], d);
    d = warp_sum(d);
    if (lane == 0) a.coef_next[k] = d;
  }
}

// final pass: U[m:, m-1] = scaled(w_{m-1}) (the lazy scaling of the last column)
template <typename T>
__global__ void scale_last_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t n,
                                  const double* fscale, int scaling, const Status* st) {
  if (failed(st)) return;
  const double f = *fscale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = Lo<T>::store(lazy_scale<T>(Lo<T>::load(src[i]), f, scaling));
}

__global__ void zero_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x)
    p[(e % rows) + (e / rows) * ld] = 0.0;
}

static int zero2d(sqb_ctx* ctx, double* p, int64_t rows, int64_t cols, int64_t ld) {
  if (rows * cols == 0) return SQB_OK;
  const unsigned g = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, 2048);
  zero_kernel<<<g, 256, 0, ctx->stream>>>(p, rows, cols, ld);
  return check_launch(ctx, "zero_kernel");
}

// ---------------------------------------------------------------------------
// driver
// ---------------------------------------------------------------------------
template <typename T>
static int rhqr_left_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N,
                       int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                       double* Tm, int64_t ldt, double* R, int64_t ldr, double* sigmas,
                       double* rhos, double* betas) {
  using A = typename Lo<T>::acc;
  const int64_t n = N - m, ell = sk->ell, od = m + ell;
  const bool srht = sk->kind == SQB_SKETCH_SRHT;
  const SrhtGeom g = srht ? srht_geom_t<T>(sk) : SrhtGeom{0, 1, 1};
  // workspace: raw sketches, column sketch, coefficients, scale, leaves
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(m, (int64_t)(64ll << 20) /
                                   std::max<size_t>(1, sketch_partials_bytes(sk, Lo<T>::code, 1))));
  WsPlan plan;
  const size_t iY0 = plan.add(sizeof(double) * od * m);
  const size_t iy = plan.add(sizeof(double) * od);
  const size_t icoef = plan.add(sizeof(double) * (m + 1));
  const size_t ifs = plan.add(sizeof(double) * 2);
  const size_t iP = plan.add(std::max(sketch_partials_bytes(sk, Lo<T>::code, chunk),
                                      sketch_partials_bytes(sk, Lo<T>::code, 1)));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* Y0 = ws_ptr<double>(ctx, plan, iY0);
  double* y = ws_ptr<double>(ctx, plan, iy);
  double* coef = ws_ptr<double>(ctx, plan, icoef);
  double* fs = ws_ptr<double>(ctx, plan, ifs);
  void* P = ws_ptr<void>(ctx, plan, iP);
  Status* st = ctx->d_status;

  SQB_TRY(zero2d(ctx, S, od, m, lds));
  SQB_TRY(zero2d(ctx, Tm, m, m, ldt));
  SQB_TRY(zero2d(ctx, R, m, m, ldr));
  // raw sketches y0 = Psi W (all columns; rhqr.py:240 for every column)
  SQB_TRY(launch_copy_top(ctx, Lo<T>::code, W, ldw, m, m, Y0, od, st));
  const size_t esz = sizeof(T);
  for (int64_t c0 = 0; c0 < m; c0 += chunk) {
    const int64_t kc = std::min(chunk, m - c0);
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)W + (c0 * ldw + m) * esz, ldw, kc,
                          Y0 + c0 * od, od, m, P, st));
  }
  // column 0: y = y0_0, w = W[:, 0]
  StepArgs sa{0, (int)m, (int)ell, (int)od, scaling, Y0, Y0, S, lds, Tm, ldt, R, ldr, U, ldu,
              sigmas, rhos, betas, coef, fs, st};
  const size_t step_smem = sizeof(double) * (od + m + 32);
  if (step_smem > 48 * 1024)
    cudaFuncSetAttribute(rhqr_step_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)step_smem);
  rhqr_step_kernel<T><<<1, STEP_NT, step_smem, ctx->stream>>>(sa);
  SQB_TRY(check_launch(ctx, "rhqr_step_kernel"));

  double scale_lo = 0.0, norm_lo = 0.0;
  if (srht) srht_constants(sk, Lo<T>::code, &scale_lo, &norm_lo);
  constexpr int VN = VecN<T>::n;
  const bool vec = ((reinterpret_cast<uintptr_t>((const char*)W + m * esz) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>((const char*)U + m * esz) & 15) == 0) &&
                   (ldw % VN == 0) && (ldu % VN == 0);
  const int tb_max = 1 << TileCfg<T>::LOG_TB;
  const int64_t n_eff_col = srht ? g.n_eff : (n + tb_max - 1) / tb_max;
  const int log_tb_col = srht ? g.log_tb : TileCfg<T>::LOG_TB;
  for (int64_t c = 1; c < m; ++c) {
    ColArgs ca{(int)c, (int)m, n, (int)ell, log_tb_col, g.n_tiles, n_eff_col, W, ldw, U, ldu,
               coef, fs, scaling, srht ? 1 : 0, srht ? sk->sign_bits : nullptr,
               srht ? sk->indices : nullptr, scale_lo, P, y, st};
    const size_t smem = sizeof(A) * ((c + 3) & ~3) + (srht ? tile_smem_bytes<A>(tb_max) : 0);
    dim3 grid((unsigned)(n_eff_col + 1));
    prof_begin(ctx);
    if (vec) {
      auto kern = rhqr_col_kernel<T, VN>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, COL_NT, smem, ctx->stream>>>(ca);
    } else {
      auto kern = rhqr_col_kernel<T, 1>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kern<<<grid, COL_NT, smem, ctx->stream>>>(ca);
    }
    // algorithmic bytes of this pass: read U[:, :c] and W[:, c], write U[:, c]
    prof_end(ctx, (double)esz * (double)N * (double)(c + 2));
    SQB_TRY(check_launch(ctx, "rhqr_col_kernel"));
    if (srht) {
      SQB_TRY(launch_srht_tree(ctx, sk, Lo<T>::code, P, 1, y, od, m, st));
    } else {
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)U + (c * ldu + m) * esz, ldu, 1, y, od,
                            m, P, st));
    }
    sa.c = (int)c;
    sa.y = y;
    rhqr_step_kernel<T><<<1, STEP_NT, step_smem, ctx->stream>>>(sa);
    SQB_TRY(check_launch(ctx, "rhqr_step_kernel"));
  }
  // lazy scaling of the last column's Omega rows
  {
    const T* src = m == 1 ? (const T*)W + m : (const T*)U + (m - 1) * ldu + m;
    T* dst = (T*)U + (m - 1) * ldu + m;
    const unsigned gb = (unsigned)std::min<int64_t>((n + 255) / 256, 8 * 148);
    scale_last_kernel<T><<<gb, 256, 0, ctx->stream>>>(src, dst, n, fs, scaling, st);
    SQB_TRY(check_launch(ctx, "scale_last_kernel"));
  }
  return SQB_OK;
}

int rhqr_left_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                       const void* W, int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu,
                       double* S, int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr,
                       double* sigmas, double* rhos, double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rhqr_left_t<double>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rhqr_left_t<float>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rhqr_left_t<__half>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rhqr_left_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
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
