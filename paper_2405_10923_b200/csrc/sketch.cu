// Sketch operators on the device: SRHT (K1, bit-exact), dense Gaussian
// (generic path; the DMMA GEMM lives in dense.cu), identity, embedded.
#include <algorithm>
#include <cmath>

#include "sketch.cuh"
#include "vec.cuh"
#include "dense.cuh"

namespace sqb {

// ---------------------------------------------------------------------------
// host rounding helpers (numpy semantics)
// ---------------------------------------------------------------------------
static uint16_t f32_to_bf16_bits_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // NaN
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

static double bf16_bits_to_double(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

// correctly rounded double -> binary16 (numpy's npy_double_to_half)
static double round_to_half(double x) {
  if (!std::isfinite(x)) return x;
  const double ax = std::fabs(x);
  if (ax >= 65520.0) return std::copysign(INFINITY, x);  // rounds to inf
  if (ax == 0.0) return x;
  int e;
  std::frexp(ax, &e);           // ax = f * 2^e, f in [0.5, 1)
  int q = e - 11;               // ulp exponent for 11 significant bits
  if (q < -24) q = -24;         // subnormal spacing 2^-24
  const double ulp = std::ldexp(1.0, q);
  const double r = std::nearbyint(ax / ulp) * ulp;  // exact scaling by powers of two; RNE
  return std::copysign(r, x);
}

double round_scalar(int dtype, double x) {
  switch (dtype) {
    case SQB_F64: return x;
    case SQB_F32: return (double)(float)x;
    case SQB_F16: return round_to_half(x);
    case SQB_BF16: return bf16_bits_to_double(f32_to_bf16_bits_rne((float)x));
  }
  return x;
}

void srht_constants(const sqb_sketch* sk, int dtype, double* scale_lo, double* norm_lo) {
  *scale_lo = round_scalar(dtype, sk->scale);
  *norm_lo = round_scalar(dtype, std::pow((double)sk->n_pad, -0.5));
}

size_t acc_bytes(int dtype) { return dtype == SQB_F64 ? 8 : 4; }
size_t elem_bytes(int dtype) {
  switch (dtype) {
    case SQB_F64: return 8;
    case SQB_F32: return 4;
    default: return 2;
  }
}

SrhtGeom srht_geom(const sqb_sketch* sk, int dtype) {
  switch (dtype) {
    case SQB_F64: return srht_geom_t<double>(sk);
    case SQB_F32: return srht_geom_t<float>(sk);
    case SQB_F16: return srht_geom_t<__half>(sk);
    default: return srht_geom_t<__nv_bfloat16>(sk);
  }
}

int validate_sketch(sqb_ctx* ctx, const sqb_sketch* sk) {
  if (!sk) return set_error(ctx, SQB_ERR_ARG, "null sketch");
  if (sk->ell < 1 || sk->n < 1)
    return set_error(ctx, SQB_ERR_ARG, "invalid sketch dimensions %lld x %lld", (long long)sk->ell,
                     (long long)sk->n);
  if (sk->kind == SQB_SKETCH_SRHT) {
    if (sk->n_pad < sk->n || (sk->n_pad & (sk->n_pad - 1)))
      return set_error(ctx, SQB_ERR_ARG, "SRHT n_pad %lld is not the padded power of two of %lld",
                       (long long)sk->n_pad, (long long)sk->n);
    if (sk->ell > sk->n_pad)
      return set_error(ctx, SQB_ERR_ARG, "ell=%lld exceeds padded length %lld", (long long)sk->ell,
                       (long long)sk->n_pad);
    if (!sk->sign_bits || !sk->indices) return set_error(ctx, SQB_ERR_ARG, "SRHT without signs/indices");
  } else if (sk->kind == SQB_SKETCH_DENSE) {
    if (!sk->G || sk->ldg < sk->n) return set_error(ctx, SQB_ERR_ARG, "dense sketch without G");
  } else if (sk->kind == SQB_SKETCH_IDENTITY) {
    if (sk->ell != sk->n) return set_error(ctx, SQB_ERR_ARG, "identity sketch must be square");
  } else {
    return set_error(ctx, SQB_ERR_ARG, "unknown sketch kind %d", sk->kind);
  }
  return SQB_OK;
}

// ---------------------------------------------------------------------------
// SRHT kernels
// ---------------------------------------------------------------------------
template <typename T, int VN>
__global__ void __launch_bounds__(SRHT_NT, 4)
srht_tile_kernel(const T* __restrict__ X, int64_t ldx, int64_t n, int log_tb,
                 const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx, int ell,
                 typename Lo<T>::acc scale_lo, typename Lo<T>::acc* __restrict__ P,
                 int64_t n_tiles, const Status* st, int64_t e_base) {
  using A = typename Lo<T>::acc;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* sm = reinterpret_cast<A*>(smem_raw);
  if (st && failed(st)) return;
  const int64_t t = blockIdx.x;
  const int64_t col = blockIdx.y;
  const T* x = X + col * ldx;
  const int tb = 1 << log_tb;
  const int64_t e0 = t << log_tb;
  for (int i = threadIdx.x * VN; i < tb; i += SRHT_NT * VN) {
    const int64_t e = e0 + i;
    A v[VN];
    if (VN > 1 && e + VN <= n) vload_stream<T>(x + e, v);
    else load_run<T, VN>(x, e, n, v);
    const int64_t eg = e_base + e;  // global Omega coordinate (sign bits)
    const uint32_t w = __ldg(bits + (eg >> 5)) >> (eg & 31);
#pragma unroll
    for (int j = 0; j < VN; ++j)
      sm[pidx<A>(i + j)] = (e + j < n) ? srht_in<T>(v[j], scale_lo, (w >> j) & 1u) : A(0);
  }
  __syncthreads();
  tile_fwht<T>(sm, log_tb);
  tile_gather<T>(sm, idx, ell, log_tb, P + (col * ell) * n_tiles + t, n_tiles);
}

// ---------------------------------------------------------------------------
// fp64 SRHT tile pipeline (K1 for the batched raw sketches and sketch_apply):
// persistent CTAs stream (tile, column) items; the next item's tile is copied
// global -> shared with cp.async (coalesced 16-byte chunks, zero-filled past n)
// while the current one is transformed, so HBM reads overlap the butterflies.
// Shared layout pads 2 doubles per 16 (keeps 16-byte chunk alignment and makes
// the radix-16 passes conflict-free: LDS.128 for bits 0-3, 2-way for 4..11).
// ---------------------------------------------------------------------------
constexpr int PIPE_NT = 256;

__device__ __forceinline__ int pidx2(int e) { return e + 2 * (e >> 4); }

template <int R>
__device__ __forceinline__ void fwht_pass2(double* sm, int b, int len) {
  const int groups = len >> R;
  const int lowmask = (1 << b) - 1;
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    const int base = (g & lowmask) | ((g >> b) << (b + R));
    double v[1 << R];
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) v[j] = sm[pidx2(base | (j << b))];
#pragma unroll
    for (int s2 = 0; s2 < R; ++s2)
#pragma unroll
      for (int j = 0; j < (1 << R); ++j)
        if (!(j & (1 << s2))) {
          const double x = v[j], y = v[j | (1 << s2)];
          v[j] = __dadd_rn(x, y);
          v[j | (1 << s2)] = __dsub_rn(x, y);
        }
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) sm[pidx2(base | (j << b))] = v[j];
  }
}

__global__ void __launch_bounds__(PIPE_NT, 3)
srht_tile_pipe_kernel(const double* __restrict__ X, int64_t ldx, int64_t n, int log_tb, int64_t n_eff,
                      int64_t k, const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx, int ell,
                      double scale_lo, double* __restrict__ P, int64_t n_tiles, const Status* st,
                      int64_t e_base) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (st && failed(st)) return;
  const int tb = 1 << log_tb;
  const int tbp = tb + 2 * (tb >> 4);
  double* buf0 = reinterpret_cast<double*>(smem_raw);
  const int64_t items = n_eff * k;
  auto issue = [&](int64_t item, double* buf) {
    if (item >= items) return;
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e0 = t << log_tb;
    const double* x = X + col * ldx + e0;
    const int64_t nv = n - e0;
    for (int q = threadIdx.x; q < (tb >> 1); q += PIPE_NT) {
      const int e = 2 * q;
      double* d = buf + pidx2(e);
      if (e + 2 <= nv) cp_async16(d, x + e, 16);
      else if (e < nv) cp_async16(d, x + e, 8);
      else { d[0] = 0.0; d[1] = 0.0; }
    }
  };
  int64_t item = blockIdx.x;
  issue(item, buf0);
  cp_async_commit_group();
  for (int it = 0; item < items; ++it, item += gridDim.x) {
    double* cur = buf0 + (it & 1) * tbp;
    double* nxt = buf0 + ((it + 1) & 1) * tbp;
    issue(item + gridDim.x, nxt);
    cp_async_commit_group();
    cp_async_wait_group<1>();
    __syncthreads();
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e0 = t << log_tb;
    // pass 0: scale, signs (sketching.py:152-153), stages h = 1..8 in registers
    for (int g = threadIdx.x; g < (tb >> 4); g += PIPE_NT) {
      double* p = cur + pidx2(g << 4);
      double v[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double2 d = *reinterpret_cast<const double2*>(p + 2 * q);
        v[2 * q] = d.x;
        v[2 * q + 1] = d.y;
      }
      const int64_t e = e0 + (g << 4);
      const int64_t eg = e_base + e;
      const uint32_t w = __ldg(bits + (eg >> 5)) >> (eg & 31);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double sv = __dmul_rn(v[j], scale_lo);
        v[j] = (e + j < n) ? (((w >> j) & 1u) ? -sv : sv) : 0.0;
      }
      reg_fwht16<double>(v);
#pragma unroll
      for (int q = 0; q < 8; ++q) *reinterpret_cast<double2*>(p + 2 * q) = make_double2(v[2 * q], v[2 * q + 1]);
    }
    __syncthreads();
    for (int b = 4; b < log_tb; b += 4) {
      const int r = log_tb - b;
      if (r >= 4) fwht_pass2<4>(cur, b, tb);
      else if (r == 3) fwht_pass2<3>(cur, b, tb);
      else if (r == 2) fwht_pass2<2>(cur, b, tb);
      else fwht_pass2<1>(cur, b, tb);
      __syncthreads();
    }
    const int64_t mask = tb - 1;
    double* leaves = P + (col * ell) * n_tiles + t;
    for (int kk = threadIdx.x; kk < ell; kk += PIPE_NT) leaves[kk * n_tiles] = cur[pidx2((int)(__ldg(idx + kk) & mask))];
    __syncthreads();
  }
  cp_async_wait_group<0>();
}

template <typename T>
__global__ void __launch_bounds__(256)
srht_tree_kernel(const typename Lo<T>::acc* __restrict__ P, int64_t n_tiles, int64_t n_eff,
                 const int64_t* __restrict__ idx, int ell, int log_tb,
                 typename Lo<T>::acc norm_lo, double* __restrict__ Y, int64_t ldy,
                 int64_t row_off, const Status* st, int apply_norm) {
  if (st && failed(st)) return;
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t col = blockIdx.y;
  if (k >= ell) return;
  const int64_t rhi = __ldg(idx + k) >> log_tb;
  const typename Lo<T>::acc v =
      warp_tile_tree<T>(P + (col * ell + k) * n_tiles, (int)n_tiles, (int)n_eff, rhi);
  if ((threadIdx.x & 31) == 0) Y[row_off + k + col * ldy] = apply_norm ? (double)Lo<T>::mul(v, norm_lo) : (double)v;
}

template <typename T>
__global__ void copy_top_kernel(const T* __restrict__ X, int64_t ldx, int64_t m,
                                double* __restrict__ Y, int64_t ldy, const Status* st) {
  if (st && failed(st)) return;
  const int64_t col = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    Y[i + col * ldy] = (double)Lo<T>::load(X[i + col * ldx]);
}

template <typename T>
__global__ void identity_kernel(const T* __restrict__ X, int64_t ldx, int64_t n,
                                double* __restrict__ Y, int64_t ldy, int64_t row_off,
                                const Status* st) {
  if (st && failed(st)) return;
  const int64_t col = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    Y[row_off + i + col * ldy] = (double)Lo<T>::load(X[i + col * ldx]);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
size_t sketch_partials_bytes(const sqb_sketch* sk, int dtype, int64_t k) {
  if (sk->kind != SQB_SKETCH_SRHT) return dense_ws_bytes(sk, dtype, k);
  const SrhtGeom g = srht_geom(sk, dtype);
  return acc_bytes(dtype) * (size_t)sk->ell * (size_t)g.n_tiles * (size_t)k;
}

template <typename T>
static int srht_tiles_geom_t(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local,
                             int64_t e_base, const void* X, int64_t ldx, int64_t k, void* P,
                             const Status* st) {
  using A = typename Lo<T>::acc;
  double sc, nm;
  srht_constants(sk, Lo<T>::code, &sc, &nm);
  const size_t smem = tile_smem_bytes<A>(1 << g.log_tb);
  constexpr int VN = VecN<T>::n;
  const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && (ldx % VN == 0) &&
                   (g.log_tb >= 3);
  dim3 grid((unsigned)g.n_eff, (unsigned)k);
  if constexpr (sizeof(T) == 8) {
    if (vec && g.log_tb >= 4 && (e_base & 15) == 0) {
      const int tb = 1 << g.log_tb;
      const size_t psmem = 2 * sizeof(double) * (size_t)(tb + 2 * (tb >> 4));
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(srht_tile_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(80 << 10));
        cudaFuncSetAttribute(srht_tile_pipe_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        attr = true;
      }
      const int64_t items = g.n_eff * k;
      const unsigned gp = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, 3 * (int64_t)ctx->sm_count));
      srht_tile_pipe_kernel<<<gp, PIPE_NT, psmem, ctx->stream>>>(
          (const double*)X, ldx, n_local, g.log_tb, g.n_eff, k, sk->sign_bits, sk->indices, (int)sk->ell, sc,
          (double*)P, g.n_tiles, st, e_base);
      return check_launch(ctx, "srht_tile_pipe_kernel");
    }
  }
  if (vec) {
    auto kern = srht_tile_kernel<T, VN>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    kern<<<grid, SRHT_NT, smem, ctx->stream>>>((const T*)X, ldx, n_local, g.log_tb, sk->sign_bits,
                                               sk->indices, (int)sk->ell, (A)sc, (A*)P, g.n_tiles, st, e_base);
  } else {
    auto kern = srht_tile_kernel<T, 1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, SRHT_NT, smem, ctx->stream>>>((const T*)X, ldx, n_local, g.log_tb, sk->sign_bits,
                                               sk->indices, (int)sk->ell, (A)sc, (A*)P, g.n_tiles, st, e_base);
  }
  return check_launch(ctx, "srht_tile_kernel");
}

template <typename T>
static int srht_tiles_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                        void* P, const Status* st) {
  return srht_tiles_geom_t<T>(ctx, sk, srht_geom_t<T>(sk), sk->n, 0, X, ldx, k, P, st);
}

template <typename T>
static int srht_tree_geom_t(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, const void* P, int64_t k,
                            double* Y, int64_t ldy, int64_t row_off, int apply_norm, const Status* st) {
  using A = typename Lo<T>::acc;
  double sc, nm;
  srht_constants(sk, Lo<T>::code, &sc, &nm);
  dim3 grid((unsigned)((sk->ell + 7) / 8), (unsigned)k);
  srht_tree_kernel<T><<<grid, 256, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                     (int)sk->ell, g.log_tb, (A)nm, Y, ldy, row_off, st,
                                                     apply_norm);
  return check_launch(ctx, "srht_tree_kernel");
}

template <typename T>
static int srht_tree_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* P, int64_t k, double* Y,
                       int64_t ldy, int64_t row_off, const Status* st) {
  using A = typename Lo<T>::acc;
  const SrhtGeom g = srht_geom_t<T>(sk);
  double sc, nm;
  srht_constants(sk, Lo<T>::code, &sc, &nm);
  dim3 grid((unsigned)((sk->ell + 7) / 8), (unsigned)k);
  srht_tree_kernel<T><<<grid, 256, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                     (int)sk->ell, g.log_tb, (A)nm, Y, ldy, row_off, st, 1);
  return check_launch(ctx, "srht_tree_kernel");
}

#define SQB_DISPATCH(dtype, FN, ...)                                   \
  switch (dtype) {                                                      \
    case SQB_F64: return FN<double>(__VA_ARGS__);                       \
    case SQB_F32: return FN<float>(__VA_ARGS__);                        \
    case SQB_F16: return FN<__half>(__VA_ARGS__);                       \
    case SQB_BF16: return FN<__nv_bfloat16>(__VA_ARGS__);               \
    default: return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", dtype); \
  }

int launch_srht_tree(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* P, int64_t k,
                     double* Y, int64_t ldy, int64_t y_row_off, const Status* st) {
  SQB_DISPATCH(dtype, srht_tree_t, ctx, sk, P, k, Y, ldy, y_row_off, st);
}

int launch_srht_tiles_geom(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const SrhtGeom& g, int64_t n_local,
                           int64_t e_base, const void* X, int64_t ldx, int64_t k, void* P, const Status* st) {
  SQB_DISPATCH(dtype, srht_tiles_geom_t, ctx, sk, g, n_local, e_base, X, ldx, k, P, st);
}

int launch_srht_tree_geom(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const SrhtGeom& g, const void* P,
                          int64_t k, double* Y, int64_t ldy, int64_t row_off, int apply_norm, const Status* st) {
  SQB_DISPATCH(dtype, srht_tree_geom_t, ctx, sk, g, P, k, Y, ldy, row_off, apply_norm, st);
}

template <typename T>
static int identity_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                      double* Y, int64_t ldy, int64_t row_off, const Status* st) {
  dim3 grid((unsigned)std::min<int64_t>((sk->n + 255) / 256, 4096), (unsigned)k);
  identity_kernel<T><<<grid, 256, 0, ctx->stream>>>((const T*)X, ldx, sk->n, Y, ldy, row_off, st);
  return check_launch(ctx, "identity_kernel");
}

template <typename T>
static int copy_top_t(sqb_ctx* ctx, const void* X, int64_t ldx, int64_t m, int64_t k, double* Y,
                      int64_t ldy, const Status* st) {
  if (m == 0 || k == 0) return SQB_OK;
  dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 1024), (unsigned)k);
  copy_top_kernel<T><<<grid, 256, 0, ctx->stream>>>((const T*)X, ldx, m, Y, ldy, st);
  return check_launch(ctx, "copy_top_kernel");
}

int launch_copy_top(sqb_ctx* ctx, int dtype, const void* X, int64_t ldx, int64_t m, int64_t k,
                    double* Y, int64_t ldy, const Status* st) {
  SQB_DISPATCH(dtype, copy_top_t, ctx, X, ldx, m, k, Y, ldy, st);
}

template <typename T>
static int sketch_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                    double* Y, int64_t ldy, int64_t row_off, void* partials, const Status* st) {
  if (k == 0) return SQB_OK;
  if (sk->kind == SQB_SKETCH_SRHT) {
    SQB_TRY(srht_tiles_t<T>(ctx, sk, X, ldx, k, partials, st));
    return srht_tree_t<T>(ctx, sk, partials, k, Y, ldy, row_off, st);
  }
  if (sk->kind == SQB_SKETCH_IDENTITY) return identity_t<T>(ctx, sk, X, ldx, k, Y, ldy, row_off, st);
  return launch_dense<T>(ctx, sk, X, ldx, k, Y, ldy, row_off, partials, st);
}

int launch_sketch(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* X, int64_t ldx,
                  int64_t k, double* Y, int64_t ldy, int64_t y_row_off, void* partials,
                  const Status* st) {
  SQB_DISPATCH(dtype, sketch_t, ctx, sk, X, ldx, k, Y, ldy, y_row_off, partials, st);
}

}  // namespace sqb
