// Sketch operators on the device: SRHT (K1, bit-exact), dense Gaussian
// (generic path; the DMMA GEMM lives in dense.cu), identity, embedded.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "sketch.cuh"
#include "vec.cuh"
#include "dense.cuh"
#include "tma.cuh"

namespace sqb {

// SQB_<NAME>=0 switches an optimisation off (A/B experiments)
static bool getenv_flag0(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '0';
}


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

int validate_left_args(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int64_t N, int64_t m) {
  SQB_TRY(validate_sketch(ctx, sk));
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need at least one column");
  if (m > 1024) return set_error(ctx, SQB_ERR_ARG, "m=%lld: the device sweep supports up to 1024 columns", (long long)m);
  if (sk->n != N - m)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld",
                     (long long)sk->n, (long long)(N - m));
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
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
  tile_gather<T>(sm, idx, ell, log_tb, P + (col * n_tiles + t) * ell, 1);
}

// ---------------------------------------------------------------------------
// K1 standalone tile kernel (batched raw sketches, sketch_apply, the compact
// updates): a 4096-coordinate tile is owned by 64 threads holding 64 values
// each, so the 12 in-tile stages are TWO register passes (bits 0-5, then
// bits 6-11) with one shared-memory round trip between them.  Persistent
// CTAs walk (tile, column) items; the next item's raw values are copied
// global -> shared by cp.async while the current one is transformed.  After
// pass 2 only the sampled coordinates are written back (a per-thread 64-bit
// mask), then gathered into the leaves.  Shared rows of 64 elements are padded
// by 16 bytes: pass-1 LDS.128 and pass-2 LDS are both conflict-free.
// ---------------------------------------------------------------------------
constexpr int S64_NT = 64, S64_LOG = 12, S64_TB = 1 << S64_LOG;

template <typename E>
__host__ __device__ constexpr int s64_pad() { return 16 / (int)sizeof(E); }
template <typename E>
__device__ __forceinline__ int s64_idx(int e) { return e + s64_pad<E>() * (e >> 6); }
template <typename E>
__host__ __device__ constexpr size_t s64_buf_bytes() {
  return sizeof(E) * (size_t)(S64_TB + s64_pad<E>() * (S64_TB >> 6));
}
// v with its sign bit flipped iff bit j of w is set
__device__ __forceinline__ double flip_sign(double v, uint32_t w, int j) {
  const int2 p = *reinterpret_cast<int2*>(&v);
  const int hi = p.y ^ (int)((w << (31 - j)) & 0x80000000u);
  return __hiloint2double(hi, p.x);
}
__device__ __forceinline__ float flip_sign(float v, uint32_t w, int j) {
  return __int_as_float(__float_as_int(v) ^ (int)((w << (31 - j)) & 0x80000000u));
}

// 6 butterfly stages over 64 register values (stages b .. b+5 of the tile)
template <typename T>
__device__ __forceinline__ void fwht64_regs(typename Lo<T>::acc (&v)[64]) {
#pragma unroll
  for (int s2 = 0; s2 < 6; ++s2)
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (!(j & (1 << s2))) {
        const typename Lo<T>::acc x = v[j], y = v[j | (1 << s2)];
        v[j] = Lo<T>::add(x, y);
        v[j | (1 << s2)] = Lo<T>::sub(x, y);
      }
}

// smem layout shared by the 4096-tile kernels:
//   [smask 64 x u64][spre 64 x int][kslot ell x int][samp ell x acc][tile buffer]
// samp holds the transformed value of every distinct sampled coordinate
// (slot = prefix count over the (t, j) mask bits), kslot maps output k to its
// slot, so the tile buffer is free as soon as pass 2 has loaded it.
constexpr int S64_MAX_ELL = 2048;
__host__ __device__ inline size_t s64_samp_off(int ell) { return (768 + 4 * (size_t)ell + 15) & ~(size_t)15; }
__host__ __device__ inline size_t s64_head_bytes(int ell, size_t acc) {
  return (s64_samp_off(ell) + (size_t)ell * acc + 127) & ~(size_t)127;
}

// build smask / spre / kslot (one CTA, S64_NT threads); ends with a barrier
__device__ __forceinline__ void s64_sample_maps(const int64_t* __restrict__ idx, int ell,
                                                unsigned long long* smask, int* spre, int* kslot) {
  const int tid = threadIdx.x;
  smask[tid] = 0ull;
  __syncthreads();
  for (int kk = tid; kk < ell; kk += S64_NT) {
    const int p = (int)(__ldg(idx + kk) & (S64_TB - 1));
    atomicOr(&smask[p & 63], 1ull << (p >> 6));
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int t = 0; t < 64; ++t) { spre[t] = acc; acc += __popcll(smask[t]); }
  }
  __syncthreads();
  for (int kk = tid; kk < ell; kk += S64_NT) {
    const int p = (int)(__ldg(idx + kk) & (S64_TB - 1));
    const int t = p & 63, j = p >> 6;
    kslot[kk] = spre[t] + __popcll(smask[t] & ((1ull << j) - 1ull));
  }
  __syncthreads();
}

// fp64 / fp32 storage (values stay in the storage type end to end)
template <typename T>
__global__ void __launch_bounds__(S64_NT)
srht64_tile_kernel(const T* __restrict__ X, int64_t ldx, int64_t n, int64_t n_eff, int64_t k,
                   const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx, int ell,
                   T scale_lo, T* __restrict__ P, int64_t n_tiles, const Status* st, int64_t e_base) {
  static_assert(sizeof(T) == sizeof(typename Lo<T>::acc), "storage = arithmetic type");
  constexpr int C = 16 / (int)sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* smask = reinterpret_cast<unsigned long long*>(smem_raw);
  int* spre = reinterpret_cast<int*>(smem_raw + 512);
  int* kslot = reinterpret_cast<int*>(smem_raw + 768);
  T* samp = reinterpret_cast<T*>(smem_raw + s64_samp_off(ell));
  T* buf = reinterpret_cast<T*>(smem_raw + s64_head_bytes(ell, sizeof(T)));
  if (st && failed(st)) return;
  const int tid = threadIdx.x;
  s64_sample_maps(idx, ell, smask, spre, kslot);
  const uint32_t mlo = (uint32_t)smask[tid], mhi = (uint32_t)(smask[tid] >> 32);
  const int mypre = spre[tid];
  const int64_t items = n_eff * k;
  auto issue = [&](int64_t item) {
    if (item >= items) return;
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e0 = t << S64_LOG;
    const T* x = X + col * ldx + e0;
    const int64_t nv = n - e0;
    if (nv >= S64_TB) {
      const T* src = x + tid * C;
      T* dst = buf + s64_idx<T>(tid * C);
#pragma unroll
      for (int i = 0; i < S64_TB / (C * S64_NT); ++i)
        cp_async16(dst + i * (S64_NT * C + s64_pad<T>() * C), src + i * S64_NT * C, 16);
    } else {
      for (int q = tid; q < S64_TB / C; q += S64_NT) {
        const int e = q * C;
        const int64_t rem = nv - e;
        const int bytes = rem >= C ? 16 : (rem > 0 ? (int)rem * (int)sizeof(T) : 0);
        cp_async16(buf + s64_idx<T>(e), bytes > 0 ? (const void*)(x + e) : (const void*)x, bytes);
      }
    }
  };
  auto sign_words = [&](int64_t item, uint32_t& a0, uint32_t& a1) {
    if (item >= items) return;
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t eg = e_base + (t << S64_LOG) + tid * 64;
    a0 = __ldg(bits + (eg >> 5));
    a1 = __ldg(bits + (eg >> 5) + 1);
  };
  int64_t item = blockIdx.x;
  uint32_t w0 = 0, w1 = 0;
  issue(item);
  cp_async_commit_group();
  sign_words(item, w0, w1);
  for (; item < items; item += gridDim.x) {
    cp_async_wait_group<0>();
    __syncthreads();
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e = (t << S64_LOG) + tid * 64;
    T v[64];
    // pass 1: coordinates 64 tid .. +63: scale, signs (sketching.py:152-153), stages h = 1..32
    {
      T* row = buf + s64_idx<T>(tid * 64);
#pragma unroll
      for (int q = 0; q < 64 / C; ++q) vload<T>(row + q * C, v + q * C);
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = flip_sign(Lo<T>::mul(v[j], scale_lo), j < 32 ? w0 : w1, j & 31);
      if (e + 64 > n) {  // zero padding past n is +0 (sketching.py:154)
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (e + j >= n) v[j] = T(0);
      }
      fwht64_regs<T>(v);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 64 / C; ++q) vstore<T>(row + q * C, v + q * C);
    }
    __syncthreads();
    // pass 2: coordinates tid + 64 j, stages h = 64 .. 2048
    {
      const T* col0 = buf + tid;  // s64_idx(tid + 64 j) = tid + j (64 + pad): constant offsets
#pragma unroll
      for (int j = 0; j < 64; ++j) v[j] = col0[j * (64 + s64_pad<T>())];
    }
    __syncthreads();  // tile buffer free: stream the next item in behind pass 2
    issue(item + gridDim.x);
    cp_async_commit_group();
    sign_words(item + gridDim.x, w0, w1);
    fwht64_regs<T>(v);
    {
      int slot = mypre;  // sampled coordinates of this thread in j order
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (((j < 32 ? mlo : mhi) & (1u << (j & 31))) != 0u) samp[slot++] = v[j];
    }
    __syncthreads();
    T* leaves = P + (col * n_tiles + t) * ell;
    for (int kk = tid; kk < ell; kk += S64_NT) leaves[kk] = samp[kslot[kk]];
  }
  cp_async_wait_group<0>();
}

template <typename T>
__device__ __forceinline__ void fwht32_regs(T (&v)[32]) {
#pragma unroll
  for (int s2 = 0; s2 < 5; ++s2)
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (!(j & (1 << s2))) {
        const T x = v[j], y = v[j | (1 << s2)];
        v[j] = Lo<T>::add(x, y);
        v[j | (1 << s2)] = Lo<T>::sub(x, y);
      }
}

template <typename T>
__host__ __device__ constexpr int wt_rs() { return 32 + 16 / (int)sizeof(T); }  // padded row (elements)

// ---------------------------------------------------------------------------
// K1 standalone for fp64 / fp32 storage: TMA-staged warp tiles.
//   * One WARP owns a 4096-coordinate leaf group as four 1024-coordinate
//     sub-tiles.  A lane holds 32 values, so a sub-tile is two 5-stage
//     register passes: bits 0-4 on the lane's contiguous run, bits 5-9 after
//     one warp-private shared-memory transpose (padded rows: conflict-free).
//   * Stages h = 1024 and 2048 are evaluated only at the sampled coordinates:
//     output k at in-group position p is (s0 +- s1) +- (s2 +- s3), s_q = the
//     sub-tile-q value at p mod 1024, signs from bits 10 and 11 of p, lower
//     operand first — exactly what the full stages compute at p (the identity
//     the cross-tile tree also uses), so the leaves are bitwise those of the
//     4096-coordinate tile and the tree kernel is shared.  2/12 fewer
//     butterflies than the CTA tile kernel.
//   * Every full sub-tile arrives through the tensor-memory accelerator: a
//     3-D tensor map (elements of one 128-byte half-run x runs of 32
//     coordinates x columns), SWIZZLE_128B, one box per half, completion on a
//     per-stage mbarrier.  Each warp owns an S-stage ring; a stage is
//     refilled (S sub-tiles ahead) as soon as pass 1 has read it, so HBM
//     latency is covered by the ring, not by registers, and no global load
//     crosses the L1 pipe.  Lane l's run is swizzled row l of each half
//     (chunk c at c ^ (l & 7)): the lane-run reads are conflict-free.
//   * Warps walk contiguous (column, group) ranges with cursors (no
//     per-sub-tile division); the tree levels 10/11 are branch-free selects.
// Measured (B200, 2^20 x 128 fp64, ell = 256; scripts/ab_srht.py): 0.54 ->
// 0.60 of HBM vs the CTA tile kernel; variants with direct lane-run loads
// (LDG.128: L1-bound at 98 %; LDG.256: 0.56; register prefetch: 0.51) lost.
// ---------------------------------------------------------------------------
template <typename T>
struct Tma {
  static constexpr int HALF = 128 / (int)sizeof(T);  // elements per swizzled row
  static constexpr int NH = 32 / HALF;                 // rows (halves) per 32-coordinate run
  static constexpr int STAGE = 32 * 32 * (int)sizeof(T);  // bytes per sub-tile
};

// byte offset of run r, element i (0..31) inside a swizzled stage buffer
template <typename T>
__device__ __forceinline__ uint32_t tma_off(uint32_t r, uint32_t i) {
  constexpr int HALF = Tma<T>::HALF;
  const uint32_t h = i / HALF, c = (i % HALF) * sizeof(T);
  return h * 4096u + r * 128u + ((((c >> 4) ^ (r & 7u)) << 4) | (c & 15u));
}

// LG: log2 of the leaf group (12: 4 sub-tiles, levels 10-11 at the sampled
// positions; 13: 8 sub-tiles, levels 10-12 — half the leaves for the tree)
template <typename T, int KPL, int S, int WPB, int LG>
__global__ void __launch_bounds__(WPB * 32)
srht_tma_tile_kernel(const __grid_constant__ CUtensorMap map, const T* __restrict__ X, int64_t ldx, int64_t n,
                     int64_t n_eff, int64_t k, const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx,
                     int ell, T scale_lo, T* __restrict__ P, int64_t n_tiles, const Status* st, int64_t e_base) {
  static_assert(sizeof(T) == sizeof(typename Lo<T>::acc), "storage = arithmetic type");
  constexpr int C = 16 / (int)sizeof(T), RS = wt_rs<T>();
  constexpr uint32_t SB = Tma<T>::STAGE;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (st && failed(st)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // [1024-aligned TMA stages: WPB x S x SB][padded transpose buffers: WPB x 32 x RS][barriers]
  // (offset from smem_raw itself so the compiler keeps the shared address space)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stages = base + (size_t)wid * S * SB;
  T* buf = reinterpret_cast<T*>(base + (size_t)WPB * S * SB) + wid * 32 * RS;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)WPB * S * SB + sizeof(T) * (size_t)WPB * 32 * RS) + wid * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  static_assert(LG == 12 || LG == 13, "leaf group of 4 or 8 sub-tiles");
  constexpr int NQ = 1 << (LG - 10);  // sub-tiles per leaf group
  // per output k = lane + 32 i: byte offset of its position p mod 1024 in the
  // transpose buffer (bits 0-15), bits 10.. of p from bit 16 up
  uint32_t mypk[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int kk = lane + 32 * i;
    const uint32_t p = kk < ell ? (uint32_t)(__ldg(idx + kk) & ((1 << LG) - 1)) : 0u;
    mypk[i] = (uint32_t)(((p & 1023u) >> 5) * RS + (p & 31u)) * (uint32_t)sizeof(T) | ((p >> 10) << 16);
  }
  // each warp owns a contiguous run of (column, group) items, walked by
  // cursors (no per-unit division): one for the unit being transformed, one
  // for the unit whose TMA load is issued S units ahead, one for sign words
  const int64_t items = n_eff * k;
  const int64_t nwarps = (int64_t)gridDim.x * WPB;
  const int64_t wg = (int64_t)blockIdx.x * WPB + wid;
  // items wg, wg + nwarps, ...: groups processed at the same time are adjacent,
  // so the 8-byte / 4-byte leaf writes of neighbouring groups meet in L2 and
  // leave as whole sectors (a contiguous range per warp doubled DRAM writes)
  const int64_t my_items = wg < items ? (items - wg + nwarps - 1) / nwarps : 0;
  const int64_t dcol = nwarps / n_eff, dg = nwarps - dcol * n_eff;
  const int64_t units = my_items * NQ;  // sub-tiles this warp processes
  struct Cur {  // (column, group, sub-tile) of a unit; advance without division
    int64_t col, g;
    int q;
    __device__ void next(int64_t ne, int64_t dc, int64_t dgg) {
      if (++q == NQ) {
        q = 0;
        g += dgg;
        col += dc;
        if (g >= ne) { g -= ne; ++col; }
      }
    }
    __device__ int64_t e0() const { return (g << LG) + ((int64_t)q << 10); }
  };
  Cur cu{wg / n_eff, wg % n_eff, 0};
  Cur ci = cu, cw = cu;
  auto issue = [&](int64_t u) {  // lane 0 only; unit u (= cursor ci) is loaded by TMA iff it lies below n
    const int64_t e0 = ci.e0();
    if (e0 + 1024 > n) return;
    const int s = (int)(u % S);
    uint64_t* b = bars + s;
    unsigned char* dst = stages + (size_t)s * SB;
    mbar_expect_tx(b, SB);
#pragma unroll
    for (int h = 0; h < Tma<T>::NH; ++h)
      tma_load_3d(dst + h * 4096, &map, h * Tma<T>::HALF, (int)(e0 >> 5), (int)ci.col, b);
  };
  if (lane == 0)
    for (int64_t u = 0; u < S && u < units; ++u) { issue(u); ci.next(n_eff, dcol, dg); }
  uint32_t phase = 0;  // bit s = parity expected next on stage s
  uint32_t w_next = units > 0 ? __ldg(bits + ((e_base + cw.e0() + lane * 32) >> 5)) : 0u;
  cw.next(n_eff, dcol, dg);
  // lane-run reads of a swizzled stage: chunk c of half h at (c ^ (lane & 7))
  const uint32_t run_base = (uint32_t)lane * 128u, run_x = ((uint32_t)lane & 7u) << 4;
  T ab[KPL], acc[KPL], ac2[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) ab[i] = acc[i] = ac2[i] = T(0);
  for (int64_t u = 0; u < units; ++u, cu.next(n_eff, dcol, dg)) {
    const int64_t col = cu.col, e0 = cu.e0();
    const int q = cu.q;
    const int s = (int)(u % S);
    const int64_t e = e0 + lane * 32;
    const uint32_t w = w_next;
    if (u + 1 < units) w_next = __ldg(bits + ((e_base + cw.e0() + lane * 32) >> 5));
    cw.next(n_eff, dcol, dg);
    T v[32];
    unsigned char* sb = stages + (size_t)s * SB;
    const bool full = e0 + 1024 <= n;
    if (full) {
      mbar_wait(bars + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    } else {  // the column tail: stage it by hand in the same swizzled layout
      const T* x = X + col * ldx;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        *reinterpret_cast<T*>(sb + tma_off<T>(lane, j)) = (e + j < n) ? x[e + j] : T(0);
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < 32 / C; ++c) {
      const uint32_t h = (uint32_t)(c * C) / Tma<T>::HALF, cc = (uint32_t)(c % (Tma<T>::HALF / C));
      const uint4 r = *reinterpret_cast<const uint4*>(sb + h * 4096u + run_base + ((cc << 4) ^ run_x));
      unpack16<T>(r, v + c * C);
    }
    // the stage is consumed: refill it with unit u + S
    __syncwarp();
    if (lane == 0 && u + S < units) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(u + S);
      ci.next(n_eff, dcol, dg);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = flip_sign(Lo<T>::mul(v[j], scale_lo), w, j);
    if (e + 32 > n) {  // zero padding past n is +0 (sketching.py:154)
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (e + j >= n) v[j] = T(0);
    }
    fwht32_regs<T>(v);  // h = 1..16
    {
      T* row = buf + lane * RS;
#pragma unroll
      for (int c = 0; c < 32 / C; ++c) vstore<T>(row + c * C, v + c * C);
    }
    __syncwarp();
    // lane-column l holds coordinates l + 32 j; reads and writes stay in the column
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = buf[j * RS + lane];
    fwht32_regs<T>(v);  // h = 32..512
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[j * RS + lane] = v[j];
    __syncwarp();
    // tree levels 10.. at the sampled positions (a binary counter over the
    // group's sub-tiles, warp-uniform in q; left operand = lower sub-tiles):
    // acc = (q odd) ? acc -+ s : s ; ab = the level-11 node of sub-tiles 0-3
    // (x - y is x + (-y) exactly, so the sign bit selects add or sub)
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const uint32_t pk = mypk[i];
      const T sv = *reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(buf) + (pk & 0xffffu));
      const T t = Lo<T>::add(acc[i], flip_sign(sv, pk, 16));
      if ((q & 3) == 2) ab[i] = acc[i];
      acc[i] = (q & 1) ? t : sv;
      if (LG == 13 && q == 3) ac2[i] = Lo<T>::add(ab[i], flip_sign(acc[i], pk, 17));
    }
    if (q == NQ - 1) {
      T* leaves = P + (col * n_tiles + (e0 >> LG)) * ell;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int kk = lane + 32 * i;
        const T l11 = Lo<T>::add(ab[i], flip_sign(acc[i], mypk[i], 17));
        if (kk < ell) leaves[kk] = LG == 13 ? Lo<T>::add(ac2[i], flip_sign(l11, mypk[i], 18)) : l11;
      }
    }
    __syncwarp();
  }
}

// Few leaf groups (a single vector, a short matrix): one CTA per 4096-
// coordinate group, warp q transforms sub-tile q (the same per-sub-tile code
// as srht_tma_tile_kernel), the four sampled values of each output meet in
// shared memory and fold as (s0 +- s1) +- (s2 +- s3) — the same operations
// in the same order, so the leaves are bitwise those of the warp-per-group
// kernel, at a quarter of its per-group latency.
template <typename T, int KPL>
__global__ void __launch_bounds__(128)
srht_tma_split_kernel(const __grid_constant__ CUtensorMap map, const T* __restrict__ X, int64_t ldx, int64_t n,
                      int64_t n_eff, int64_t k, const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx,
                      int ell, T scale_lo, T* __restrict__ P, int64_t n_tiles, const Status* st, int64_t e_base) {
  constexpr int C = 16 / (int)sizeof(T), RS = wt_rs<T>();
  constexpr uint32_t SB = Tma<T>::STAGE;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (st && failed(st)) return;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  // [1024-aligned stages: 4 x SB][transpose buffers: 4 x 32 x RS][samples: 4 x 32 KPL][barriers: 4]
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sb = base + (size_t)q * SB;
  T* buf = reinterpret_cast<T*>(base + 4 * (size_t)SB) + q * 32 * RS;
  T* samp = reinterpret_cast<T*>(base + 4 * (size_t)SB + sizeof(T) * 4 * 32 * RS);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 4 * (size_t)SB + sizeof(T) * 4 * 32 * (RS + KPL)) + q;
  if (lane == 0) mbar_init(bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t mypk[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int kk = lane + 32 * i;
    const uint32_t p = kk < ell ? (uint32_t)(__ldg(idx + kk) & 1023) : 0u;
    mypk[i] = (uint32_t)((p >> 5) * RS + (p & 31u)) * (uint32_t)sizeof(T);
  }
  const uint32_t run_base = (uint32_t)lane * 128u, run_x = ((uint32_t)lane & 7u) << 4;
  uint32_t phase = 0;
  const int64_t items = n_eff * k;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t col = item / n_eff, g = item - col * n_eff;
    const int64_t e0 = (g << 12) + ((int64_t)q << 10), e = e0 + lane * 32;
    const bool full = e0 + 1024 <= n;
    if (full) {
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, SB);
#pragma unroll
        for (int h = 0; h < Tma<T>::NH; ++h)
          tma_load_3d(sb + h * 4096, &map, h * Tma<T>::HALF, (int)(e0 >> 5), (int)col, bar);
      }
    }
    const uint32_t w = __ldg(bits + ((e_base + e) >> 5));
    if (full) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {  // the column tail / padding: staged by hand in the same swizzled layout
      const T* x = X + col * ldx;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        *reinterpret_cast<T*>(sb + tma_off<T>(lane, j)) = (e + j < n) ? x[e + j] : T(0);
      __syncwarp();
    }
    T v[32];
#pragma unroll
    for (int c = 0; c < 32 / C; ++c) {
      const uint32_t h = (uint32_t)(c * C) / Tma<T>::HALF, cc = (uint32_t)(c % (Tma<T>::HALF / C));
      const uint4 r = *reinterpret_cast<const uint4*>(sb + h * 4096u + run_base + ((cc << 4) ^ run_x));
      unpack16<T>(r, v + c * C);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = flip_sign(Lo<T>::mul(v[j], scale_lo), w, j);
    if (e + 32 > n) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (e + j >= n) v[j] = T(0);
    }
    fwht32_regs<T>(v);  // h = 1..16
    {
      T* row = buf + lane * RS;
#pragma unroll
      for (int c = 0; c < 32 / C; ++c) vstore<T>(row + c * C, v + c * C);
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = buf[j * RS + lane];
    fwht32_regs<T>(v);  // h = 32..512
#pragma unroll
    for (int j = 0; j < 32; ++j) buf[j * RS + lane] = v[j];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < KPL; ++i)
      samp[q * 32 * KPL + lane + 32 * i] =
          *reinterpret_cast<const T*>(reinterpret_cast<const unsigned char*>(buf) + mypk[i]);
    __syncthreads();
    T* leaves = P + (col * n_tiles + g) * ell;
    for (int kk = threadIdx.x; kk < ell; kk += 128) {
      const uint32_t p = (uint32_t)(__ldg(idx + kk) & 4095);
      const T s0 = samp[kk], s1 = samp[32 * KPL + kk], s2 = samp[64 * KPL + kk], s3 = samp[96 * KPL + kk];
      const T a = Lo<T>::add(s0, flip_sign(s1, p, 10));
      const T b = Lo<T>::add(s2, flip_sign(s3, p, 10));
      leaves[kk] = Lo<T>::add(a, flip_sign(b, p, 11));
    }
    __syncthreads();  // samples and stages are reused by the next item
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <typename T, int KPL, int S, int WPB, int LG>
static int launch_tma(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local, int64_t e_base,
                      const T* X, int64_t ldx, int64_t k, T sc, T* P, const Status* st) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return set_error(ctx, SQB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  const cuuint64_t runs = (cuuint64_t)(n_local >> 5);
  const cuuint64_t dims[3] = {(cuuint64_t)Tma<T>::HALF * Tma<T>::NH, std::max<cuuint64_t>(runs, 1), (cuuint64_t)k};
  const cuuint64_t strides[2] = {32 * sizeof(T), (cuuint64_t)ldx * sizeof(T)};
  const cuuint32_t box[3] = {(cuuint32_t)Tma<T>::HALF, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                         const_cast<T*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ctx, SQB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  const size_t smem = 1024 + (size_t)WPB * S * Tma<T>::STAGE + sizeof(T) * (size_t)WPB * 32 * wt_rs<T>() +
                       (size_t)WPB * S * 8;
  auto kern = srht_tma_tile_kernel<T, KPL, S, WPB, LG>;
  allow_dyn_smem(kern, (size_t)(smem));
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, smem);
  per_sm = std::max(1, per_sm);
  const int64_t items = g.n_eff * k;
  const int64_t ctas =
      std::max<int64_t>(1, std::min<int64_t>((items + WPB - 1) / WPB, (int64_t)per_sm * ctx->sm_count));
  kern<<<(unsigned)ctas, WPB * 32, smem, ctx->stream>>>(map, X, ldx, n_local, g.n_eff, k, sk->sign_bits,
                                                         sk->indices, (int)sk->ell, sc, P, g.n_tiles, st, e_base);
  return check_launch(ctx, "srht_tma_tile_kernel");
}

template <typename T, int KPL>
static int launch_tma_split(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local, int64_t e_base,
                            const T* X, int64_t ldx, int64_t k, T sc, T* P, const Status* st) {
  EncodeTiledFn enc = encode_tiled();
  CUtensorMap map;
  const cuuint64_t runs = (cuuint64_t)(n_local >> 5);
  const cuuint64_t dims[3] = {(cuuint64_t)Tma<T>::HALF * Tma<T>::NH, std::max<cuuint64_t>(runs, 1), (cuuint64_t)k};
  const cuuint64_t strides[2] = {32 * sizeof(T), (cuuint64_t)ldx * sizeof(T)};
  const cuuint32_t box[3] = {(cuuint32_t)Tma<T>::HALF, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(&map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                         const_cast<T*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ctx, SQB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  const size_t smem = 1024 + 4 * (size_t)Tma<T>::STAGE + sizeof(T) * 4 * 32 * (size_t)(wt_rs<T>() + KPL) + 4 * 8;
  auto kern = srht_tma_split_kernel<T, KPL>;
  allow_dyn_smem(kern, (size_t)(smem));
  const int64_t items = g.n_eff * k;
  kern<<<(unsigned)std::min<int64_t>(items, 65535), 128, smem, ctx->stream>>>(
      map, X, ldx, n_local, g.n_eff, k, sk->sign_bits, sk->indices, (int)sk->ell, sc, P, g.n_tiles, st, e_base);
  return check_launch(ctx, "srht_tma_split_kernel");
}

template <typename T, int S, int WPB>
static int launch_tma_kpl(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local, int64_t e_base,
                          const T* X, int64_t ldx, int64_t k, T sc, T* P, const Status* st) {
  const int kpl = (int)((sk->ell + 31) / 32);
  // few 4096-coordinate groups (<= 4 per SM): one CTA per group, a warp per
  // sub-tile (SQB_K1_SPLIT=0: the warp-per-group kernel).  Measured (digests
  // unchanged): 2^20 x 1 14.5 vs 18.9 us, 16352 x 32 14.2 vs 18.1 us,
  // 5000 x 3 13.8 vs 17.9 us; at 2^22 x 1 (1024 groups) 26.2 vs 23.9 us, so
  // many groups keep the warp-per-group kernel
  if (g.log_tb == S64_LOG && g.n_eff * k <= 4 * (int64_t)ctx->sm_count && !getenv_flag0("SQB_K1_SPLIT")) {
    if (kpl <= 4) return launch_tma_split<T, 4>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
    if (kpl <= 8) return launch_tma_split<T, 8>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
    return launch_tma_split<T, 16>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
  }
  if (g.log_tb == 13) {  // 8-sub-tile leaf groups (standalone geometry, ell <= 256)
    if (kpl <= 4) return launch_tma<T, 4, S, WPB, 13>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
    return launch_tma<T, 8, S, WPB, 13>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
  }
  if (kpl <= 4) return launch_tma<T, 4, S, WPB, 12>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
  if (kpl <= 8) return launch_tma<T, 8, S, WPB, 12>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
  return launch_tma<T, 16, S, WPB, 12>(ctx, sk, g, n_local, e_base, X, ldx, k, sc, P, st);
}

// ---------------------------------------------------------------------------
// 16-bit storage (bf16 / fp16): the same two-pass tile kernel on PACKED pairs.
// Every butterfly op of the reference is one correctly rounded 16-bit op
// (numpy/ml_dtypes round each op once), which add/sub/mul.rn.{bf16,f16}x2
// compute natively two at a time.  Values stay in the 16-bit format in
// shared memory as well (half the traffic of fp32 staging).
// ---------------------------------------------------------------------------
// stages b..b+5 over 64 values packed as v[i] = (x_{2i}, x_{2i+1})
template <typename T>
__device__ __forceinline__ void fwht64_packed(uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = pk_inner<T>(v[i]);
#pragma unroll
  for (int s2 = 0; s2 < 5; ++s2)
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (!(i & (1 << s2))) {
        const uint32_t x = v[i], y = v[i | (1 << s2)];
        v[i] = Pk<T>::add(x, y);
        v[i | (1 << s2)] = Pk<T>::sub(x, y);
      }
}

template <typename T>
__device__ __forceinline__ float h16_to_float(uint16_t h) {
  if constexpr (std::is_same<T, __half>::value) return __half2float(__ushort_as_half(h));
  else return __bfloat162float(__ushort_as_bfloat16(h));
}

template <typename T>
__global__ void __launch_bounds__(S64_NT)
srht64h_tile_kernel(const T* __restrict__ X, int64_t ldx, int64_t n, int64_t n_eff, int64_t k,
                    const uint32_t* __restrict__ bits, const int64_t* __restrict__ idx, int ell,
                    uint32_t scale2, float* __restrict__ P, int64_t n_tiles, const Status* st, int64_t e_base) {
  constexpr int C = 8;  // elements per 16-byte chunk
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* smask = reinterpret_cast<unsigned long long*>(smem_raw);
  int* spre = reinterpret_cast<int*>(smem_raw + 512);
  int* kslot = reinterpret_cast<int*>(smem_raw + 768);
  uint16_t* samp = reinterpret_cast<uint16_t*>(smem_raw + s64_samp_off(ell));
  T* buf = reinterpret_cast<T*>(smem_raw + s64_head_bytes(ell, 2));
  if (st && failed(st)) return;
  const int tid = threadIdx.x;
  s64_sample_maps(idx, ell, smask, spre, kslot);
  const uint32_t mlo = (uint32_t)smask[tid], mhi = (uint32_t)(smask[tid] >> 32);
  const int mypre = spre[tid];
  const int64_t items = n_eff * k;
  auto issue = [&](int64_t item) {
    if (item >= items) return;
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e0 = t << S64_LOG;
    const T* x = X + col * ldx + e0;
    const int64_t nv = n - e0;
    if (nv >= S64_TB) {
      const T* src = x + tid * C;
      T* dst = buf + s64_idx<T>(tid * C);
#pragma unroll
      for (int i = 0; i < S64_TB / (C * S64_NT); ++i)
        cp_async16(dst + i * (S64_NT * C + s64_pad<T>() * C), src + i * S64_NT * C, 16);
    } else {
      for (int q = tid; q < S64_TB / C; q += S64_NT) {
        const int e = q * C;
        const int64_t rem = nv - e;
        const int bytes = rem >= C ? 16 : (rem > 0 ? (int)rem * 2 : 0);
        cp_async16(buf + s64_idx<T>(e), bytes > 0 ? (const void*)(x + e) : (const void*)x, bytes);
      }
    }
  };
  auto sign_words = [&](int64_t item, uint32_t& a0, uint32_t& a1) {
    if (item >= items) return;
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t eg = e_base + (t << S64_LOG) + tid * 64;
    a0 = __ldg(bits + (eg >> 5));
    a1 = __ldg(bits + (eg >> 5) + 1);
  };
  int64_t item = blockIdx.x;
  uint32_t w0 = 0, w1 = 0;
  issue(item);
  cp_async_commit_group();
  sign_words(item, w0, w1);
  for (; item < items; item += gridDim.x) {
    cp_async_wait_group<0>();
    __syncthreads();
    const int64_t col = item / n_eff, t = item - col * n_eff;
    const int64_t e = (t << S64_LOG) + tid * 64;
    uint32_t v[32];
    {
      uint4* row = reinterpret_cast<uint4*>(buf + s64_idx<T>(tid * 64));
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 d = row[q];
        v[4 * q] = d.x; v[4 * q + 1] = d.y; v[4 * q + 2] = d.z; v[4 * q + 3] = d.w;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint32_t w = (i < 16 ? w0 : w1) >> ((2 * i) & 31);
        const uint32_t flip = ((w & 1u) << 15) | ((w & 2u) << 30);
        v[i] = Pk<T>::mul(v[i], scale2) ^ flip;  // fl(x * scale), then the sign
      }
      if (e + 64 > n) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          if (e + 2 * i >= n) v[i] &= 0xffff0000u;
          if (e + 2 * i + 1 >= n) v[i] &= 0x0000ffffu;
        }
      }
      fwht64_packed<T>(v);
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) row[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncthreads();
    // pass 2: coordinates tid + 64 j packed as (j, j+1) pairs
    {
      const uint16_t* col0 = reinterpret_cast<const uint16_t*>(buf) + tid;
      constexpr int RS = 64 + s64_pad<T>();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        v[i] = __byte_perm((uint32_t)col0[(2 * i) * RS], (uint32_t)col0[(2 * i + 1) * RS], 0x5410);
    }
    __syncthreads();  // tile buffer free: stream the next item in behind pass 2
    issue(item + gridDim.x);
    cp_async_commit_group();
    sign_words(item + gridDim.x, w0, w1);
    fwht64_packed<T>(v);
    {
      int slot = mypre;
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if (((j < 32 ? mlo : mhi) & (1u << (j & 31))) != 0u)
          samp[slot++] = (uint16_t)((j & 1) ? (v[j >> 1] >> 16) : (v[j >> 1] & 0xffffu));
    }
    __syncthreads();
    float* leaves = P + (col * n_tiles + t) * ell;
    for (int kk = tid; kk < ell; kk += S64_NT) leaves[kk] = h16_to_float<T>(samp[kslot[kk]]);
  }
  cp_async_wait_group<0>();
}

// ---------------------------------------------------------------------------
// K1 standalone for 16-bit storage: TMA-staged warp tiles on PACKED pairs.
// A warp owns a 4096-coordinate leaf group as two 2048-coordinate
// sub-tiles; lane l holds run l (64 coordinates = 32 bf16x2/f16x2 words, one
// 128-byte swizzled row of the TMA box).  Pass 1: the pair bit and bits 1-5
// in registers.  Pass 2: lane l takes word l (coordinates 2l, 2l+1) of all
// 32 runs, so the five run-bit stages (bits 6-10) act on both halves of
// every word at once.  Bit 11 is one correctly rounded op at the sampled
// coordinates (left operand = sub-tile 0), as in the fp64 kernel.  Every
// butterfly is one add/sub.rn.{bf16,f16}x2 (the reference rounds each op).
// ---------------------------------------------------------------------------
template <typename T, int KPL, int S, int WPB>
__global__ void __launch_bounds__(WPB * 32)
srht_tma16_tile_kernel(const __grid_constant__ CUtensorMap map, const T* __restrict__ X, int64_t ldx, int64_t n,
                       int64_t n_eff, int64_t k, const uint32_t* __restrict__ bits,
                       const int64_t* __restrict__ idx, int ell, uint32_t scale2, float* __restrict__ P,
                       int64_t n_tiles, const Status* st, int64_t e_base) {
  constexpr uint32_t SB = 4096;  // bytes per 2048-coordinate sub-tile
  constexpr int RW = 36;         // transpose-buffer row: 32 words + 16-byte pad
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  if (st && failed(st)) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stages = base + (size_t)wid * S * SB;
  uint32_t* buf = reinterpret_cast<uint32_t*>(base + (size_t)WPB * S * SB) + wid * 32 * RW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)WPB * S * SB + 4 * (size_t)WPB * 32 * RW) + wid * S;
  if (lane == 0)
    for (int s = 0; s < S; ++s) mbar_init(bars + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  // per output k = lane + 32 i: byte offset of its 16-bit value in the
  // transpose buffer (bits 0-15), bit 11 of its in-group position at bit 16
  uint32_t mypk[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int kk = lane + 32 * i;
    const uint32_t p = kk < ell ? (uint32_t)(__ldg(idx + kk) & 4095) : 0u;
    const uint32_t run = (p >> 6) & 31u, pos = p & 63u;
    mypk[i] = ((run * RW + (pos >> 1)) * 4u + (pos & 1u) * 2u) | (((p >> 11) & 1u) << 16);
  }
  const int64_t items = n_eff * k;
  const int64_t nwarps = (int64_t)gridDim.x * WPB;
  const int64_t wg = (int64_t)blockIdx.x * WPB + wid;
  // items wg, wg + nwarps, ...: groups processed at the same time are adjacent,
  // so the 8-byte / 4-byte leaf writes of neighbouring groups meet in L2 and
  // leave as whole sectors (a contiguous range per warp doubled DRAM writes)
  const int64_t my_items = wg < items ? (items - wg + nwarps - 1) / nwarps : 0;
  const int64_t dcol = nwarps / n_eff, dg = nwarps - dcol * n_eff;
  const int64_t units = my_items * 2;  // 2048-coordinate sub-tiles of this warp
  struct Cur {  // (column, group, sub-tile) of a unit; advance without division
    int64_t col, g;
    int q;
    __device__ void next(int64_t ne, int64_t dc, int64_t dgg) {
      if (++q == 2) {
        q = 0;
        g += dgg;
        col += dc;
        if (g >= ne) { g -= ne; ++col; }
      }
    }
    __device__ int64_t e0() const { return (g << 12) + ((int64_t)q << 11); }
  };
  Cur cu{wg / n_eff, wg % n_eff, 0};
  Cur ci = cu, cw = cu;
  auto issue = [&](int64_t u) {  // lane 0 only
    const int64_t e0 = ci.e0();
    if (e0 + 2048 > n) return;
    const int s = (int)(u % S);
    mbar_expect_tx(bars + s, SB);
    tma_load_3d(stages + (size_t)s * SB, &map, 0, (int)(e0 >> 6), (int)ci.col, bars + s);
  };
  if (lane == 0)
    for (int64_t u = 0; u < S && u < units; ++u) { issue(u); ci.next(n_eff, dcol, dg); }
  uint32_t phase = 0;
  uint2 w_next = make_uint2(0u, 0u);
  if (units > 0) w_next = __ldg(reinterpret_cast<const uint2*>(bits + ((e_base + cw.e0() + lane * 64) >> 5)));
  cw.next(n_eff, dcol, dg);
  const uint32_t run_base = (uint32_t)lane * 128u, run_x = ((uint32_t)lane & 7u) << 4;
  float acc[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) acc[i] = 0.f;
  for (int64_t u = 0; u < units; ++u, cu.next(n_eff, dcol, dg)) {
    const int64_t col = cu.col, e0 = cu.e0();
    const int q = cu.q;
    const int s = (int)(u % S);
    const int64_t e = e0 + lane * 64;
    const uint2 w = w_next;
    if (u + 1 < units) w_next = __ldg(reinterpret_cast<const uint2*>(bits + ((e_base + cw.e0() + lane * 64) >> 5)));
    cw.next(n_eff, dcol, dg);
    unsigned char* sb = stages + (size_t)s * SB;
    if (e0 + 2048 <= n) {
      mbar_wait(bars + s, (phase >> s) & 1u);
      phase ^= 1u << s;
    } else {  // column tail: stage it by hand in the same swizzled layout
      const uint16_t* x = reinterpret_cast<const uint16_t*>(X + col * ldx);
#pragma unroll
      for (int j = 0; j < 64; j += 2) {
        const uint32_t lo = (e + j < n) ? x[e + j] : 0u, hi = (e + j + 1 < n) ? x[e + j + 1] : 0u;
        *reinterpret_cast<uint32_t*>(sb + run_base + ((((uint32_t)j * 2u) & ~15u) ^ run_x) + ((j * 2) & 15)) =
            lo | (hi << 16);
      }
      __syncwarp();
    }
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 r = *reinterpret_cast<const uint4*>(sb + run_base + (((uint32_t)c << 4) ^ run_x));
      v[4 * c] = r.x; v[4 * c + 1] = r.y; v[4 * c + 2] = r.z; v[4 * c + 3] = r.w;
    }
    __syncwarp();
    if (lane == 0 && u + S < units) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(u + S);
      ci.next(n_eff, dcol, dg);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {  // fl(x * scale), then the signs (sketching.py:152-153)
      const uint32_t ww = (i < 16 ? w.x : w.y) >> ((2 * i) & 31);
      v[i] = Pk<T>::mul(v[i], scale2) ^ (((ww & 1u) << 15) | ((ww & 2u) << 30));
    }
    if (e + 64 > n) {  // zero padding past n is +0 (sketching.py:154)
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (e + 2 * i >= n) v[i] &= 0xffff0000u;
        if (e + 2 * i + 1 >= n) v[i] &= 0x0000ffffu;
      }
    }
    fwht64_packed<T>(v);  // h = 1..32
    {
      uint4* row = reinterpret_cast<uint4*>(buf + lane * RW);
#pragma unroll
      for (int c = 0; c < 8; ++c) row[c] = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = buf[r * RW + lane];
#pragma unroll
    for (int s2 = 0; s2 < 5; ++s2)  // h = 64..1024 on both halves of each word
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (!(r & (1 << s2))) {
          const uint32_t x = v[r], y = v[r | (1 << s2)];
          v[r] = Pk<T>::add(x, y);
          v[r | (1 << s2)] = Pk<T>::sub(x, y);
        }
#pragma unroll
    for (int r = 0; r < 32; ++r) buf[r * RW + lane] = v[r];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const uint32_t pk = mypk[i];
      const float sv =
          pk_lo_float<T>(*reinterpret_cast<const uint16_t*>(reinterpret_cast<const unsigned char*>(buf) + (pk & 0xffffu)));
      if (q == 0) {
        acc[i] = sv;
      } else {
        const int kk = lane + 32 * i;
        if (kk < ell)
          P[(col * n_tiles + (e0 >> 12)) * ell + kk] = ((pk >> 16) & 1u) ? Lo<T>::sub(acc[i], sv) : Lo<T>::add(acc[i], sv);
      }
    }
    __syncwarp();
  }
}

template <typename T, int KPL, int S, int WPB>
static int launch_tma16(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local, int64_t e_base,
                        const T* X, int64_t ldx, int64_t k, uint32_t scale2, float* P, const Status* st) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return set_error(ctx, SQB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  const cuuint64_t dims[3] = {64, (cuuint64_t)(n_local >> 6), (cuuint64_t)k};
  const cuuint64_t strides[2] = {128, (cuuint64_t)ldx * 2};
  const cuuint32_t box[3] = {64, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(&map, std::is_same<T, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                         3, const_cast<T*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ctx, SQB_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  const size_t smem = 1024 + (size_t)WPB * S * 4096 + 4 * (size_t)WPB * 32 * 36 + (size_t)WPB * S * 8;
  auto kern = srht_tma16_tile_kernel<T, KPL, S, WPB>;
  allow_dyn_smem(kern, (size_t)(smem));
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, smem);
  per_sm = std::max(1, per_sm);
  const int64_t items = g.n_eff * k;
  const int64_t ctas =
      std::max<int64_t>(1, std::min<int64_t>((items + WPB - 1) / WPB, (int64_t)per_sm * ctx->sm_count));
  kern<<<(unsigned)ctas, WPB * 32, smem, ctx->stream>>>(map, X, ldx, n_local, g.n_eff, k, sk->sign_bits,
                                                         sk->indices, (int)sk->ell, scale2, P, g.n_tiles, st, e_base);
  return check_launch(ctx, "srht_tma16_tile_kernel");
}

template <typename T, int S, int WPB>
static int launch_tma16_kpl(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, int64_t n_local,
                            int64_t e_base, const T* X, int64_t ldx, int64_t k, uint32_t scale2, float* P,
                            const Status* st) {
  const int kpl = (int)((sk->ell + 31) / 32);
  if (kpl <= 4) return launch_tma16<T, 4, S, WPB>(ctx, sk, g, n_local, e_base, X, ldx, k, scale2, P, st);
  if (kpl <= 8) return launch_tma16<T, 8, S, WPB>(ctx, sk, g, n_local, e_base, X, ldx, k, scale2, P, st);
  return launch_tma16<T, 16, S, WPB>(ctx, sk, g, n_local, e_base, X, ldx, k, scale2, P, st);
}

// Leaves of the fused column kernel (rhqr_col_kernel) are k-major,
// P[(col ell + k) n_tiles + t]: one warp per output (the row-partitioned
// sweep's rank-local subtree, rhqr_dist.cu).
// group-major leaves, one warp per output with lanes over tiles (strided
// reads): the latency-friendly choice when there are few outputs (a single
// vector: the Arnoldi sketches)
template <typename T>
__global__ void __launch_bounds__(256)
srht_tree_gmw_kernel(const typename Lo<T>::acc* __restrict__ P, int64_t n_tiles, int64_t n_eff,
                     const int64_t* __restrict__ idx, int ell, int log_tb,
                     typename Lo<T>::acc norm_lo, double* __restrict__ Y, int64_t ldy,
                     int64_t row_off, const Status* st, int apply_norm, const T* __restrict__ Xtop = nullptr,
                     int64_t ldxtop = 0, int mtop = 0) {
  if (st && failed(st)) return;
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t col = blockIdx.y;
  {  // a deferred copy of the identity-block rows Y[0:mtop] = X[0:mtop] (defer_copy_top)
    const int gi = blockIdx.x * 256 + threadIdx.x;
    if (Xtop && gi < mtop) Y[gi + col * ldy] = (double)Lo<T>::load(Xtop[gi + col * ldxtop]);
  }
  if (k >= ell) return;
  const int64_t rhi = __ldg(idx + k) >> log_tb;
  const typename Lo<T>::acc v =
      warp_tile_tree<T>(P + col * n_tiles * ell + k, (int)n_tiles, (int)n_eff, rhi, ell);
  if ((threadIdx.x & 31) == 0) Y[row_off + k + col * ldy] = apply_norm ? (double)Lo<T>::mul(v, norm_lo) : (double)v;
}

template <typename T>
__global__ void __launch_bounds__(256)
srht_tree_km_kernel(const typename Lo<T>::acc* __restrict__ P, int64_t n_tiles, int64_t n_eff,
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

// Standalone leaves are GROUP-major, P[(col n_tiles + t) ell + k]: the tile
// kernels write each group's ell leaves as one coalesced run, and here lane
// = output k reads them coalesced.  CTA = 32 outputs x 8 warps; warp w folds
// the aligned tile chunk [w cs, (w+1) cs) with a binary counter (the node of
// height h combines left +- right by bit h of r_hi = idx div TB, left =
// lower tiles; all-padding tiles are exact +0 leaves) — the same binary tree
// as one pass over all tiles — then warp 0 folds the chunk roots.
template <typename T, int NW>
__global__ void __launch_bounds__(NW * 32)
srht_tree_kernel(const typename Lo<T>::acc* __restrict__ P, int64_t n_tiles, int64_t n_eff,
                 const int64_t* __restrict__ idx, int ell, int log_tb,
                 typename Lo<T>::acc norm_lo, double* __restrict__ Y, int64_t ldy,
                 int64_t row_off, const Status* st, int apply_norm) {
  using A = typename Lo<T>::acc;
  __shared__ A roots[NW][32];
  if (st && failed(st)) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + lane;
  const int64_t col = blockIdx.y;
  const int nch = n_tiles >= NW ? NW : (int)n_tiles;
  const int64_t cs = n_tiles / nch;  // power of two
  int lc = 0;
  while ((int64_t(1) << lc) < cs) ++lc;
  const int64_t rhi = k < ell ? (__ldg(idx + k) >> log_tb) : 0;
  if (w < nch) {
    A acc[40];
    const A* pc = P + (col * n_tiles + (int64_t)w * cs) * ell + k;
    const int64_t t0 = (int64_t)w * cs;
    for (int64_t tb = 0; tb < cs; tb += 8) {
      A v8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v8[j] = (k < ell && tb + j < cs && t0 + tb + j < n_eff) ? pc[(tb + j) * ell] : A(0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (tb + j >= cs) break;
        const int64_t tt = tb + j;
        A v = v8[j];
        int h = 0;
        while ((tt >> h) & 1) {
          v = ((rhi >> h) & 1) ? Lo<T>::sub(acc[h], v) : Lo<T>::add(acc[h], v);
          ++h;
        }
        acc[h] = v;
      }
    }
    roots[w][lane] = acc[lc];
  }
  __syncthreads();
  if (w == 0 && k < ell) {
    A r[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) r[q] = q < nch ? roots[q][lane] : A(0);
    int lvl = lc;
    for (int s2 = 1; s2 < nch; s2 <<= 1, ++lvl) {
      const bool neg = (rhi >> lvl) & 1;
#pragma unroll
      for (int q = 0; q < NW; q += 2)
        if ((q % (2 * s2)) == 0 && q + s2 < nch) r[q] = neg ? Lo<T>::sub(r[q], r[q + s2]) : Lo<T>::add(r[q], r[q + s2]);
    }
    Y[row_off + k + col * ldy] = apply_norm ? (double)Lo<T>::mul(r[0], norm_lo) : (double)r[0];
  }
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
// standalone sketches use 4096-coordinate tiles for every dtype (the tile size
// only regroups the same butterflies: any power of two gives the same bits)
// fp64 / fp32 with ell <= 256: 8192-coordinate leaf groups (the TMA warp-tile
// kernel folds 8 sub-tiles at the sampled positions), half the leaves of the
// 4096-coordinate groups for the tile kernel to write and the tree to read
// (bitwise the same sketch).  SQB_K1_G13=0 keeps 4096 (A/B).
// Only with enough groups to fill the GPU ((n_pad / 8192) k >= 2048 warp
// items): halving the items of a single vector or a short matrix costs more
// latency than the leaves save (2^20 x 1: 16.9 -> 19.1 us; 5000 x 3: 15.1 ->
// 21.0 us; 2^20 x 128: 236.9 -> 223.5 us).
static SrhtGeom standalone_geom(const sqb_sketch* sk, int dtype, int64_t k) {
  SrhtGeom g;
  const int lp = ilog2_exact(sk->n_pad);
  g.log_tb = lp < S64_LOG ? lp : S64_LOG;
  if ((dtype == SQB_F64 || dtype == SQB_F32) && sk->ell <= 256 && lp > S64_LOG &&
      (sk->n_pad >> (S64_LOG + 1)) * k >= 2048 && !getenv_flag0("SQB_K1_G13"))
    g.log_tb = S64_LOG + 1;
  g.n_tiles = sk->n_pad >> g.log_tb;
  const int64_t tb = int64_t(1) << g.log_tb;
  g.n_eff = (sk->n + tb - 1) / tb;
  return g;
}

size_t sketch_partials_bytes(const sqb_sketch* sk, int dtype, int64_t k) {
  if (sk->kind != SQB_SKETCH_SRHT) return dense_ws_bytes(sk, dtype, k);
  // room for the standalone geometry and for the fused column kernels' own tiles
  const SrhtGeom g = srht_geom(sk, dtype), g2 = standalone_geom(sk, dtype, k), g12 = standalone_geom(sk, SQB_F16, k);
  return acc_bytes(dtype) * (size_t)sk->ell * (size_t)std::max(std::max(g.n_tiles, g2.n_tiles), g12.n_tiles) * (size_t)k;
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
  if constexpr (sizeof(T) == 2) {
    if (vec && g.log_tb == S64_LOG && (e_base & 63) == 0 && sk->ell <= 512 && n_local >= 64 && encode_tiled()) {
      const T s1 = T((float)sc);  // sc is already a value of T (srht_constants): exact
      uint16_t s16b;
      memcpy(&s16b, &s1, 2);
      const uint32_t s16 = s16b;
      return launch_tma16_kpl<T, 2, 4>(ctx, sk, g, n_local, e_base, (const T*)X, ldx, k, s16 | (s16 << 16),
                                       (float*)P, st);
    }
    if (vec && g.log_tb == S64_LOG && (e_base & 63) == 0 && sk->ell <= S64_MAX_ELL) {
      const size_t smemh = s64_head_bytes((int)sk->ell, 2) + s64_buf_bytes<T>();
      allow_dyn_smem(srht64h_tile_kernel<T>, (size_t)(smemh));
      cudaFuncSetAttribute(srht64h_tile_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srht64h_tile_kernel<T>, S64_NT, smemh);
      per_sm = std::max(1, per_sm);
      const int64_t items = g.n_eff * k;
      const unsigned gp = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)per_sm * ctx->sm_count));
      const T s1 = T((float)sc);  // sc is already a value of T (srht_constants): exact
      uint16_t s16b;
      memcpy(&s16b, &s1, 2);
      const uint32_t s16 = s16b;
      srht64h_tile_kernel<T><<<gp, S64_NT, smemh, ctx->stream>>>((const T*)X, ldx, n_local, g.n_eff, k,
                                                                 sk->sign_bits, sk->indices, (int)sk->ell,
                                                                 s16 | (s16 << 16), (float*)P, g.n_tiles, st, e_base);
      return check_launch(ctx, "srht64h_tile_kernel");
    }
  }
  if constexpr (sizeof(T) >= 4) {
    // TMA-staged warp tiles (ell <= 512: the per-lane output registers)
    const bool tma_geom = g.log_tb == S64_LOG || (g.log_tb == S64_LOG + 1 && sk->ell <= 256);
    if (vec && tma_geom && (e_base & 63) == 0 && sk->ell <= 512 && n_local >= 32 && encode_tiled())
      return launch_tma_kpl<T, 2, 4>(ctx, sk, g, n_local, e_base, (const T*)X, ldx, k, (T)sc, (T*)P, st);
    if (vec && g.log_tb == S64_LOG && (e_base & 63) == 0 && sk->ell <= S64_MAX_ELL) {
      const size_t smem64 = s64_head_bytes((int)sk->ell, sizeof(T)) + s64_buf_bytes<T>();
      allow_dyn_smem(srht64_tile_kernel<T>, (size_t)(smem64));
      cudaFuncSetAttribute(srht64_tile_kernel<T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, srht64_tile_kernel<T>, S64_NT, smem64);
      per_sm = std::max(1, per_sm);
      const int64_t items = g.n_eff * k;
      const unsigned gp = (unsigned)std::max<int64_t>(1, std::min<int64_t>(items, (int64_t)per_sm * ctx->sm_count));
      srht64_tile_kernel<T><<<gp, S64_NT, smem64, ctx->stream>>>((const T*)X, ldx, n_local, g.n_eff, k,
                                                                 sk->sign_bits, sk->indices, (int)sk->ell, (T)sc,
                                                                 (T*)P, g.n_tiles, st, e_base);
      return check_launch(ctx, "srht64_tile_kernel");
    }
  }
  if (vec) {
    auto kern = srht_tile_kernel<T, VN>;
    allow_dyn_smem(kern, (size_t)(smem));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    kern<<<grid, SRHT_NT, smem, ctx->stream>>>((const T*)X, ldx, n_local, g.log_tb, sk->sign_bits,
                                               sk->indices, (int)sk->ell, (A)sc, (A*)P, g.n_tiles, st, e_base);
  } else {
    auto kern = srht_tile_kernel<T, 1>;
    allow_dyn_smem(kern, (size_t)(smem));
    kern<<<grid, SRHT_NT, smem, ctx->stream>>>((const T*)X, ldx, n_local, g.log_tb, sk->sign_bits,
                                               sk->indices, (int)sk->ell, (A)sc, (A*)P, g.n_tiles, st, e_base);
  }
  return check_launch(ctx, "srht_tile_kernel");
}

template <typename T>
static int srht_tiles_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                        void* P, const Status* st) {
  return srht_tiles_geom_t<T>(ctx, sk, standalone_geom(sk, Lo<T>::code, k), sk->n, 0, X, ldx, k, P, st);
}

// group-major tree launch: 8 chunk warps per 32 outputs, or 32 when the
// grid would not fill the GPU (few columns: single-vector Arnoldi sketches)
template <typename T>
static int launch_tree_gm(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, const void* P, int64_t k,
                          double* Y, int64_t ldy, int64_t row_off, typename Lo<T>::acc nm, int apply_norm,
                          const Status* st) {
  using A = typename Lo<T>::acc;
  dim3 grid((unsigned)((sk->ell + 31) / 32), (unsigned)k);
  if (k <= 2 && g.n_tiles <= 65536) {  // warp_tile_tree's chunk stack limit
    dim3 gw((unsigned)((sk->ell + 7) / 8), (unsigned)k);
    const T* xtop = nullptr;
    if (ctx->top_pending && ctx->top_dtype == Lo<T>::code && ctx->top_k == k && ctx->top_Y == Y &&
        ctx->top_ldy == ldy && ctx->top_m <= (int64_t)gw.x * 256 && ctx->top_m <= row_off) {
      xtop = static_cast<const T*>(ctx->top_X);  // the deferred copy_top rides on this launch
      ctx->top_pending = false;
    }
    srht_tree_gmw_kernel<T><<<gw, 256, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                         (int)sk->ell, g.log_tb, nm, Y, ldy, row_off, st, apply_norm,
                                                         xtop, ctx->top_ldx, (int)ctx->top_m);
    return check_launch(ctx, "srht_tree_gmw_kernel");
  }
  if ((int64_t)grid.x * grid.y < 2 * ctx->sm_count && g.n_tiles >= 64)
    srht_tree_kernel<T, 32><<<grid, 1024, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                            (int)sk->ell, g.log_tb, nm, Y, ldy, row_off, st,
                                                            apply_norm);
  else
    srht_tree_kernel<T, 8><<<grid, 256, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                          (int)sk->ell, g.log_tb, nm, Y, ldy, row_off, st,
                                                          apply_norm);
  return check_launch(ctx, "srht_tree_kernel");
}

template <typename T>
static int srht_tree_geom_t(sqb_ctx* ctx, const sqb_sketch* sk, const SrhtGeom& g, const void* P, int64_t k,
                            double* Y, int64_t ldy, int64_t row_off, int apply_norm, const Status* st,
                            int kmajor) {
  using A = typename Lo<T>::acc;
  double sc, nm;
  srht_constants(sk, Lo<T>::code, &sc, &nm);
  if (kmajor) {
    dim3 gk((unsigned)((sk->ell + 7) / 8), (unsigned)k);
    srht_tree_km_kernel<T><<<gk, 256, 0, ctx->stream>>>((const A*)P, g.n_tiles, g.n_eff, sk->indices,
                                                        (int)sk->ell, g.log_tb, (A)nm, Y, ldy, row_off, st,
                                                        apply_norm);
    return check_launch(ctx, "srht_tree_km_kernel");
  }
  return launch_tree_gm<T>(ctx, sk, g, P, k, Y, ldy, row_off, (A)nm, apply_norm, st);
}

template <typename T>
static int srht_tree_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* P, int64_t k, double* Y,
                       int64_t ldy, int64_t row_off, const Status* st) {
  using A = typename Lo<T>::acc;
  const SrhtGeom g = standalone_geom(sk, Lo<T>::code, k);
  double sc, nm;
  srht_constants(sk, Lo<T>::code, &sc, &nm);
  return launch_tree_gm<T>(ctx, sk, g, P, k, Y, ldy, row_off, (A)nm, 1, st);
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
                          int64_t k, double* Y, int64_t ldy, int64_t row_off, int apply_norm, const Status* st,
                          int kmajor) {
  SQB_DISPATCH(dtype, srht_tree_geom_t, ctx, sk, g, P, k, Y, ldy, row_off, apply_norm, st, kmajor);
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

// Y[0:m, :k] = X[0:m, :k] deferred until the sketch that follows: a single-vector SRHT tree launch
// (srht_tree_gmw_kernel) performs it; flush_copy_top launches copy_top_kernel if nothing took it
void defer_copy_top(sqb_ctx* ctx, int dtype, const void* X, int64_t ldx, int64_t m, int64_t k, double* Y, int64_t ldy) {
  ctx->top_pending = m > 0 && k > 0;
  ctx->top_dtype = dtype; ctx->top_X = X; ctx->top_ldx = ldx; ctx->top_m = m; ctx->top_k = k; ctx->top_Y = Y;
  ctx->top_ldy = ldy;
}
int flush_copy_top(sqb_ctx* ctx, const Status* st) {
  if (!ctx->top_pending) return SQB_OK;
  ctx->top_pending = false;
  return launch_copy_top(ctx, ctx->top_dtype, ctx->top_X, ctx->top_ldx, ctx->top_m, ctx->top_k, ctx->top_Y,
                         ctx->top_ldy, st);
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

template <typename T>
static int resketch_head_t(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t upto,
                           double* Y, int64_t ldy, int64_t row_off, void* partials, const Status* st) {
  if (sk->kind != SQB_SKETCH_SRHT || getenv_flag0("SQB_RESKETCH_HEAD"))
    return sketch_t<T>(ctx, sk, X, ldx, 1, Y, ldy, row_off, partials, st);
  SrhtGeom g = standalone_geom(sk, Lo<T>::code, 1);
  const int64_t tb = int64_t(1) << g.log_tb;
  if (upto > tb) return sketch_t<T>(ctx, sk, X, ldx, 1, Y, ldy, row_off, partials, st);
  SrhtGeom g0 = g;
  g0.n_eff = 1;  // tile 0 only; leaves stay at their (col 0, tile 0) slots of the full geometry
  SQB_TRY(srht_tiles_geom_t<T>(ctx, sk, g0, std::min<int64_t>(sk->n, tb), 0, X, ldx, 1, partials, st));
  return srht_tree_t<T>(ctx, sk, partials, 1, Y, ldy, row_off, st);
}

int launch_sketch_resketch_head(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* X, int64_t ldx,
                                int64_t upto, double* Y, int64_t ldy, int64_t y_row_off, void* partials,
                                const Status* st) {
  SQB_DISPATCH(dtype, resketch_head_t, ctx, sk, X, ldx, upto, Y, ldy, y_row_off, partials, st);
}

}  // namespace sqb
