// K1 — subsampled randomized Hadamard transform, bit-exact with the reference.
//
// Reference: SRHTSketch._apply (sketching.py:149-155) + fwht (:21-43):
//   work = fl(x * dtype(scale)); work *= signs; pad with zeros to n_pad;
//   butterfly stages h = 1, 2, 4, ... n_pad/2 with (a+b, a-b) on (i, i+h);
//   multiply by dtype(n_pad^-1/2); gather rows `indices` in order.
//
// B200 decomposition (CPU replay in tests/test_tile_tree_design.py):
//   * the padded vector is cut into tiles of TB = 2^t consecutive Omega
//     coordinates; one CTA streams one tile (coalesced 128-bit loads) into
//     shared memory and runs the stages h = 1..TB/2 IN ORDER as radix-8
//     register passes (3 stages per pass, one smem round trip per pass);
//   * from each tile only the ell sampled rows r_lo = idx mod TB are kept
//     (a "leaf" per output);
//   * the remaining log2(n_pad/TB) stages only ever touch the sampled rows:
//     output k is the binary tree over tiles, level l combining adjacent
//     subtrees as (left + right) or (left - right) by bit l of
//     r_hi = idx div TB, left = lower tile.  Tiles wholly inside the zero
//     padding contribute exact +0 leaves.
//   Every add/sub/mul is an explicit round-to-nearest intrinsic (no FMA
//   contraction), so the result is bitwise identical to the reference.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace sqb {

constexpr int SRHT_NT = 256;  // threads per tile CTA

template <typename T> struct TileCfg;
template <> struct TileCfg<double> { static constexpr int LOG_TB = 12; };  // 32 KB smem
template <> struct TileCfg<float> { static constexpr int LOG_TB = 13; };
template <> struct TileCfg<__nv_bfloat16> { static constexpr int LOG_TB = 13; };
template <> struct TileCfg<__half> { static constexpr int LOG_TB = 13; };

// shared-memory padding: one spare slot every 16 doubles / 8 floats keeps the
// radix-8 passes at the minimum number of wavefronts
template <typename A> struct Pad;
template <> struct Pad<double> { static constexpr int shift = 4; };
template <> struct Pad<float> { static constexpr int shift = 3; };

template <typename A>
__device__ __forceinline__ int pidx(int e) { return e + (e >> Pad<A>::shift); }

template <typename A>
__host__ __device__ constexpr size_t tile_smem_bytes(int tb) {
  return sizeof(A) * (size_t)(tb + (tb >> Pad<A>::shift) + 1);
}

// one radix-2^R pass over bits [b, b+R) of the in-tile index; `len` = number
// of transformed elements (the tile, or n_pad if that is smaller)
template <typename T, int R>
__device__ __forceinline__ void fwht_pass(typename Lo<T>::acc* sm, int b, int len) {
  using A = typename Lo<T>::acc;
  const int groups = len >> R;
  const int lowmask = (1 << b) - 1;
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    const int base = (g & lowmask) | ((g >> b) << (b + R));
    A v[1 << R];
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) v[j] = sm[pidx<A>(base | (j << b))];
#pragma unroll
    for (int s = 0; s < R; ++s) {
#pragma unroll
      for (int j = 0; j < (1 << R); ++j) {
        if (!(j & (1 << s))) {
          const A x = v[j], y = v[j | (1 << s)];
          v[j] = Lo<T>::add(x, y);
          v[j | (1 << s)] = Lo<T>::sub(x, y);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) sm[pidx<A>(base | (j << b))] = v[j];
  }
}

// in-tile FWHT stages h = 2^b0 .. len/2 in order as radix-16 passes (one smem
// round trip per 4 stages); caller has synced
template <typename T>
__device__ __forceinline__ void tile_fwht_from(typename Lo<T>::acc* sm, int b0, int log_len) {
  const int len = 1 << log_len;
  for (int b = b0; b < log_len; b += 4) {
    const int r = log_len - b;
    if (r >= 4) fwht_pass<T, 4>(sm, b, len);
    else if (r == 3) fwht_pass<T, 3>(sm, b, len);
    else if (r == 2) fwht_pass<T, 2>(sm, b, len);
    else fwht_pass<T, 1>(sm, b, len);
    __syncthreads();
  }
}

// full in-tile FWHT (stages h = 1 .. len/2 in order)
template <typename T>
__device__ __forceinline__ void tile_fwht(typename Lo<T>::acc* sm, int log_len) {
  tile_fwht_from<T>(sm, 0, log_len);
}

// stages h = 1, 2, 4, 8 on 16 consecutive elements held in registers
template <typename T>
__device__ __forceinline__ void reg_fwht16(typename Lo<T>::acc* v) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (!(j & (1 << s))) {
        const typename Lo<T>::acc x = v[j], y = v[j | (1 << s)];
        v[j] = Lo<T>::add(x, y);
        v[j | (1 << s)] = Lo<T>::sub(x, y);
      }
    }
  }
}

__device__ __forceinline__ bool sign_neg(const uint32_t* bits, int64_t e) {
  return (__ldg(bits + (e >> 5)) >> (e & 31)) & 1u;
}

// x -> fl(fl(x * scale) * sign)  (sketching.py:152-153)
template <typename T>
__device__ __forceinline__ typename Lo<T>::acc srht_in(typename Lo<T>::acc x,
                                                      typename Lo<T>::acc scale, bool neg) {
  const typename Lo<T>::acc v = Lo<T>::mul(x, scale);
  return neg ? -v : v;
}

// gather the sampled rows of a transformed tile into leaves P[k * ldp]
template <typename T>
__device__ __forceinline__ void tile_gather(const typename Lo<T>::acc* sm, const int64_t* idx,
                                            int ell, int log_tb, typename Lo<T>::acc* P,
                                            int64_t ldp) {
  using A = typename Lo<T>::acc;
  const int64_t mask = (int64_t(1) << log_tb) - 1;
  for (int k = threadIdx.x; k < ell; k += blockDim.x)
    P[k * ldp] = sm[pidx<A>((int)(__ldg(idx + k) & mask))];
}

// ---------------------------------------------------------------------------
// Packed 16-bit arithmetic (bf16 / fp16 storage).  Every butterfly op of the
// reference is one correctly rounded 16-bit op (numpy/ml_dtypes round each
// op once), which add/sub/mul.rn.{bf16,f16}x2 compute natively two at a time.
// ---------------------------------------------------------------------------
template <typename T> struct Pk;
template <> struct Pk<__nv_bfloat16> {
  __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) {
    uint32_t r; asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
  __device__ __forceinline__ static uint32_t sub(uint32_t a, uint32_t b) {
    uint32_t r; asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
  __device__ __forceinline__ static uint32_t mul(uint32_t a, uint32_t b) {
    uint32_t r; asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
};
template <> struct Pk<__half> {
  __device__ __forceinline__ static uint32_t add(uint32_t a, uint32_t b) {
    uint32_t r; asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
  __device__ __forceinline__ static uint32_t sub(uint32_t a, uint32_t b) {
    uint32_t r; asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
  __device__ __forceinline__ static uint32_t mul(uint32_t a, uint32_t b) {
    uint32_t r; asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
  }
};

// stage on the two halves of each register: (x, y) -> (x + y, x - y)
template <typename T>
__device__ __forceinline__ uint32_t pk_inner(uint32_t r) {
  const uint32_t sw = __byte_perm(r, 0, 0x1032);
  const uint32_t sm = Pk<T>::add(r, sw), df = Pk<T>::sub(r, sw);
  return __byte_perm(sm, df, 0x5410);  // (sm.lo, df.lo)
}

// exact pack of two values already representable in T (lo -> low half)
template <typename T>
__device__ __forceinline__ uint32_t pk_pack(float lo, float hi) {
  if constexpr (std::is_same<T, __half>::value) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

template <typename T>
__device__ __forceinline__ float pk_lo_float(uint16_t h) {
  if constexpr (std::is_same<T, __half>::value) return __half2float(__ushort_as_half(h));
  else return __bfloat162float(__ushort_as_bfloat16(h));
}

// stages over 32 values packed as v[i] = (x_{2i}, x_{2i+1}): the pair bit
// first, then bits 1..4 of i, in order
template <typename T>
__device__ __forceinline__ void fwht32_packed(uint32_t (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = pk_inner<T>(v[i]);
#pragma unroll
  for (int s2 = 0; s2 < 4; ++s2)
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (!(i & (1 << s2))) {
        const uint32_t x = v[i], y = v[i | (1 << s2)];
        v[i] = Pk<T>::add(x, y);
        v[i | (1 << s2)] = Pk<T>::sub(x, y);
      }
}

// ---------------------------------------------------------------------------
// In-tile FWHT of the column pass for 16-bit storage: a 2^13 tile held as
// 16-bit values in shared memory (one 8-element pad per 256), 256 threads.
//   p16_run_in   a run of 8 consecutive coordinates from registers: scale,
//                sign, zero past the data, stages h = 1, 2, 4, one 16-byte store
//   p16_pass     5 stages (bits b..b+4) with 32 values per thread in registers
// Stage order is the reference's (h = 1, 2, 4, ...), so leaves are bitwise
// those of the fp32-staged path.
// ---------------------------------------------------------------------------
constexpr int P16_LOG = 13;
__device__ __forceinline__ int p16(int e) { return e + ((e >> 8) << 3); }

template <typename T>
__device__ __forceinline__ void p16_run_in(uint16_t* sm, int i, const float* x, uint32_t scale2, uint32_t sb,
                                           int valid) {
  uint32_t p[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    p[q] = pk_pack<T>(x[2 * q], x[2 * q + 1]);
    const uint32_t flip = (((sb >> (2 * q)) & 1u) << 15) | (((sb >> (2 * q + 1)) & 1u) << 31);
    p[q] = Pk<T>::mul(p[q], scale2) ^ flip;  // fl(x * scale), then the sign (sketching.py:152-153)
  }
  if (valid < 8) {  // zero padding past n is +0 (sketching.py:154)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (2 * q >= valid) p[q] &= 0xffff0000u;
      if (2 * q + 1 >= valid) p[q] &= 0x0000ffffu;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) p[q] = pk_inner<T>(p[q]);  // h = 1
#pragma unroll
  for (int s2 = 0; s2 < 2; ++s2)  // h = 2, 4
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (!(q & (1 << s2))) {
        const uint32_t x0 = p[q], y0 = p[q | (1 << s2)];
        p[q] = Pk<T>::add(x0, y0);
        p[q | (1 << s2)] = Pk<T>::sub(x0, y0);
      }
  *reinterpret_cast<uint4*>(sm + p16(i)) = make_uint4(p[0], p[1], p[2], p[3]);
}

// bits 3..7 (pass A) and 8..12 (pass B) of the in-tile coordinate
template <typename T>
__device__ __forceinline__ void p16_passes(uint16_t* sm) {
  const int t = threadIdx.x;
  {
    // thread t: coordinates (t & 7) + 8 j + 256 (t >> 3), j = 0..31
    uint16_t* base = sm + (t & 7) + 264 * (t >> 3);
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __byte_perm((uint32_t)base[16 * i], (uint32_t)base[16 * i + 8], 0x5410);
    fwht32_packed<T>(v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      base[16 * i] = (uint16_t)(v[i] & 0xffffu);
      base[16 * i + 8] = (uint16_t)(v[i] >> 16);
    }
  }
  __syncthreads();
  {
    // thread t: coordinates t + 256 j
    uint16_t* base = sm + t;
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __byte_perm((uint32_t)base[528 * i], (uint32_t)base[528 * i + 264], 0x5410);
    fwht32_packed<T>(v);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      base[528 * i] = (uint16_t)(v[i] & 0xffffu);
      base[528 * i + 264] = (uint16_t)(v[i] >> 16);
    }
  }
  __syncthreads();
}

// Tree over tile leaves for output k, done by one warp.  leaves[t] for
// t < n_eff, +0 for n_eff <= t < n_tiles (all-padding tiles).  The warp walks
// the leaves in CHUNKS of 32*R consecutive tiles (R = 8, or fewer for small
// n_tiles), one coalesced run per chunk, loaded one chunk ahead: lane L holds
// the R tiles [L*R, (L+1)*R) of the chunk (levels 0..log2 R - 1 in registers),
// the next 5 levels are lane shuffles, and the chunk values are combined by a
// binary-counter stack with static register indices — every level in order,
// lower tile range as the left operand.  Supports up to 256 chunks
// (n_tiles <= 65536).  `stride`: distance between consecutive tiles' leaves.
// Global leaves are read with L1-bypassing loads: they are produced by other
// CTAs (a previous kernel, or the same persistent grid before a grid
// barrier); SMEM = true reads a shared-memory copy.
template <typename A, bool SMEM>
__device__ __forceinline__ A tree_leaf(const A* p) {
  if constexpr (SMEM) return *p;
  else return __ldcg(p);
}

template <typename T, bool SMEM = false>
__device__ __forceinline__ typename Lo<T>::acc warp_tile_tree(const typename Lo<T>::acc* leaves,
                                                              int n_tiles, int n_eff, int64_t rhi,
                                                              int64_t stride = 1) {
  using A = typename Lo<T>::acc;
  const int lane = threadIdx.x & 31;
  const int lanes = n_tiles >= 32 ? 32 : n_tiles;                    // lanes holding tiles
  const int R = n_tiles >= 256 ? 8 : (n_tiles >= 32 ? (n_tiles >> 5) : 1);
  int lr = 0;
  while ((1 << lr) < R) ++lr;
  int ll = 0;
  while ((1 << ll) < lanes) ++ll;
  const int csz = lanes * R;            // tiles per chunk
  const int nq = n_tiles / csz;         // chunks
  A stk[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) stk[l] = A(0);
  A nx[8];
  const int tl = lane * R;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) nx[jj] = (lane < lanes && jj < R && tl + jj < n_eff) ? tree_leaf<A, SMEM>(leaves + (tl + jj) * stride) : A(0);
  for (int q = 0; q < nq; ++q) {
    A v[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) v[jj] = nx[jj];
    if (q + 1 < nq) {
      const int tb = (q + 1) * csz + tl;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) nx[jj] = (lane < lanes && jj < R && tb + jj < n_eff) ? tree_leaf<A, SMEM>(leaves + (tb + jj) * stride) : A(0);
    }
    // levels 0 .. lr-1 inside the lane
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if ((1 << l) < R) {
        const bool neg = (rhi >> l) & 1;
#pragma unroll
        for (int jj = 0; jj < 8; jj += (2 << l))
          if (jj + (1 << l) < R)
            v[jj] = neg ? Lo<T>::sub(v[jj], v[jj + (1 << l)]) : Lo<T>::add(v[jj], v[jj + (1 << l)]);
      }
    }
    // levels lr .. lr+ll-1 across lanes
    A lv = v[0];
    for (int l = 0; l < ll; ++l) {
      const A o = __shfl_xor_sync(0xffffffffu, lv, 1 << l);
      const bool upper = (lane >> l) & 1;
      const A a = upper ? o : lv, b = upper ? lv : o;
      lv = ((rhi >> (lr + l)) & 1) ? Lo<T>::sub(a, b) : Lo<T>::add(a, b);
    }
    A cv = __shfl_sync(0xffffffffu, lv, 0);
    // levels lr+ll+l across chunks: binary counter
    bool open = true;
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      if (open) {
        if ((q >> l) & 1) {
          cv = ((rhi >> (lr + ll + l)) & 1) ? Lo<T>::sub(stk[l], cv) : Lo<T>::add(stk[l], cv);
        } else {
          stk[l] = cv;
          open = false;
        }
      }
    }
  }
  int top = 0;
  while ((1 << top) < nq) ++top;
  A out = stk[0];
#pragma unroll
  for (int l = 1; l < 8; ++l)
    if (l == top) out = stk[l];
  return out;
}

}  // namespace sqb
