// Shared definitions for the sm_100a RHQR library.
//
// Storage model: every n-dimensional operand
// (W, U, X, Krylov vectors) is COLUMN-MAJOR on the device — column j starts at
// base + j*ld and its rows are contiguous — so one column is one coalesced
// stream.  Sketch-space objects (S, T, R, coefficients, scalars) are fp64.
// The reference's arrays are C-order numpy; the facade converts once at the
// boundary.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/sketchqr_b200.h"

namespace sqb {

// ---------------------------------------------------------------------------
// low-precision storage types.  The reference's emulation model
// (precision.py:1-7) rounds every elementary op to the storage format.  For
// bf16/fp16 we compute each op in fp32 and round once: fp32 carries
// >= 2p+2 bits for p in {8, 11}, so the double rounding is innocuous and the
// result equals the correctly rounded op (what numpy / ml_dtypes do).
// ---------------------------------------------------------------------------
template <typename T> struct Lo;

template <> struct Lo<double> {
  using acc = double;                       // butterfly / GEMV arithmetic type
  static constexpr int code = SQB_F64;
  __device__ __forceinline__ static acc load(double v) { return v; }
  __device__ __forceinline__ static double store(acc v) { return v; }
  __device__ __forceinline__ static acc rnd(acc v) { return v; }
  // float64 -> storage exactly as numpy astype does it
  __device__ __forceinline__ static acc from_double(double v) { return v; }
  __device__ __forceinline__ static acc add(acc a, acc b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static acc sub(acc a, acc b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static acc mul(acc a, acc b) { return __dmul_rn(a, b); }
};

template <> struct Lo<float> {
  using acc = float;
  static constexpr int code = SQB_F32;
  __device__ __forceinline__ static acc load(float v) { return v; }
  __device__ __forceinline__ static float store(acc v) { return v; }
  __device__ __forceinline__ static acc rnd(acc v) { return v; }
  __device__ __forceinline__ static acc from_double(double v) { return __double2float_rn(v); }
  __device__ __forceinline__ static acc add(acc a, acc b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static acc sub(acc a, acc b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static acc mul(acc a, acc b) { return __fmul_rn(a, b); }
};

template <> struct Lo<__nv_bfloat16> {
  using acc = float;
  static constexpr int code = SQB_BF16;
  __device__ __forceinline__ static acc load(__nv_bfloat16 v) { return __bfloat162float(v); }
  __device__ __forceinline__ static __nv_bfloat16 store(acc v) { return __float2bfloat16_rn(v); }
  __device__ __forceinline__ static acc rnd(acc v) { return __bfloat162float(__float2bfloat16_rn(v)); }
  // ml_dtypes converts float64 -> bfloat16 through float32 (two RN steps)
  __device__ __forceinline__ static acc from_double(double v) { return rnd(__double2float_rn(v)); }
  __device__ __forceinline__ static acc add(acc a, acc b) { return rnd(__fadd_rn(a, b)); }
  __device__ __forceinline__ static acc sub(acc a, acc b) { return rnd(__fsub_rn(a, b)); }
  __device__ __forceinline__ static acc mul(acc a, acc b) { return rnd(__fmul_rn(a, b)); }
};

template <> struct Lo<__half> {
  using acc = float;
  static constexpr int code = SQB_F16;
  __device__ __forceinline__ static acc load(__half v) { return __half2float(v); }
  __device__ __forceinline__ static __half store(acc v) { return __float2half_rn(v); }
  __device__ __forceinline__ static acc rnd(acc v) { return __half2float(__float2half_rn(v)); }
  // numpy converts float64 -> float16 directly (one RN step)
  __device__ __forceinline__ static acc from_double(double v) { return __half2float(__double2half(v)); }
  __device__ __forceinline__ static acc add(acc a, acc b) { return rnd(__fadd_rn(a, b)); }
  __device__ __forceinline__ static acc sub(acc a, acc b) { return rnd(__fsub_rn(a, b)); }
  __device__ __forceinline__ static acc mul(acc a, acc b) { return rnd(__fmul_rn(a, b)); }
};

// ---------------------------------------------------------------------------
// device status word shared by every kernel of one call chain: once a kernel
// records a breakdown the rest of the chain becomes a no-op (the reference
// raises at the failing column, rhqr.py:73-79).
// ---------------------------------------------------------------------------
struct Status {
  int code;   // SQB_OK or SQB_ERR_*
  int col;    // 1-based column for breakdowns
  double val; // diagnostic value (rho, diagonal entry, ...)
};

// internal status: the Krylov space closed (happy breakdown), krylov.py:115-125
constexpr int SQB_CLOSED = 100;

__device__ __forceinline__ bool failed(const Status* st) {
  return *((volatile const int*)&st->code) != SQB_OK;
}

__device__ __forceinline__ void fail(Status* st, int code, int col, double val) {
  if (atomicCAS(&st->code, SQB_OK, code) == SQB_OK) {
    st->col = col;
    st->val = val;
  }
}

// warp / block reductions (fp64)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// dot(a[lo:hi], b[lo:hi]) by one warp (all lanes get it): lanes stride the
// range with four independent accumulators, so four loads per lane are in
// flight (the sketch-space dots are L2-latency bound, not bandwidth bound)
__device__ __forceinline__ double warp_dot(const double* a, const double* b, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
  int i = lo + lane;
  for (; i + 96 < hi; i += 128) {
    d0 = fma(a[i], b[i], d0);
    d1 = fma(a[i + 32], b[i + 32], d1);
    d2 = fma(a[i + 64], b[i + 64], d2);
    d3 = fma(a[i + 96], b[i + 96], d3);
  }
  for (; i < hi; i += 32) d0 = fma(a[i], b[i], d0);
  return warp_sum((d0 + d1) + (d2 + d3));
}

// the same with a strided first operand: sum_i a[i * sa] b[i]
__device__ __forceinline__ double warp_dot_strided(const double* a, int64_t sa, const double* b, int lo, int hi) {
  const int lane = threadIdx.x & 31;
  double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
  int i = lo + lane;
  for (; i + 96 < hi; i += 128) {
    d0 = fma(a[(int64_t)i * sa], b[i], d0);
    d1 = fma(a[(int64_t)(i + 32) * sa], b[i + 32], d1);
    d2 = fma(a[(int64_t)(i + 64) * sa], b[i + 64], d2);
    d3 = fma(a[(int64_t)(i + 96) * sa], b[i + 96], d3);
  }
  for (; i < hi; i += 32) d0 = fma(a[(int64_t)i * sa], b[i], d0);
  return warp_sum((d0 + d1) + (d2 + d3));
}

// block-wide sum; `red` must hold >= 32 doubles; all threads get the result
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < nw ? red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) red[0] = r;
  }
  __syncthreads();
  r = red[0];
  __syncthreads();
  return r;
}

}  // namespace sqb

#define SQB_CUDA_TRY(expr)                                       \
  do {                                                           \
    cudaError_t e__ = (expr);                                    \
    if (e__ != cudaSuccess) return sqb::set_cuda_error(ctx, e__, #expr, __FILE__, __LINE__); \
  } while (0)
