// 128-bit vector loads/stores of storage-type elements, widened to the
// arithmetic type.
#pragma once

#include "common.cuh"

namespace sqb {

template <typename T> struct VecN { static constexpr int n = 16 / sizeof(T); };

template <typename T>
__device__ __forceinline__ void vload(const T* p, typename Lo<T>::acc* out);

template <>
__device__ __forceinline__ void vload<double>(const double* p, double* out) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  out[0] = v.x;
  out[1] = v.y;
}
template <>
__device__ __forceinline__ void vload<float>(const float* p, float* out) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <>
__device__ __forceinline__ void vload<__nv_bfloat16>(const __nv_bfloat16* p, float* out) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    out[2 * i] = f.x;
    out[2 * i + 1] = f.y;
  }
}
template <>
__device__ __forceinline__ void vload<__half>(const __half* p, float* out) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    out[2 * i] = f.x;
    out[2 * i + 1] = f.y;
  }
}

// values are already representable in T (rounded by the caller)
template <typename T>
__device__ __forceinline__ void vstore(T* p, const typename Lo<T>::acc* in);

template <>
__device__ __forceinline__ void vstore<double>(double* p, const double* in) {
  *reinterpret_cast<double2*>(p) = make_double2(in[0], in[1]);
}
template <>
__device__ __forceinline__ void vstore<float>(float* p, const float* in) {
  *reinterpret_cast<float4*>(p) = make_float4(in[0], in[1], in[2], in[3]);
}
template <>
__device__ __forceinline__ void vstore<__nv_bfloat16>(__nv_bfloat16* p, const float* in) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}
template <>
__device__ __forceinline__ void vstore<__half>(__half* p, const float* in) {
  uint4 v;
  __half2* h = reinterpret_cast<__half2*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(in[2 * i], in[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}

// streaming 128-bit load for data that is read-only during the kernel: no L1
// allocation, 256-byte L2 prefetch granularity
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// 256-bit streaming load (sm_100 LDG.256): one full 32-byte sector per lane,
// so a lane-contiguous run costs one sector request per sector
__device__ __forceinline__ void ldg256_stream(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ void ldg256(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// 128-bit load of data this kernel later overwrites (coherent path, no L1
// allocation)
__device__ __forceinline__ uint4 ldg_l2only(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

template <typename T>
__device__ __forceinline__ void vload_stream(const T* p, typename Lo<T>::acc* out) {
  const uint4 v = ldg_stream(p);
  if constexpr (sizeof(T) == 8) {
    out[0] = __hiloint2double((int)v.y, (int)v.x);
    out[1] = __hiloint2double((int)v.w, (int)v.z);
  } else if constexpr (sizeof(T) == 4) {
    out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
    out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
  } else {
    const T* h = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = Lo<T>::load(h[i]);
  }
}

// widen one raw 128-bit word of storage elements to the arithmetic type
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, typename Lo<T>::acc* out) {
  if constexpr (sizeof(T) == 8) {
    out[0] = __hiloint2double((int)v.y, (int)v.x);
    out[1] = __hiloint2double((int)v.w, (int)v.z);
  } else if constexpr (sizeof(T) == 4) {
    out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
    out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
  } else if constexpr (Lo<T>::code == SQB_BF16) {
    // bf16 -> fp32 is a placement of the 16 bits: low half by a shift, high
    // half by a mask (one integer op per element, no PRMT)
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      out[2 * i] = __uint_as_float(w[i] << 16);
      out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  } else {
    const T* h = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = Lo<T>::load(h[i]);
  }
}

// cp.async (LDGSTS): 16-byte global -> shared copy; src_bytes < 16 zero-fills the rest
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// load VN consecutive elements starting at e (relative to p), zero beyond n
template <typename T, int VN>
__device__ __forceinline__ void load_run(const T* p, int64_t e, int64_t n,
                                         typename Lo<T>::acc* out) {
  if (VN > 1 && e + VN <= n) {
    vload<T>(p + e, out);
  } else {
#pragma unroll
    for (int j = 0; j < VN; ++j) out[j] = (e + j < n) ? Lo<T>::load(p[e + j]) : typename Lo<T>::acc(0);
  }
}

template <typename T, int VN>
__device__ __forceinline__ void store_run(T* p, int64_t e, int64_t n,
                                          const typename Lo<T>::acc* in) {
  if (VN > 1 && e + VN <= n) {
    vstore<T>(p + e, in);
  } else {
#pragma unroll
    for (int j = 0; j < VN; ++j)
      if (e + j < n) p[e + j] = Lo<T>::store(in[j]);
  }
}

}  // namespace sqb
