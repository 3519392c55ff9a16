// Streaming-read microbenchmark for the rhqr_col_kernel access pattern:
// CTA b reads segment b of every column of a column-major matrix
// (SEG bytes per column per CTA, column stride = n_cta * SEG) and reduces it.
// Compares register-pipelined LDG.128, TMA bulk copies into an mbarrier ring
// and cp.async (LDGSTS) into a shared ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ double fold(uint4 v) {
  return __hiloint2double(v.y, v.x) + __hiloint2double(v.w, v.z);
}

// A: every thread keeps D columns of 16-byte vectors in flight
template <int NV, int D>
__global__ void __launch_bounds__(256) k_ldg(const char* U, int64_t ld, int K, double* out) {
  const char* base = U + (int64_t)blockIdx.x * (NV * 256 * 16);
  double acc = 0;
  uint4 x[D][NV];
#pragma unroll
  for (int d = 0; d < D; ++d)
#pragma unroll
    for (int v = 0; v < NV; ++v) x[d][v] = ldg_stream(base + (int64_t)d * ld + (v * 256 + threadIdx.x) * 16);
  for (int k = 0; k < K; k += D) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
#pragma unroll
      for (int v = 0; v < NV; ++v) acc += fold(x[d][v]);
      if (k + d + D < K) {
#pragma unroll
        for (int v = 0; v < NV; ++v) x[d][v] = ldg_stream(base + (int64_t)(k + d + D) * ld + (v * 256 + threadIdx.x) * 16);
      }
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// B: TMA bulk copies, nst stages of SEG bytes, split into `pieces` copies each
__global__ void __launch_bounds__(256) k_tma(const char* U, int64_t ld, int K, int seg, int nst, int pieces, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 16;
  unsigned char* ring = sm + 256;
  const char* base = U + (int64_t)blockIdx.x * seg;
  auto issue = [&](int k, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(seg) : "memory");
    const int pb = seg / pieces;
    for (int p = 0; p < pieces; ++p)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(ring + s * seg + p * pb)), "l"(base + (int64_t)k * ld + p * pb), "r"(pb), "r"(sa(&full[s])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int s = 0; s < nst && s < K; ++s) issue(s, s);
  }
  __syncthreads();
  double acc = 0;
  const int nv = seg / (256 * 16);
  for (int k = 0; k < K; ++k) {
    const int s = k % nst;
    const unsigned ph = (k / nst) & 1;
    asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(sa(&full[s])), "r"(ph) : "memory");
    const uint4* sg = (const uint4*)(ring + s * seg);
    for (int v = 0; v < nv; ++v) acc += fold(sg[v * 256 + threadIdx.x]);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    if (threadIdx.x == 0 && k >= 1 && k - 1 + nst < K) {
      const int ps = (k - 1) % nst;
      asm volatile("{ .reg .pred P; W2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W2; }" ::"r"(sa(&empty[ps])), "r"(((k - 1) / nst) & 1) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k - 1 + nst, ps);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

// C: cp.async 16 B per thread into an NST-stage ring, wait_group NST-1 (thread-private data: no __syncthreads needed,
// each thread reads back only what it copied)
template <int NST>
__global__ void __launch_bounds__(256) k_cpa2(const char* U, int64_t ld, int K, int seg, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const char* base = U + (int64_t)blockIdx.x * seg;
  const int nv = seg / (256 * 16);
  auto issue = [&](int k, int s) {
    for (int v = 0; v < nv; ++v) {
      const int o = (v * 256 + threadIdx.x) * 16;
      asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(sa(sm + s * seg + o)), "l"(base + (int64_t)k * ld + o) : "memory");
    }
  };
  for (int s = 0; s < NST - 1; ++s) {
    if (s < K) issue(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double acc = 0;
  for (int k = 0; k < K; ++k) {
    if (k + NST - 1 < K) issue(k + NST - 1, (k + NST - 1) % NST);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
    const uint4* sg = (const uint4*)(sm + (k % NST) * seg);
    for (int v = 0; v < nv; ++v) acc += fold(sg[v * 256 + threadIdx.x]);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t bytes = 1ll << 30;
  char* U;
  double* out;
  CK(cudaMalloc(&U, bytes + 4096));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(U, 0, bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch, const char* name, int ncta) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    printf("%-44s ncta=%5d  %8.1f GB/s %s\n", name, ncta, bytes * 5 / (ms * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
  };
  char nm[128];
  // tiles of 32 KB (fp64 TB=4096) and 16 KB (bf16 TB=8192)
  for (int seg : {32768, 16384}) {
    for (int ncta : {256, 296, 444, 592, 2048}) {
      const int64_t ld = (int64_t)ncta * seg;
      const int K = (int)(bytes / ld);
      if (seg == 32768) {
        snprintf(nm, sizeof nm, "ldg seg=%d NV=8 D=1", seg);
        timeit([&] { k_ldg<8, 1><<<ncta, 256>>>(U, ld, K, out); }, nm, ncta);
        snprintf(nm, sizeof nm, "ldg seg=%d NV=8 D=2", seg);
        timeit([&] { k_ldg<8, 2><<<ncta, 256>>>(U, ld, K, out); }, nm, ncta);
      } else {
        snprintf(nm, sizeof nm, "ldg seg=%d NV=4 D=1", seg);
        timeit([&] { k_ldg<4, 1><<<ncta, 256>>>(U, ld, K, out); }, nm, ncta);
        snprintf(nm, sizeof nm, "ldg seg=%d NV=4 D=2", seg);
        timeit([&] { k_ldg<4, 2><<<ncta, 256>>>(U, ld, K, out); }, nm, ncta);
        snprintf(nm, sizeof nm, "ldg seg=%d NV=4 D=4", seg);
        timeit([&] { k_ldg<4, 4><<<ncta, 256>>>(U, ld, K, out); }, nm, ncta);
      }
      for (int nst : {2, 3, 6}) {
        if ((size_t)nst * seg > 200 * 1024) continue;
        const size_t smem = 256 + (size_t)nst * seg;
        cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int pieces : {1, 8}) {
          snprintf(nm, sizeof nm, "tma seg=%d nst=%d pieces=%d", seg, nst, pieces);
          timeit([&] { k_tma<<<ncta, 256, smem>>>(U, ld, K, seg, nst, pieces, out); }, nm, ncta);
        }
      }
      {
        const size_t smem = 3 * (size_t)seg;
        cudaFuncSetAttribute(k_cpa2<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        snprintf(nm, sizeof nm, "cp.async seg=%d nst=3", seg);
        timeit([&] { k_cpa2<3><<<ncta, 256, smem>>>(U, ld, K, seg, out); }, nm, ncta);
      }
    }
  }
  return 0;
}
