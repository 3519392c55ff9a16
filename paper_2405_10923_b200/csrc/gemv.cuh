// Streaming tall-skinny GEMV: acc = U[rows, :K] c for a block of rows, the
// bandwidth-bound core of the compact-form update (rhqr.py:118) and of the
// Arnoldi basis vector q = e_j - U_j coef (krylov.py:137).  Each thread owns
// NV runs of VN consecutive rows (one 128-bit load per run and column, runs
// coalesced across the block); columns are software-pipelined one ahead so
// 2*NV loads are in flight per thread.
#pragma once

#include "vec.cuh"

namespace sqb {

constexpr int GEMV_NT = 256;

template <typename T, int NV>
__device__ __forceinline__ void gemv_rows(const T* __restrict__ U, int64_t ldu, int64_t r0, int64_t n, int K,
                                          const typename Lo<T>::acc* c, typename Lo<T>::acc (&acc)[NV][VecN<T>::n]) {
  using A = typename Lo<T>::acc;
  constexpr int VN = VecN<T>::n;
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < VN; ++j) acc[v][j] = A(0);
  const bool full = r0 + (int64_t)GEMV_NT * NV * VN <= n;
  if (full) {
    A x0[NV][VN], x1[NV][VN];
    auto ld = [&](A (&x)[NV][VN], int k) {
      const T* col = U + r0 + (int64_t)k * ldu;
#pragma unroll
      for (int v = 0; v < NV; ++v) vload_stream<T>(col + (v * GEMV_NT + threadIdx.x) * VN, x[v]);
    };
    auto fm = [&](A (&x)[NV][VN], int k) {
      const A ck = c[k];
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(x[v][j], ck, acc[v][j]);
    };
    if (K > 0) ld(x0, 0);
    int k = 0;
    for (; k + 2 <= K; k += 2) {
      ld(x1, k + 1);
      fm(x0, k);
      if (k + 2 < K) ld(x0, k + 2);
      fm(x1, k + 1);
    }
    if (k < K) fm(x0, k);
  } else if ((n - r0) % VN == 0) {
    // partial last block made of whole 16-byte runs: the same pipeline with
    // the runs past n masked (the generic loop below waits for every column
    // before it issues the next one — one block then outlasts the others)
    const int64_t rows = n - r0;
    uint4 y0[NV], y1[NV];
    auto ldp = [&](uint4 (&x)[NV], int k) {
      const T* col = U + r0 + (int64_t)k * ldu;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int64_t i = (int64_t)(v * GEMV_NT + threadIdx.x) * VN;
        x[v] = i < rows ? ldg_stream(col + i) : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto fmp = [&](const uint4 (&x)[NV], int k) {
      const A ck = c[k];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        A w[VN];
        unpack16<T>(x[v], w);
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(w[j], ck, acc[v][j]);
      }
    };
    if (K > 0) ldp(y0, 0);
    int k = 0;
    for (; k + 2 <= K; k += 2) {
      ldp(y1, k + 1);
      fmp(y0, k);
      if (k + 2 < K) ldp(y0, k + 2);
      fmp(y1, k + 1);
    }
    if (k < K) fmp(y0, k);
  } else {
    for (int k = 0; k < K; ++k) {
      const T* col = U + r0 + (int64_t)k * ldu;
      const A ck = c[k];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        A x[VN];
        load_run<T, VN>(col, (v * GEMV_NT + threadIdx.x) * VN, n - r0, x);
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(x[j], ck, acc[v][j]);
      }
    }
  }
}

}  // namespace sqb
