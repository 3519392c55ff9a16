// K2 — dense (Gaussian) sketch Y = G X (GaussianSketch._apply, sketching.py:109-125).
#pragma once

#include "ctx.cuh"

namespace sqb {

size_t dense_ws_bytes(const sqb_sketch* sk, int dtype, int64_t k);

// split-K pieces of launch_dense<double> (streamed host input)
int dense_slab_plan(const sqb_sketch* sk, int64_t k, int64_t* kslab);
int launch_dense_slabs(sqb_ctx* ctx, cudaStream_t stream, const sqb_sketch* sk, const double* X, int64_t ldx,
                       int64_t k, int z0, int z1, int64_t kslab, void* ws, const Status* st);
int launch_dense_reduce(sqb_ctx* ctx, const sqb_sketch* sk, int64_t k, int S, const void* ws, double* Y,
                        int64_t ldy, int64_t row_off, const Status* st);

template <typename T>
int launch_dense(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                 double* Y, int64_t ldy, int64_t row_off, void* ws, const Status* st);

}  // namespace sqb
