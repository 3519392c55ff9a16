// K2 — dense (Gaussian) sketch Y = G X (GaussianSketch._apply, sketching.py:109-125).
#pragma once

#include "ctx.cuh"

namespace sqb {

size_t dense_ws_bytes(const sqb_sketch* sk, int dtype, int64_t k);

template <typename T>
int launch_dense(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                 double* Y, int64_t ldy, int64_t row_off, void* ws, const Status* st);

}  // namespace sqb
