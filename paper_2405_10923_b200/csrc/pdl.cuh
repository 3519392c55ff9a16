// Programmatic dependent launch (PDL): the per-column kernels are launched with
// programmatic stream serialization so kernel c+1 is scheduled while kernel c
// drains; each kernel waits (griddepcontrol.wait) before touching data its
// predecessor produced.
#pragma once

#include <cstdlib>

#include "ctx.cuh"

namespace sqb {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline int launch_pdl(sqb_ctx* ctx, const char* what, void (*kern)(KArgs...), dim3 grid, dim3 block,
                      size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const int no_pdl = [] { const char* e = getenv("SQB_NO_PDL"); return e && e[0] == '1'; }();
  cfg.numAttrs = no_pdl ? 0 : 1;  // SQB_NO_PDL=1: plain stream order (A/B of the look-ahead)
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, what, __FILE__, __LINE__);
  return check_launch(ctx, what);
}

}  // namespace sqb
