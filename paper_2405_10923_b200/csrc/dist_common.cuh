// Pieces shared by the row-partitioned paths (rhqr_dist.cu, krylov.cu):
// the lazily loaded NCCL API, the all-gather (NCCL or, for virtual ranks on
// one device, device copies) and the rank-order combine of gathered SRHT
// partials — the top log2(P) levels of the single-GPU tree, so a combined
// sketch is bitwise the single-GPU one.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <vector>

#include "sketch.cuh"
#include "p2p.cuh"

namespace sqb {

// ---------------------------------------------------------------------------
// NCCL, loaded lazily (single-GPU users never need it)
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.h = h;
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.send = (decltype(api.send))dlsym(h, "ncclSend");
      api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
      api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
      api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
    }
  }
  return (api.getUniqueId && api.commInitRank && api.allGather) ? &api : nullptr;
}

// ---------------------------------------------------------------------------
// combine the gathered raw-sketch partials: Y0[row, col] (od x m)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void rank_combine_kernel(const double* __restrict__ G, int nranks, int ell, int m, int ncols, int rank_level,
                                    const int64_t* __restrict__ idx, int log_tb, double norm_lo,
                                    double* __restrict__ Y0, int64_t ldy, const Status* st,
                                    int64_t rank_stride = -1, const unsigned long long* flags = nullptr,
                                    int parity = 0, unsigned long long seq = 0) {
  using A = typename Lo<T>::acc;
  p2p_wait(flags, nranks, parity, seq, st);  // peer-memory exchange: the peers' partials have landed
  if (failed(st)) return;
  const int64_t rs = rank_stride < 0 ? (int64_t)ncols * (ell + m) : rank_stride;
  const int pl = ell + m;
  const int col = blockIdx.y;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < m + ell; row += gridDim.x * blockDim.x) {
    double y;
    if (row < m) {
      y = __ldcg(G + (int64_t)col * pl + ell + row);  // rank 0's slot
    } else {
      const int o = row - m;
      const int64_t rhi = __ldg(idx + o) >> log_tb;
      A v[8];
      for (int q = 0; q < nranks; ++q) v[q] = (A)__ldcg(G + (int64_t)q * rs + (int64_t)col * pl + o);
      int lvl = rank_level;
      for (int w = 1; w < nranks; w <<= 1, ++lvl) {
        const bool neg = (rhi >> lvl) & 1;
        for (int q = 0; q + w < nranks; q += 2 * w) v[q] = neg ? Lo<T>::sub(v[q], v[q + w]) : Lo<T>::add(v[q], v[q + w]);
      }
      y = (double)Lo<T>::mul(v[0], (A)norm_lo);
    }
    Y0[row + (int64_t)col * ldy] = y;
  }
}


// all-gather `bytes` from every (local) rank's send buffer into G ([rank][bytes])
inline int dist_allgather(sqb_ctx* ctx, bool virt, const std::vector<int>& ids, const std::vector<const void*>& send,
                          size_t bytes, void* G) {
  if (virt) {
    for (size_t r = 0; r < send.size(); ++r)
      SQB_CUDA_TRY(cudaMemcpyAsync((char*)G + (size_t)ids[r] * bytes, send[r], bytes, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
    return SQB_OK;
  }
  NcclApi* nc = nccl_api();
  if (!nc || !ctx->nccl) return set_error(ctx, SQB_ERR_NCCL, "NCCL communicator not initialised");
  ncclResult_t e = nc->allGather(send[0], G, bytes, ncclUint8, (ncclComm_t)ctx->nccl, ctx->stream);
  if (e != ncclSuccess)
    return set_error(ctx, SQB_ERR_NCCL, "ncclAllGather: %s", nc->getErrorString ? nc->getErrorString(e) : "?");
  return SQB_OK;
}

// Halo exchange of a row-partitioned vector into the gathered [rank][seg]
// layout: rank r receives only [lo, hi) of rank p's segment, the range its
// CSR rows reference (halo[(r P + p) 2 + {0, 1}]), plus its own segment.
// NCCL: one group of point-to-point sends/receives (for the 5-point stencil
// one grid row to/from each neighbour instead of the whole vector); virtual
// ranks: device copies into each rank's own gathered buffer.
inline int dist_halo_exchange(sqb_ctx* ctx, bool virt, const std::vector<int>& ids, int nranks,
                              const std::vector<const void*>& local, const std::vector<int64_t>& rows,
                              size_t esz, int64_t seg, const std::vector<void*>& G) {
  const std::vector<int64_t>& h = ctx->halo;
  for (size_t i = 0; i < local.size(); ++i) {
    const int r = ids[i];
    if (rows[i] > 0)
      SQB_CUDA_TRY(cudaMemcpyAsync((char*)G[i] + (size_t)r * seg * esz, local[i], (size_t)rows[i] * esz,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (virt) {
    for (size_t i = 0; i < local.size(); ++i) {
      const int r = ids[i];
      for (size_t j = 0; j < local.size(); ++j) {
        const int p = ids[j];
        if (p == r) continue;
        const int64_t lo = h[((size_t)r * nranks + p) * 2], hi = h[((size_t)r * nranks + p) * 2 + 1];
        if (hi > lo)
          SQB_CUDA_TRY(cudaMemcpyAsync((char*)G[i] + ((size_t)p * seg + lo) * esz, (const char*)local[j] + lo * esz,
                                       (size_t)(hi - lo) * esz, cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
    return SQB_OK;
  }
  NcclApi* nc = nccl_api();
  if (!nc || !ctx->nccl || !nc->send || !nc->recv || !nc->groupStart || !nc->groupEnd)
    return set_error(ctx, SQB_ERR_NCCL, "NCCL point-to-point API not available");
  const int r = ids[0];
  ncclComm_t comm = (ncclComm_t)ctx->nccl;
  ncclResult_t e = nc->groupStart();
  for (int p = 0; p < nranks && e == ncclSuccess; ++p) {
    if (p == r) continue;
    const int64_t slo = h[((size_t)p * nranks + r) * 2], shi = h[((size_t)p * nranks + r) * 2 + 1];
    if (shi > slo) e = nc->send((const char*)local[0] + slo * esz, (size_t)(shi - slo) * esz, ncclUint8, p, comm,
                                ctx->stream);
    const int64_t rlo = h[((size_t)r * nranks + p) * 2], rhi = h[((size_t)r * nranks + p) * 2 + 1];
    if (e == ncclSuccess && rhi > rlo)
      e = nc->recv((char*)G[0] + ((size_t)p * seg + rlo) * esz, (size_t)(rhi - rlo) * esz, ncclUint8, p, comm,
                   ctx->stream);
  }
  const ncclResult_t e2 = nc->groupEnd();
  if (e == ncclSuccess) e = e2;
  if (e != ncclSuccess)
    return set_error(ctx, SQB_ERR_NCCL, "halo exchange: %s", nc->getErrorString ? nc->getErrorString(e) : "?");
  return SQB_OK;
}

}  // namespace sqb
