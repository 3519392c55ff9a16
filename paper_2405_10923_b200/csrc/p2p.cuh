// In-kernel peer-memory exchange of the row-partitioned sweep:
// mailboxes mapped into every peer through CUDA IPC, payloads stored over
// NVLink, release/acquire flags instead of a collective launch.
#pragma once

#include "ctx.cuh"

namespace sqb {

// ---------------------------------------------------------------------------
// Peer-memory mailboxes (in-kernel NVLink exchange, sqb_p2p_*).  Layout of a
// mailbox: uint64 flags [2][nranks] (padded to 256 bytes), then doubles
// [2][nranks][count].  Exchange s (1, 2, ...) uses parity s & 1: rank r stores
// its payload into slot [parity][r] of EVERY peer's mailbox (NVLink stores),
// then releases flag [parity][r] = s in each of them (system scope); the
// consumer acquires all flags >= s before reading its own mailbox.  Slot
// reuse two exchanges later is safe: an exchange is consumed by a kernel every
// rank runs before it produces the next payload (stream order).
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t p2p_flag_bytes(int nranks) {
  return ((size_t)2 * nranks * sizeof(unsigned long long) + 255) & ~size_t(255);
}
__host__ __device__ inline size_t p2p_mailbox_bytes(int nranks, int64_t count) {
  return p2p_flag_bytes(nranks) + sizeof(double) * 2 * (size_t)nranks * (size_t)count;
}
__host__ __device__ inline double* p2p_slot(void* base, int nranks, int64_t count, int parity, int rank) {
  return reinterpret_cast<double*>(static_cast<char*>(base) + p2p_flag_bytes(nranks)) +
         ((int64_t)parity * nranks + rank) * count;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// spin until every rank's flag of this parity reached seq (threads < nranks
// poll, the block then proceeds); flags == nullptr: nothing to wait for
__device__ __forceinline__ void p2p_wait(const unsigned long long* flags, int nranks, int parity,
                                         unsigned long long seq) {
  if (!flags) return;
  if ((int)threadIdx.x < nranks)
    while (ld_acquire_sys(flags + parity * nranks + threadIdx.x) < seq) {
    }
  __syncthreads();
}

// CTA q of the grid stores `pay` (count doubles) into slot [parity][rank] of
// peer q's mailbox, then releases q's flag [parity][rank] = seq
static __global__ void p2p_push_kernel(const double* __restrict__ pay, int64_t count, void* const* peers, int nranks,
                                int rank, int parity, int64_t slot_count, unsigned long long seq) {
  const int q = blockIdx.x;
  void* base = peers[q];
  double* dst = p2p_slot(base, nranks, slot_count, parity, rank);
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = pay[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<unsigned long long*>(base) + parity * nranks + rank, seq);
  }
}

inline int p2p_push(sqb_ctx* ctx, const double* pay, int64_t count, int local, int rank, unsigned long long seq) {
  p2p_push_kernel<<<ctx->p2p_nranks, 256, 0, ctx->stream>>>(pay, count, ctx->p2p_table + (size_t)local * ctx->p2p_nranks,
                                                            ctx->p2p_nranks, rank, (int)(seq & 1), ctx->p2p_count, seq);
  return check_launch(ctx, "p2p_push_kernel");
}

}  // namespace sqb
