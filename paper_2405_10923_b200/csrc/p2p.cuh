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
  // [2][nranks] flags, then one word: the wait timeout in ns (0 = P2P_TIMEOUT_NS)
  return ((size_t)(2 * nranks + 1) * sizeof(unsigned long long) + 255) & ~size_t(255);
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
// poll, the block then proceeds); flags == nullptr: nothing to wait for.
// A peer that never arrives (a rank that died, a mapping that went away)
// must not hang the stream: after P2P_TIMEOUT_NS of polling the waiter
// records SQB_ERR_NCCL (col = -(peer + 1), val = seq) in the device status
// and the call chain becomes a no-op like any other failure.  The word after
// the flags of the waiter's own mailbox overrides the limit
// (sqb_p2p_set_timeout_ms).
constexpr long long P2P_TIMEOUT_NS = 20LL * 1000 * 1000 * 1000;

__device__ __forceinline__ long long p2p_now_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void p2p_wait(const unsigned long long* flags, int nranks, int parity,
                                         unsigned long long seq, const Status* st = nullptr) {
  if (!flags) return;
  if ((int)threadIdx.x < nranks) {
    const unsigned long long* f = flags + parity * nranks + threadIdx.x;
    if (ld_acquire_sys(f) < seq) {
      const long long t0 = p2p_now_ns();
      const long long tset = (long long)__ldcg(flags + 2 * nranks);
      const long long limit = tset > 0 ? tset : P2P_TIMEOUT_NS;
      unsigned polls = 0;
      while (ld_acquire_sys(f) < seq) {
        if ((++polls & 0xffu) == 0 && p2p_now_ns() - t0 > limit) {
          if (st) fail(const_cast<Status*>(st), SQB_ERR_NCCL, -((int)threadIdx.x + 1), (double)seq);
          break;
        }
      }
    }
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
