// Left-looking randomized Householder QR on the device (rhqr_left, rhqr.py:254-267;
// the hot loop _left_sweep, rhqr.py:219-251).
//
// Per column c two PDL-chained launches:
//
//   rhqr_col_kernel (K3+K1, ~all HBM traffic)  one pass over rows >= m:
//       lazily scale column c-1 (u = fl(w * f), rhqr.py:86-95 + round_to),
//       w_c = fl(W[:,c] - fl(U[:, :c] coef_c)) (:242), store w_c unscaled in
//       U[:, c], emit the in-tile SRHT leaves of w_c.  Extra CTAs: the m-row
//       identity block (y[0:m] = w_c[0:m]) and one HELPER doing the sketch-
//       space work that is off the critical path (T column c-1, a_{c+1}).
//
//   rhqr_step_kernel (K4, an 8-CTA cluster)  finishes the SRHT tree
//       (y[m:] = Omega w_c, bit-exact), rh_vector's scalars (:71-94), s = Psi u,
//       the R column (:248-249), v = S_c^t s (the _extend_t product, :138) and
//       the last entry of the next coefficients — cross-CTA sums through DSMEM.
//
// Coefficients (rhqr.py:241, coef_{c+1} = T_{c+1}^t S_{c+1}^t y0_{c+1}) are
// split so that only two dots sit on the critical path:
//   a_{c+1} = T_c^t (S_c^t y0_{c+1})          (helper, during pass c)
//   coef_{c+1}[:c] = a_{c+1}
//   coef_{c+1}[c]  = beta_c (s_c^t y0_{c+1} - v_c^t a_{c+1})   (step c)
// which is T_{c+1}^t g with T_{c+1}[:c, c] = -beta_c T_c v_c, T[c,c] = beta_c
// (_extend_t) expanded algebraically; T's column c itself is written by the
// helper of pass c+1 exactly as _extend_t forms it.
// The raw sketches y0 = Psi W[:, c] of all columns are computed once up front
// (bitwise equal to the per-column psi.apply(w)).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>

#include "p2p.cuh"
#include "pdl.cuh"
#include "sketch.cuh"
#include "vec.cuh"

namespace cg = cooperative_groups;

namespace sqb {

constexpr int COL_NT = 256;
constexpr int STEP_NT = 512;
constexpr int STEP_CL = 8;  // cluster size of the step kernel

struct ColArgs {
  int c;            // current column of the sweep (>= 1)
  int m;            // identity-block rows of Psi (= columns of the whole W)
  int ncol;         // columns of this sweep (m, or a panel width for rhqr_block)
  int mrow;         // identity-block rows held in this rank's storage (m on rank 0, else 0)
  int64_t e_base;   // global Omega coordinate of this rank's first local coordinate
  int64_t n;        // Omega input length (N - m)
  int ell, od;
  int log_tb;
  int64_t n_tiles;
  int64_t n_eff;
  const void* W;    // column-major, ldw
  int64_t ldw;
  void* U;          // column-major, ldu
  int64_t ldu;
  const double* acur;   // [c-1] coef_c[:c-1] = a_c (written by the helper of pass c-1)
  const double* clast;  // [m] clast[c] = coef_c[c-1] (written by step c-1)
  const double* fscale; // [1] f (sqrt2) or gamma (unit) of column c-1
  int scaling;
  int srht;             // emit SRHT leaves (else the sketch runs separately)
  const uint32_t* bits;
  const int64_t* idx;
  double scale_lo;
  void* P;              // leaves [ell][n_tiles] (acc type)
  double* y;            // (m + ell) sketch of w_c; [0, m) written here
  // helper (sketch-space work off the critical path)
  double* S; int64_t lds;
  double* T; int64_t ldt;
  const double* Y0;     // raw sketches, od x m
  const double* vprev;  // v_{c-1} = S_{c-1}^t s_{c-1}
  const double* betas;
  double* anext;        // out: a_{c+1}
  Status* st;
  int helper_first;     // block order: 1 = helper, identity block, tiles; 0 = tiles, identity, helper
  int no_p16;           // 1: 16-bit storage stages its tile FWHT in fp32 (test hook, SQB_NO_P16)
  int no_pre;           // 1: no pre-wait loads of w_{c-1} / W[:, c] (A/B hook, SQB_NO_PRE)
  int no_part;          // 1: partial last tile on the generic unpipelined loop (test hook, SQB_NO_PART)
  // cross-pass overlap: tflag[b] = last pass block b (tile / identity block /
  // helper) has completed.  With the step kernel triggering its dependents
  // BEFORE its own wait, the CTAs of pass c are dispatched into the slots the
  // last wave of pass c-1 frees and stream their bulk as soon as their own
  // tile of pass c-1 (and its helper) are done, instead of after the whole
  // pass, the step launch and this launch.  null: plain PDL order.
  int* tflag;
  long long* dbg;       // optional block timeline (sqb_debug_col_stamps)
};

__device__ __forceinline__ long long gtime_ns() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}
#define SQB_CSTAMP(i) \
  do { if (a.dbg && threadIdx.x == 0) a.dbg[blockIdx.x * 8 + (i)] = gtime_ns(); } while (0)

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// every thread of the block has issued its stores: publish "block b finished pass c"
__device__ __forceinline__ void col_flag_done(const ColArgs& a) {
  if (!a.tflag) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release_gpu(a.tflag + blockIdx.x, a.c);
  }
}

// wait until this block's own pass c-1 and the helper of pass c-1 are done
// (they are resident or finished: pass c-1 was dispatched completely before
// step c-1, hence before this grid, became eligible).  A recorded failure
// releases the waiters: every block returns at its post-wait status check.
__device__ __forceinline__ void col_flag_wait(const ColArgs& a, int64_t helper_id) {
  if (!a.tflag) return;
  if (a.c >= 2 && (threadIdx.x == 0 || threadIdx.x == 32)) {
    const int* f = a.tflag + (threadIdx.x == 0 ? helper_id : (int64_t)blockIdx.x);
    while (ld_acquire_gpu(f) < a.c - 1 && !failed(a.st)) __nanosleep(40);
  }
  __syncthreads();
}

// SQB_EARLY=0 restores the plain PDL order (A/B experiments)
inline int early_env() {
  const char* e = getenv("SQB_EARLY");
  return e ? atoi(e) : 1;
}

// SQB_HELPER_FIRST=0 restores the old block order (A/B experiments)
inline int helper_first_default() {
  const char* e = getenv("SQB_HELPER_FIRST");
  return e ? atoi(e) : 1;
}
inline int no_pre_env() {
  const char* e = getenv("SQB_NO_PRE");
  return e && e[0] == '1';
}
inline int no_part_env() {
  const char* e = getenv("SQB_NO_PART");
  return e && e[0] == '1';
}
inline int no_p16_env() {
  const char* e = getenv("SQB_NO_P16");
  return e && e[0] == '1';
}

template <typename T>
__device__ __forceinline__ typename Lo<T>::acc lazy_scale(typename Lo<T>::acc w, double f, int scaling) {
  // rhqr.py:86-95 then round_to(u, low): u = fl64(w * f) or fl64(w / gamma)
  const double u = scaling == SQB_SCALE_SQRT2 ? __dmul_rn((double)w, f) : __ddiv_rn((double)w, f);
  return Lo<T>::from_double(u);
}

// identity block: y[r] = w_c[r] = fl(W[r,c] - fl(sum_k U[r,k] coef[k])), r < m.
// Columns k <= c-2 are final before step c-1 ends, so they are summed before
// the PDL wait; column c-1 (its top rows come from step c-1) after it.
template <typename T>
__device__ void col_top_block(const ColArgs& a, typename Lo<T>::acc* sc) {
  using A = typename Lo<T>::acc;
  const T* W = (const T*)a.W;
  const T* U = (const T*)a.U;
  const int c = a.c;
  constexpr int RPT = 4;  // rows per thread (m <= RPT * blockDim)
  A acc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = threadIdx.x + q * blockDim.x;
    A acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    if (r < a.m) {
      int k = 0;
      for (; k + 4 <= c - 1; k += 4) {
        acc0 = fma(Lo<T>::load(U[r + (int64_t)k * a.ldu]), sc[k], acc0);
        acc1 = fma(Lo<T>::load(U[r + (int64_t)(k + 1) * a.ldu]), sc[k + 1], acc1);
        acc2 = fma(Lo<T>::load(U[r + (int64_t)(k + 2) * a.ldu]), sc[k + 2], acc2);
        acc3 = fma(Lo<T>::load(U[r + (int64_t)(k + 3) * a.ldu]), sc[k + 3], acc3);
      }
      for (; k < c - 1; ++k) acc0 = fma(Lo<T>::load(U[r + (int64_t)k * a.ldu]), sc[k], acc0);
    }
    acc[q] = (acc0 + acc1) + (acc2 + acc3);
  }
  pdl_wait();
  if (failed(a.st)) return;
  const A cl = Lo<T>::from_double(a.clast[c]);
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int r = threadIdx.x + q * blockDim.x;
    if (r < a.m) {
      const A dot = fma(Lo<T>::load(U[r + (int64_t)(c - 1) * a.ldu]), cl, acc[q]);
      const A w = Lo<T>::sub(Lo<T>::load(W[r + (int64_t)c * a.ldw]), Lo<T>::rnd(dot));
      a.y[r] = (double)w;
    }
  }
}

// T[:kk, kk] = -beta * T[:kk,:kk] v ; T[kk,kk] = beta   (_extend_t, rhqr.py:135-140)
// One thread per row with coalesced column reads, eight independent loads in
// flight per step (an L2-latency chain per lane made this the longest CTA of
// the pass at m = 256).  T holds explicit zeros below its diagonal; entries
// k < i are masked to exact zeros anyway.
__device__ inline void complete_t_column(double* T, int64_t ldt, int kk, const double* v, double beta) {
  for (int i0 = 0; i0 < kk; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const int kb = i0 + (threadIdx.x & ~31);  // warp-uniform first column
    if (kb >= kk) break;
    const bool on = i < kk;
    const double* Ti = T + (on ? i : kb);
    double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int k = kb;
    for (; k + 8 <= kk; k += 8) {
      double t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) t[u] = Ti[(int64_t)(k + u) * ldt];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (k + u < i) t[u] = 0.0;
      d0 = fma(t[0], v[k], d0);
      d1 = fma(t[1], v[k + 1], d1);
      d2 = fma(t[2], v[k + 2], d2);
      d3 = fma(t[3], v[k + 3], d3);
      d0 = fma(t[4], v[k + 4], d0);
      d1 = fma(t[5], v[k + 5], d1);
      d2 = fma(t[6], v[k + 6], d2);
      d3 = fma(t[7], v[k + 7], d3);
    }
    for (; k < kk; ++k) {
      const double t = k < i ? 0.0 : Ti[(int64_t)k * ldt];
      d0 = fma(t, v[k], d0);
    }
    if (on) T[i + (int64_t)kk * ldt] = __dmul_rn(-beta, (d0 + d1) + (d2 + d3));
  }
  if (threadIdx.x == 0) T[kk + (int64_t)kk * ldt] = beta;
}

// helper CTA of pass c: complete T column c-1, then a_{c+1} = T_c^t (S_c^t y0_{c+1})
__device__ inline void col_helper(const ColArgs& a, double* g) {
  const int c = a.c;
  complete_t_column(a.T, a.ldt, c - 1, a.vprev, a.betas[c - 1]);
  if (c + 1 >= a.ncol) return;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* y0 = a.Y0 + (int64_t)(c + 1) * a.od;
  // g = S_c^t y0 (S[:, k] is zero above row k): 8 independent loads per lane
  for (int k = warp; k < c; k += nw) {
    const double* sk = a.S + (int64_t)k * a.lds;
    double d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) d[u] = 0.0;
    for (int r0 = k; r0 < a.od; r0 += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u * 32 + lane;
        if (r < a.od) d[u] = fma(sk[r], y0[r], d[u]);
      }
    }
    const double dd = warp_sum(((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7])));
    if (lane == 0) g[k] = dd;
  }
  __syncthreads();
  // a_{c+1}[j] = T[:j+1, j] . g[:j+1]
  for (int j = warp; j < c; j += nw) {
    const double* tj = a.T + (int64_t)j * a.ldt;
    double d[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) d[u] = 0.0;
    for (int i0 = 0; i0 <= j; i0 += 256) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * 32 + lane;
        if (i <= j) d[u] = fma(tj[i], g[i], d[u]);
      }
    }
    const double dd = warp_sum(((d[0] + d[1]) + (d[2] + d[3])) + ((d[4] + d[5]) + (d[6] + d[7])));
    if (lane == 0) a.anext[j] = dd;
  }
}

// DEP = 0: loads widened at issue, one column ahead; DEP >= 2: raw ring of
// DEP column buffers (see the bulk loop)
// LOGT: log2 of the tile (SRHT leaf group) size; small problems use 512-row
// tiles so the pass spreads over enough CTAs (the leaves and the step
// kernel's tree adapt: the same binary tree, the same bits)
template <typename T, int VN, int DEP = 0, int MINB = 2, int LOGT = TileCfg<T>::LOG_TB>
__global__ void __launch_bounds__(COL_NT, MINB) rhqr_col_kernel(ColArgs a) {
  using A = typename Lo<T>::acc;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* sc = reinterpret_cast<A*>(smem_raw);                      // coef rounded to low [c]
  A* sm = sc + ((a.c + 3) & ~3);                              // tile buffer
  pdl_trigger();
  if (a.dbg && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;\n" : "=r"(smid));
    a.dbg[blockIdx.x * 8] = smid;
  }
  SQB_CSTAMP(1);
  const int c = a.c;
  // block roles: with helper_first the helper (block 0) and the identity block
  // (block 1) are dispatched first, so the helper's latency-bound sketch-space
  // work overlaps the first wave of tiles instead of trailing the last one
  const int64_t bid = blockIdx.x;
  const int64_t helper_id = a.helper_first ? 0 : a.n_eff + 1;
  const int64_t top_id = a.helper_first ? 1 : a.n_eff;
  const int64_t tile = a.helper_first ? bid - 2 : bid;
  if (bid == helper_id) {
    pdl_wait();
    SQB_CSTAMP(4);
    if (!failed(a.st)) col_helper(a, reinterpret_cast<double*>(sm));
    SQB_CSTAMP(5);
    col_flag_done(a);
    return;
  }
  col_flag_wait(a, helper_id);
  SQB_CSTAMP(2);
  // coef_c[:c-1] = a_c is final before step c-1 ends (helper of pass c-1): load
  // it and stream the bulk of the GEMV BEFORE waiting on step c-1 (look-ahead
  // overlap of the HBM pass with the sketch-space step, via PDL)
  for (int k = threadIdx.x; k < c - 1; k += COL_NT) sc[k] = Lo<T>::from_double(a.acur[k]);
  __syncthreads();
  if (bid == top_id) {
    if (a.mrow > 0) col_top_block<T>(a, sc);
    SQB_CSTAMP(5);
    col_flag_done(a);
    return;
  }
  constexpr int TB = 1 << LOGT;
  constexpr int NV = TB / (COL_NT * VN);  // runs of VN rows per thread
  const int tb = 1 << a.log_tb;
  const int64_t e0 = tile << a.log_tb;  // first Omega coordinate of the tile
  const int64_t lim = a.n - e0;                       // valid rows in this tile (may exceed tb)
  const int64_t rows = lim < tb ? lim : tb;
  const int64_t ro = (int64_t)a.mrow + e0;             // first row of the tile in W / U
  T* U = (T*)a.U;
  const T* W = (const T*)a.W;

  A acc[NV][VN];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int j = 0; j < VN; ++j) acc[v][j] = A(0);

  // final columns 0 .. c-2
  const int K = c - 1;
  if (DEP >= 2 && VN > 1 && rows == TB && tb == TB) {
    // full tile: streaming loads kept RAW (one uint4 per 16 bytes) in a ring
    // of D column buffers, widened only at the FMA — 2-byte storage keeps
    // four columns in flight per thread in the registers fp32 widening of
    // two would take (ncu: the bf16 pass was L1TEX-latency bound at D = 2)
    constexpr int D = DEP >= 2 ? DEP : 2;
    uint4 rb[D][NV];
    auto ldr = [&](uint4 (&x)[NV], int k) {
      const T* col = U + ro + (int64_t)k * a.ldu;
#pragma unroll
      for (int v = 0; v < NV; ++v) x[v] = ldg_stream(col + (v * COL_NT + threadIdx.x) * VN);
    };
    auto fmr = [&](const uint4 (&x)[NV], int k) {
      const A ck = sc[k];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        A w[VN];
        unpack16<T>(x[v], w);
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(w[j], ck, acc[v][j]);
      }
    };
#pragma unroll
    for (int d = 0; d < D - 1; ++d)
      if (d < K) ldr(rb[d], d);
    for (int k0 = 0; k0 < K; k0 += D) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const int k = k0 + j;
        if (k < K) {
          if (k + D - 1 < K) ldr(rb[(j + D - 1) % D], k + D - 1);
          fmr(rb[j], k);
        }
      }
    }
  } else if (VN > 1 && rows == TB && tb == TB) {
    // full tile: streaming loads, software-pipelined one column ahead
    A x0[NV][VN], x1[NV][VN];
    auto ld = [&](A (&x)[NV][VN], int k) {
      const T* col = U + ro + (int64_t)k * a.ldu;
#pragma unroll
      for (int v = 0; v < NV; ++v) vload_stream<T>(col + (v * COL_NT + threadIdx.x) * VN, x[v]);
    };
    auto fm = [&](A (&x)[NV][VN], int k) {
      const A ck = sc[k];
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
  } else if (VN > 1 && tb == TB && rows > 0 && rows % VN == 0 && !a.no_part) {
    // partial last tile made of whole 16-byte runs (n = N - m is normally a
    // multiple of the run): the same one-column-ahead pipeline with the runs
    // beyond `rows` masked.  The generic loop below issues one column, waits
    // for it, then the next — at config 4 that single block took 270 us of
    // an 830 us pass whose other 2049 blocks were done after 657 us
    // (scripts/col_timeline.py); same summation order, same bits.
    uint4 r0[NV], r1[NV];
    auto ldp = [&](uint4 (&x)[NV], int k) {
      const T* col = U + ro + (int64_t)k * a.ldu;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = (v * COL_NT + threadIdx.x) * VN;
        x[v] = i < rows ? ldg_stream(col + i) : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    auto fmp = [&](const uint4 (&x)[NV], int k) {
      const A ck = sc[k];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        A w[VN];
        unpack16<T>(x[v], w);
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(w[j], ck, acc[v][j]);
      }
    };
    if (K > 0) ldp(r0, 0);
    int k = 0;
    for (; k + 2 <= K; k += 2) {
      ldp(r1, k + 1);
      fmp(r0, k);
      if (k + 2 < K) ldp(r0, k + 2);
      fmp(r1, k + 1);
    }
    if (k < K) fmp(r0, k);
  } else {
    for (int k = 0; k < K; ++k) {
      const T* col = U + ro + (int64_t)k * a.ldu;
      const A ck = sc[k];
      A v0[NV][VN];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int i = (v * COL_NT + threadIdx.x) * VN;
        if (i < tb) load_run<T, VN>(col, i, rows, v0[v]);
      }
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int j = 0; j < VN; ++j) acc[v][j] = fma(v0[v][j], ck, acc[v][j]);
    }
  }
  // The stored w_{c-1} (pass c-1 is complete: step c-1 waited on it before
  // launching this pass) and W[:, c] do not depend on step c-1 either: on a
  // full tile both are loaded raw BEFORE the wait, into the registers the
  // bulk ring just released, so the tail after the wait starts with its
  // operands in flight instead of two serial DRAM round trips.
  // (the 3-CTA/SM 16-bit variant has registers for W[:, c] only; its w_{c-1}
  // was written by pass c-1 moments ago and is mostly still in L2)
  const bool full = VN > 1 && rows == TB && tb == TB && !a.no_pre;
  constexpr bool PRE_U = MINB <= 2;
  const T* src = (c == 1 ? W : (const T*)U) + ro + (int64_t)(c - 1) * (c == 1 ? 0 : a.ldu);
  const T* wc = W + ro + (int64_t)c * a.ldw;
  uint4 pre_u[NV], pre_w[NV];
  if (full) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if constexpr (PRE_U) pre_u[v] = ldg_l2only(src + i);
      pre_w[v] = ldg_stream(wc + i);
    }
  }
  // ---- wait for step c-1 (f_{c-1}, coef_c[c-1], breakdown status)
  SQB_CSTAMP(3);
  pdl_wait();
  SQB_CSTAMP(4);
  if (failed(a.st)) { col_flag_done(a); return; }
  // column c-1: lazy scaling of the stored w_{c-1}, write back u_{c-1}
  {
    T* dst = U + ro + (int64_t)(c - 1) * a.ldu;
    const double f = *a.fscale;
    const A ck = Lo<T>::from_double(a.clast[c]);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if (i < tb) {
        A x[VN];
        if (PRE_U && full) unpack16<T>(pre_u[v], x);
        else load_run<T, VN>(src, i, rows, x);
#pragma unroll
        for (int j = 0; j < VN; ++j) {
          x[j] = lazy_scale<T>(x[j], f, a.scaling);
          acc[v][j] = fma(x[j], ck, acc[v][j]);
        }
        store_run<T, VN>(dst, i, rows, x);
      }
    }
  }
  // w_c = fl(W[:, c] - fl(dot)); store unscaled into U[:, c]; SRHT input to smem
  // 16-bit storage with a full tile runs the in-tile FWHT on packed pairs in
  // 16-bit shared memory (srht.cuh p16_*): ~6x fewer butterfly instructions
  // than fp32 staging with a rounding per op, half the shared traffic
  constexpr bool P16OK = sizeof(T) == 2 && VN == 8 && TileCfg<T>::LOG_TB == P16_LOG;
  const bool p16path = P16OK && a.srht && a.log_tb == P16_LOG && !a.no_p16;
  {
    T* uc = U + ro + (int64_t)c * a.ldu;
    const A s_lo = (A)a.scale_lo;
    uint32_t scale2 = 0;
    if constexpr (P16OK) {
      const uint32_t h = pk_pack<T>((float)a.scale_lo, 0.f) & 0xffffu;
      scale2 = h | (h << 16);
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int i = (v * COL_NT + threadIdx.x) * VN;
      if (i < tb) {
        A x[VN];
        if (full) unpack16<T>(pre_w[v], x);
        else load_run<T, VN>(wc, i, rows, x);
#pragma unroll
        for (int j = 0; j < VN; ++j) x[j] = Lo<T>::sub(x[j], Lo<T>::rnd(acc[v][j]));
        store_run<T, VN>(uc, i, rows, x);
        if constexpr (P16OK) {
          if (p16path) {
            const int64_t e = a.e_base + e0 + i;
            const uint32_t sb = __ldg(a.bits + (e >> 5)) >> (e & 31);
            const int64_t vl = rows - i;
            p16_run_in<T>(reinterpret_cast<uint16_t*>(sm), i, x, scale2, sb, vl >= 8 ? 8 : (vl > 0 ? (int)vl : 0));
            continue;
          }
        }
        if (a.srht) {
          const int64_t e = a.e_base + e0 + i;  // global Omega coordinate (sign bits)
          const uint32_t sb = __ldg(a.bits + (e >> 5)) >> (e & 31);
#pragma unroll
          for (int j = 0; j < VN; ++j)
            sm[pidx<A>(i + j)] = (i + j < rows) ? srht_in<T>(x[j], s_lo, (sb >> j) & 1u) : A(0);
        }
      }
    }
  }
  if (!a.srht) { col_flag_done(a); return; }
  __syncthreads();
  if constexpr (P16OK) {
    if (p16path) {
      const uint16_t* s16 = reinterpret_cast<const uint16_t*>(sm);
      p16_passes<T>(reinterpret_cast<uint16_t*>(sm));
      float* P = (float*)a.P + tile;
      for (int k = threadIdx.x; k < a.ell; k += COL_NT)
        P[k * a.n_tiles] = pk_lo_float<T>(s16[p16((int)(__ldg(a.idx + k) & ((1 << P16_LOG) - 1)))]);
      SQB_CSTAMP(5);
      col_flag_done(a);
      return;
    }
  }
  tile_fwht<T>(sm, a.log_tb);
  tile_gather<T>(sm, a.idx, a.ell, a.log_tb, (A*)a.P + tile, a.n_tiles);
  SQB_CSTAMP(5);
  col_flag_done(a);
}

// Bulk-loop variant of the column pass.  2-byte storage: a raw 2-deep ring
// at 3 CTAs/SM (78 registers, 24 resident warps instead of 16) — the pass is
// bound by load latency (ncu: L1TEX-scoreboard stalls at the first use of
// each load), +5% on config 4.  4/8-byte storage: widened loads one column
// ahead at 2 CTAs/SM (0.9+ of the HBM copy peak).  SQB_COL_VARIANT=base
// forces the latter for 2-byte storage too (A/B experiments).
template <typename T, int VN>
inline void (*col_kernel_select(bool vec))(ColArgs) {
  if (!vec) return rhqr_col_kernel<T, 1>;
  if constexpr (sizeof(T) == 2) {
    const char* e = getenv("SQB_COL_VARIANT");
    if (!(e && e[0] == 'b')) return rhqr_col_kernel<T, VN, 2, 3>;
  }
  return rhqr_col_kernel<T, VN>;
}

// ---------------------------------------------------------------------------
// K4: cluster step kernel for column c.  The od = m + ell rows of Psi-space are
// split into STEP_CL contiguous blocks, one per CTA of the cluster (top-block
// rows < m first, then the Omega rows whose sketch values the tree produces).
// ---------------------------------------------------------------------------
struct StepArgs {
  int c, m, ell, od;
  int off, ncol;              // sweep offset (pivot row = off + c) and width (rhqr.py:219-251)
  int scaling;
  int early;                  // 1: trigger the dependents (pass c+1) before waiting for pass c (ColArgs::tflag)
  int tree;                   // 1: finish the SRHT tree from the tile leaves; 0: y[m:] given;
                              // 2: combine the gathered per-rank partials (multi-GPU);
                              // 3: fused exchange — this kernel folds the rank-local subtree of the
                              //    tile leaves, stores the partials straight into every peer's mailbox
                              //    (NVLink), releases its flags, then proceeds as 2 on its own mailbox
  void* const* peers;         // tree == 3: mailbox base of every rank (own included), device table
  int my_rank;                // tree == 3
  int64_t slot_count;         // tree == 3: doubles per mailbox slot
  const double* toprows;      // tree == 3: this rank's identity-block rows of w_c (rank 0), else null
  const double* gath;         // tree == 2: [nranks][gstride] per-rank partials (+ rank 0's top rows)
  int64_t gstride;            // tree == 2: doubles between ranks' partials (ell + m for a gather buffer)
  const unsigned long long* flags;  // tree == 2, peer-memory exchange: acquire flags >= seq first
  unsigned long long seq;
  int nranks, rank_level;     // tree == 2: P and the tree level of the rank split (log2 local tiles)
  const void* P;              // leaves [ell][n_tiles]
  int64_t n_tiles, n_eff;
  const int64_t* idx;
  int log_tb;
  double norm_lo;
  double* y;                  // (od) sketch of w_c: [0, m) given, [m, od) tree output
  const double* Y0;           // raw sketches (od x m, ld od)
  double* S; int64_t lds;
  double* R; int64_t ldr;
  void* U; int64_t ldu;       // identity-block rows of U[:, c] are written here
  double* sigmas; double* rhos; double* betas;
  double* fscale;             // out: f of column c
  double* vbuf;               // out: v_c = S_c^t s_c
  const double* anext;        // in: a_{c+1} (helper of pass c)
  double* clast;              // out: clast[c+1] = coef_{c+1}[c]
  Status* st;
  long long* dbg;             // optional per-phase clock64 stamps [STEP_CL][8] (instrumentation)
  long long* gdbg;            // optional globaltimer stamps {entry, after wait, exit} of rank 0
};

#define SQB_STAMP(i) \
  do { if (a.dbg && threadIdx.x == 0) a.dbg[rank * 8 + (i)] = clock64(); } while (0)

constexpr int STEP_KC = 128;                 // columns staged per chunk
constexpr int STEP_NPART = STEP_NT / STEP_KC;

__host__ __device__ inline int step_rows(int od) { return (od + STEP_CL - 1) / STEP_CL; }
__host__ __device__ inline int step_ldst(int od) { return step_rows(od) | 1; }
inline size_t step_smem_bytes(int od, int m) {
  const int B = step_rows(od);
  return sizeof(double) * (2 * (size_t)B + (size_t)STEP_KC * step_ldst(od) + STEP_CL * (size_t)(m + 1) +
                           STEP_NPART * STEP_KC + STEP_CL + 32);
}

template <typename T>
__global__ void __cluster_dims__(STEP_CL, 1, 1) __launch_bounds__(STEP_NT)
rhqr_step_kernel(StepArgs a) {
  using A = typename Lo<T>::acc;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int c = a.c, m = a.m, od = a.od, tid = threadIdx.x;
  const int pv = a.off + c;  // pivot row j-1 of this column (rhqr.py:233)
  const int lane = tid & 31, warp = tid >> 5, nw = STEP_NT / 32;
  const int B = step_rows(od), ldst = step_ldst(od);
  const int r0 = rank * B, r1 = min(od, r0 + B), nrow = max(0, r1 - r0);
  const int nk = c + 1;  // partial vector: v[0..c-1], s^t y0_{c+1}
  double* yv = reinterpret_cast<double*>(smem_raw);  // [B] sketch rows owned
  double* sv = yv + B;                               // [B] s rows owned
  double* stage = sv + B;                            // [STEP_KC][ldst] staged S / y0 block
  double* gath = stage + (size_t)STEP_KC * ldst;     // [STEP_CL][nk] partial vectors (rank 0)
  double* cpart = gath + STEP_CL * (m + 1);          // [STEP_NPART][STEP_KC]
  double* part = cpart + STEP_NPART * STEP_KC;       // [STEP_CL] rho^2 partials
  double* red = part + STEP_CL;                      // [32]
  __shared__ double scal[4];
  SQB_STAMP(0);
  // early: pass c+1 becomes eligible as soon as this cluster is resident; its
  // blocks order themselves behind pass c with per-block flags and behind
  // this step with their own griddepcontrol.wait
  if (a.gdbg && rank == 0 && tid == 0) a.gdbg[0] = gtime_ns();
  if (a.early) pdl_trigger();
  pdl_wait();
  if (!a.early) pdl_trigger();
  if (a.gdbg && rank == 0 && tid == 0) a.gdbg[1] = gtime_ns();
  if (a.tree == 3) {
    // the exchange of column c inside the step: no tree / push launches on the
    // column's critical path.  Runs even after a recorded failure (every rank
    // fails at the same column, and every rank still waits for the flags).
    const int par = (int)(a.seq & 1);
    const int rr0 = rank * step_rows(od), rr1 = min(od, rr0 + step_rows(od));
    for (int row = max(rr0, m) + warp; row < rr1; row += nw) {
      const int o = row - m;
      const int64_t rhi = __ldg(a.idx + o) >> a.log_tb;
      const A v = warp_tile_tree<T>((const A*)a.P + (int64_t)o * a.n_tiles, (int)a.n_tiles, (int)a.n_eff, rhi);
      if (lane < a.nranks) p2p_slot(a.peers[lane], a.nranks, a.slot_count, par, a.my_rank)[o] = (double)v;
    }
    if (a.toprows)
      for (int row = rr0 + tid; row < min(rr1, m); row += STEP_NT) {
        const double y = a.toprows[row];
        for (int q = 0; q < a.nranks; ++q) p2p_slot(a.peers[q], a.nranks, a.slot_count, par, a.my_rank)[a.ell + row] = y;
      }
    __threadfence_system();
    cluster.sync();  // every CTA's stores are issued and fenced
    if (rank == 0 && tid < a.nranks) {
      __threadfence_system();
      st_release_sys(reinterpret_cast<unsigned long long*>(a.peers[tid]) + par * a.nranks + a.my_rank, a.seq);
    }
  }
  if (a.tree >= 2) p2p_wait(a.flags, a.nranks, (int)(a.seq & 1), a.seq, a.st);
  SQB_STAMP(1);
  const bool dead = failed(a.st);  // uniform across the cluster; still take part in the sync
  // ---- phase A: y on the owned rows (identity block given; Omega rows from the tree)
  if (!dead) {
    if (a.tree >= 2) {
      // upper log2(P) levels of the SRHT tree across ranks (left = lower rank)
      // plus the identity block from rank 0's payload
      for (int i = tid; i < nrow; i += STEP_NT) {
        const int row = r0 + i;
        double y;
        if (row < m) {
          y = __ldcg(a.gath + a.ell + row);
        } else {
          const int o = row - m;
          const int64_t rhi = __ldg(a.idx + o) >> a.log_tb;
          A v[8];
          for (int q = 0; q < a.nranks; ++q) v[q] = (A)__ldcg(a.gath + q * a.gstride + o);
          int lvl = a.rank_level;
          for (int w2 = 1; w2 < a.nranks; w2 <<= 1, ++lvl) {
            const bool neg = (rhi >> lvl) & 1;
            for (int q = 0; q + w2 < a.nranks; q += 2 * w2)
              v[q] = neg ? Lo<T>::sub(v[q], v[q + w2]) : Lo<T>::add(v[q], v[q + w2]);
          }
          y = (double)Lo<T>::mul(v[0], (A)a.norm_lo);
          a.y[row] = y;
        }
        yv[i] = y;
        if (row < m) a.y[row] = y;
      }
    } else {
    for (int i = tid; i < nrow; i += STEP_NT) {
      const int row = r0 + i;
      if (row < m || !a.tree) yv[i] = a.y[row];
    }
    }
    if (a.tree == 1) {
      const int ob = max(r0, m), oe = r1;
      for (int row = ob + warp; row < oe; row += nw) {
        const int o = row - m;
        const int64_t rhi = __ldg(a.idx + o) >> a.log_tb;
        const A v = warp_tile_tree<T>((const A*)a.P + (int64_t)o * a.n_tiles, (int)a.n_tiles,
                                      (int)a.n_eff, rhi);
        if (lane == 0) {
          const double y = (double)Lo<T>::mul(v, (A)a.norm_lo);
          yv[row - r0] = y;
          a.y[row] = y;
        }
      }
    }
  }
  __syncthreads();
  SQB_STAMP(2);
  // ---- phase B: rho = ||y[c:]|| (rhqr.py:72); partials pushed to every CTA
  double p = 0.0;
  if (!dead)
    for (int i = tid; i < nrow; i += STEP_NT)
      if (r0 + i >= pv) p = fma(yv[i], yv[i], p);
  p = block_sum(p, red);
  if (tid < STEP_CL) *cluster.map_shared_rank(&part[rank], tid) = p;
  cluster.sync();
  SQB_STAMP(3);
  if (dead) return;
  if (tid == 0) {
    double r2 = 0.0;
    for (int q = 0; q < STEP_CL; ++q) r2 += part[q];
    const double rho = sqrt(r2);
    const double yc = a.y[pv];
    const double sigma = yc >= 0.0 ? 1.0 : -1.0;                                 // linalg.py:200-202
    const double gamma = __dadd_rn(yc, sigma * rho);                               // rhqr.py:76
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));   // :77
    bool bad = false;
    if (rho == 0.0) { bad = true; if (rank == 0) fail(a.st, SQB_ERR_BREAKDOWN, pv + 1, 0.0); }
    else if (!isfinite(beta)) { bad = true; if (rank == 0) fail(a.st, SQB_ERR_BREAKDOWN, pv + 1, rho); }
    double f, bo;
    if (a.scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
    else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    scal[0] = -sigma * rho; scal[1] = gamma; scal[2] = f; scal[3] = bad ? -1.0 : bo;
    if (rank == 0 && !bad) {
      a.sigmas[c] = sigma; a.rhos[c] = rho; a.betas[c] = bo;
      *a.fscale = f;
    }
  }
  __syncthreads();
  const double rdiag = scal[0], gamma = scal[1], f = scal[2], bo = scal[3];
  // a breakdown is seen identically by every CTA: leave together (no more DSMEM)
  if (bo < 0.0) return;
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  SQB_STAMP(4);
  // ---- phase C: s = Psi u (rhqr.py:83-96), u's identity-block rows, R column (:248-249)
  T* U = (T*)a.U;
  for (int i = tid; i < nrow; i += STEP_NT) {
    const int row = r0 + i;
    const double yh = row < pv ? 0.0 : (row == pv ? gamma : yv[i]);
    const double s = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    sv[i] = s;
    a.S[row + (int64_t)c * a.lds] = s;
    if (row < m) {
      U[row + (int64_t)c * a.ldu] = Lo<T>::store(Lo<T>::from_double(s));
      a.R[row + (int64_t)c * a.ldr] = row < pv ? yv[i] : (row == pv ? rdiag : 0.0);
    }
  }
  // partial vector over the owned rows >= c (s vanishes above c):
  // v[k] = S[:, k]^t s (k < c), d = s^t y0_{c+1}; staged through smem, pushed to rank 0
  const bool has_next = c + 1 < a.ncol;
  const double* y0n = has_next ? a.Y0 + (int64_t)(c + 1) * od : nullptr;
  const int nkk = has_next ? nk : c;
  const int rs = max(r0, pv), nr = max(0, r1 - rs), ls = rs - r0;
  double* dst0 = cluster.map_shared_rank(gath, 0) + rank * nk;
  for (int k0 = 0; k0 < nkk; k0 += STEP_KC) {
    const int kc = min(STEP_KC, nkk - k0);
    __syncthreads();
#pragma unroll 4
    for (int e = tid; e < nr * kc; e += STEP_NT) {
      const int i = e % nr, kk = e / nr, k = k0 + kk;
      const double* col = (k < c) ? a.S + (int64_t)k * a.lds : y0n;
      stage[kk * ldst + i] = col[rs + i];
    }
    __syncthreads();
    {
      const int kk = tid % STEP_KC, pp = tid / STEP_KC;
      double d = 0.0;
      if (kk < kc)
        for (int i = pp; i < nr; i += STEP_NPART) d = fma(stage[kk * ldst + i], sv[ls + i], d);
      cpart[pp * STEP_KC + kk] = d;
    }
    __syncthreads();
    if (tid < kc) {
      double d = 0.0;
      for (int q = 0; q < STEP_NPART; ++q) d += cpart[q * STEP_KC + tid];
      dst0[k0 + tid] = d;
    }
  }
  SQB_STAMP(5);
  cluster.sync();
  SQB_STAMP(6);
  if (rank != 0) return;
  // ---- phase D (rank 0): v_c, and coef_{c+1}[c] = beta (d - v^t a_{c+1})
  double va = 0.0;
  for (int k = tid; k < c; k += STEP_NT) {
    double v = 0.0;
    for (int q = 0; q < STEP_CL; ++q) v += gath[q * nk + k];
    a.vbuf[k] = v;
    if (has_next) va = fma(v, a.anext[k], va);
  }
  if (!has_next) return;
  va = block_sum(va, red);
  if (tid == 0) {
    double d = 0.0;
    for (int q = 0; q < STEP_CL; ++q) d += gath[q * nk + c];
    a.clast[c + 1] = __dmul_rn(bo, d - va);
    if (a.gdbg) a.gdbg[2] = gtime_ns();
  }
  SQB_STAMP(7);
}

// last column: lazy scaling of its Omega rows + its T column (_extend_t)
template <typename T>
__global__ void finish_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t n,
                              const double* fscale, int scaling, double* Tm, int64_t ldt, int m,
                              const double* v, const double* betas, const Status* st) {
  pdl_wait();
  if (failed(st)) return;
  if (blockIdx.x == gridDim.x - 1) {
    complete_t_column(Tm, ldt, m - 1, v, betas[m - 1]);
    return;
  }
  const double f = *fscale;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)(gridDim.x - 1) * blockDim.x)
    dst[i] = Lo<T>::store(lazy_scale<T>(Lo<T>::load(src[i]), f, scaling));
}

}  // namespace sqb
