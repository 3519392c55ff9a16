// Persistent single-kernel left-looking RHQR for small fp64 problems
// (BASELINE config 1: 2^14 x 32, SRHT 128; _left_sweep, rhqr.py:219-251).
//
// The per-column launch chain (rhqr_col_kernel -> rhqr_step_kernel, 2 launches
// per column) is latency-bound at this size: 77.6 MB of traffic against
// 32 x ~13 us of dependent launches.  Here ONE cooperative grid
// runs every column:
//
//   CTA g < n_eff   owns the 512 Omega rows of tile g for the whole sweep: its
//                   W/U rows stay in shared memory (the GEMV over U[:, :c]
//                   reads shared memory, not L2), it emits the tile's SRHT
//                   leaves of w_c;
//   CTA n_eff       the identity-block rows (y[0:m]) and the helper work of
//                   the column pass (T column c-1, a_{c+1}), and it writes the
//                   sketch-space outputs (S, R, U's top rows, scalars).
//
// Per column: phase A (the column pass) -> one grid barrier -> phase B, the
// step, computed REDUNDANTLY by every CTA (each finishes the SRHT tree of all
// ell sampled rows from the leaves and derives f_c and coef_{c+1}), so there
// is no second barrier.  Every reduction of phase B replays the 8-CTA x
// 512-thread cluster step kernel's association order exactly, and phase A
// the column kernel's, so the factors are BITWISE those of the launch-chain
// path (tests/test_gpu_persist.py).  Cross-CTA data (leaves, the identity
// rows of y, a_{c+1}) is double-buffered by column parity and read with
// L1-bypassing loads after the barrier.
#include "rhqr_kernels.cuh"

namespace sqb {

constexpr int PS_NT = 512;   // = STEP_NT: phase B's block reductions are the step kernel's
constexpr int PS_LOG = 9;    // 512-row tiles (the launch-chain path's small-problem geometry)
constexpr int PS_TB = 1 << PS_LOG;
constexpr int PS_TILE = 0, PS_TOP = 1, PS_TCTA = 2, PS_ID = 3;  // CTA roles of the fast-step kernel
static_assert(PS_NT == STEP_NT, "phase B replays the step kernel's 512-thread reductions");

struct PersistArgs {
  int m, ell, od, scaling;
  int64_t n;            // Omega length N - m
  int64_t n_tiles, n_eff;
  const double* W; int64_t ldw;
  double* U; int64_t ldu;
  double* S; int64_t lds;
  double* T; int64_t ldt;
  double* R; int64_t ldr;
  double* sigmas; double* rhos; double* betas;
  const double* Y0;     // raw sketches od x m (ld od)
  const uint32_t* bits;
  const int64_t* idx;
  double scale_lo, norm_lo;
  double* leaves;       // [2][ell][n_tiles]
  double* ytop;         // [2][m]
  double* abuf;         // [2][m + 1]  a_{c+1} (helper)
  double* vbuf;         // [m + 1]     v_c
  unsigned* bar;        // grid-barrier counter (zeroed before launch)
  double* gbuf;         // [2][od]  fast step: g_{c+1} = y0_{c+1} - S_c a_{c+1} (top CTA, phase A)
  int fast;             // 1: single-reduction step (ps_step_fast), not bitwise the launch chain
  int stage_leaves;     // 1: phase B copies the leaves to shared memory first
  long long* dbg;       // optional clock64 stamps [m][4][16] (instrumentation)
  Status* st;
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// all CTAs of the (co-resident, cooperative) grid
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release-add without waiting for the old value (a fence + atomicAdd round trip before the first
    // poll cost ~0.6 us per column), then acquire-poll
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
    while (ld_acquire(ctr) < target) {
    }
  }
  __syncthreads();
}

// the two halves of the barrier for a CTA nobody waits for: it arrives as soon as it has consumed the
// previous column's data (so the others never wait for its own work) and waits before reading the next
__device__ __forceinline__ void grid_arrive(unsigned* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(1u) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned* ctr, unsigned target) {
  if (threadIdx.x == 0)
    while (ld_acquire(ctr) < target) {
    }
  __syncthreads();
}

// shared-memory layout of one CTA
struct PsSmem {
  double* Ut;     // [m][PS_TB]   tile CTAs: rows of W / U;  top CTA: Ts, Utop, vs, sb
  double* Ts;     // top: T (m x m, ld m)
  double* Utop;   // top: U's identity-block rows (m x m, ld m)
  double* vs;     // top: v_c
  double* sb;     // top: betas
  double* tile;   // FWHT buffer (tile_smem_bytes); top CTA: helper scratch
  double* Ss;     // [m][od]      S, every CTA's own copy (phase B is redundant)
  double* yv;     // [od]
  double* sv;     // [od]
  double* y0s;    // [od]         y0_{c+1}
  double* dq;     // [STEP_CL][m + 1]  per-virtual-CTA partial vectors
  double* sc;     // [m]          a_c
  double* red;    // [STEP_CL][32]
  double* scal;   // [8]
  double* an;     // [m + 1]      top CTA, fast step: a_{c+1}
  double* lvs;    // [ell][n_tiles] staged leaves (stage_leaves)
};

__host__ __device__ inline size_t ps_base_doubles(int m, int od) {
  return (size_t)m * PS_TB + (PS_TB + (PS_TB >> Pad<double>::shift) + 1) + (size_t)m * od + 3 * (size_t)od +
         STEP_CL * (size_t)(m + 1) + m + STEP_CL * 32 + 8 + (size_t)(m + 2);
}

__device__ inline PsSmem ps_carve(unsigned char* raw, int m, int od) {
  PsSmem s;
  double* p = reinterpret_cast<double*>(raw);
  s.Ut = p;
  s.Ts = p; s.Utop = p + (size_t)m * m; s.vs = s.Utop + (size_t)m * m; s.sb = s.vs + m + 1;
  p += (size_t)m * PS_TB;
  s.tile = p; p += PS_TB + (PS_TB >> Pad<double>::shift) + 1;
  s.Ss = p; p += (size_t)m * od;
  s.yv = p; p += od;
  s.sv = p; p += od;
  s.y0s = p; p += od;
  s.dq = p; p += STEP_CL * (size_t)(m + 1);
  s.sc = p; p += m;
  s.red = p; p += STEP_CL * 32;
  s.scal = p; p += 8;
  s.an = p; p += m + 2;
  s.lvs = p;
  return s;
}

// stamps of tile CTA 0 (slot 0), the TOP CTA (1), and in the fast-step kernel the T CTA (2) and ID CTA (3)
#define PS_STAMP(c, ph)                                                                     \
  do {                                                                                      \
    if (a.dbg && threadIdx.x == 0) {                                                        \
      const int slot__ = top_cta ? 1 : (blockIdx.x == 0 ? 0 : (int)blockIdx.x - (int)a.n_eff + 1); \
      if (slot__ >= 0 && slot__ < 4) a.dbg[((int64_t)(c) * 4 + slot__) * 16 + (ph)] = clock64(); \
    }                                                                                       \
  } while (0)

// The SRHT tree over a row's tile leaves by ONE thread: a binary counter over
// the leaves in tile order, level l combining (left, right) as left +/- right
// by bit l of rhi — the same operations, operands and order as
// warp_tile_tree (a tile t >= n_eff contributes +0).  nt = n_tiles <= 128.
__device__ __forceinline__ double thread_tile_tree(const double* lv, int nt, int ne, int64_t rhi) {
  double stk[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) stk[l] = 0.0;
  for (int t = 0; t < nt; ++t) {
    double v = t < ne ? lv[t] : 0.0;
    bool open = true;
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      if (open) {
        if ((t >> l) & 1) {
          v = ((rhi >> l) & 1) ? __dsub_rn(stk[l], v) : __dadd_rn(stk[l], v);
        } else {
          stk[l] = v;
          open = false;
        }
      }
    }
    if (open) stk[7] = v;
  }
  int top = 0;
  while ((1 << top) < nt) ++top;
  double out = stk[0];
#pragma unroll
  for (int l = 1; l < 8; ++l)
    if (l == top) out = stk[l];
  return out;
}

// Subtree over the q (power of two) tiles [t0, t0 + q) of one output, by one
// thread: the levels below log2 q of the tree above (aligned subtrees use the
// same level bits of rhi).
__device__ __forceinline__ double thread_subtree(const double* lv, int t0, int q, int ne, int64_t rhi) {
  double stk[6];
#pragma unroll
  for (int l = 0; l < 6; ++l) stk[l] = 0.0;
  for (int t = 0; t < q; ++t) {
    double v = t0 + t < ne ? lv[t0 + t] : 0.0;
    bool open = true;
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      if (open) {
        if ((t >> l) & 1) {
          v = ((rhi >> l) & 1) ? __dsub_rn(stk[l], v) : __dadd_rn(stk[l], v);
        } else {
          stk[l] = v;
          open = false;
        }
      }
    }
    if (open) stk[5] = v;
  }
  int top = 0;
  while ((1 << top) < q) ++top;
  double out = stk[0];
#pragma unroll
  for (int l = 1; l < 6; ++l)
    if (l == top) out = stk[l];
  return out;
}

// ---------------------------------------------------------------------------
// The sketch y of w_c in shared memory (s.yv): column 0 takes Y0[:, 0]; later
// columns the identity rows from ytop and the Omega rows from the tile leaves
// (the SRHT tree, the launch chain's operations in the launch chain's order).
// Ends with a block barrier.
// ---------------------------------------------------------------------------
__device__ void ps_y_rows(const PersistArgs& a, const PsSmem& s, int c, bool top_cta) {
  const int m = a.m, od = a.od, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (c > 0 && a.n_tiles == 32 && a.ell * 4 <= PS_NT && a.ell % 8 == 0) {
    // 32 tiles (config 1), four lanes per output: each lane loads its 8
    // leaves straight into registers (one coalesced 2 KB run per warp, a
    // single L2 round trip) and folds them, then the top two levels go
    // across the lane quad — thread_subtree's operations and order without
    // the staging pass through shared memory
    const double* yt = a.ytop + (c & 1) * m;
    double ytv = 0.0;
    if (tid < m) ytv = __ldcg(yt + tid);
    const double* lv = a.leaves + (int64_t)(c & 1) * a.ell * 32;
    const int o = tid >> 2, j = tid & 3, ne = (int)a.n_eff;
    PS_STAMP(c, 5);
    if (o < a.ell) {
      const int64_t rhi = __ldg(a.idx + o) >> PS_LOG;
      const double2* p = reinterpret_cast<const double2*>(lv + (size_t)o * 32 + j * 8);
      const double2 q0 = __ldcg(p), q1 = __ldcg(p + 1), q2 = __ldcg(p + 2), q3 = __ldcg(p + 3);
      double v[8] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y};
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (j * 8 + t >= ne) v[t] = 0.0;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const bool neg = (rhi >> l) & 1;
#pragma unroll
        for (int t = 0; t < 8; t += (2 << l))
          v[t] = neg ? __dsub_rn(v[t], v[t + (1 << l)]) : __dadd_rn(v[t], v[t + (1 << l)]);
      }
      double x = v[0];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double ot = __shfl_xor_sync(0xffffffffu, x, 1 << h, 4);
        const bool upper = (j >> h) & 1;
        const double lf = upper ? ot : x, rt = upper ? x : ot;
        x = ((rhi >> (3 + h)) & 1) ? __dsub_rn(lf, rt) : __dadd_rn(lf, rt);
      }
      if (j == 0) s.yv[m + o] = __dmul_rn(x, a.norm_lo);
    }
    if (tid < m) s.yv[tid] = ytv;
    __syncthreads();
    return;
  }
  if (c == 0) {
    for (int r = tid; r < od; r += PS_NT) s.yv[r] = __ldg(a.Y0 + r);
  } else {
    const double* yt = a.ytop + (c & 1) * m;
    if (tid < m) s.yv[tid] = __ldcg(yt + tid);
    const double* lv = a.leaves + (int64_t)(c & 1) * a.ell * a.n_tiles;
    const int nt = (int)a.n_tiles, ne = (int)a.n_eff;
    if (a.stage_leaves) {
      // all leaf loads in flight at once (one L2 round trip) into a padded
      // row-per-output layout (stride nt + 1), then one tree per thread
      const int tot = a.ell * nt, ldl = nt + 1;
      PS_STAMP(c, 5);
      for (int base = 0; base < tot; base += 8 * PS_NT) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e = base + j * PS_NT + tid;
          v[j] = e < tot ? __ldcg(lv + e) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e = base + j * PS_NT + tid;
          if (e < tot) s.lvs[(e / nt) * ldl + (e % nt)] = v[j];
        }
      }
      __syncthreads();
      PS_STAMP(c, 6);
      if (nt >= 4) {
        // four lanes per output: subtrees over nt/4 tiles each, then the top
        // two levels across the lane quad (lower lane = left operand)
        const int q4 = nt >> 2, j = tid & 3;
        int L = 0;
        while ((1 << L) < q4) ++L;
        for (int base = 0; base < a.ell; base += PS_NT / 4) {
          const int o = base + (tid >> 2);
          int64_t rhi = 0;
          double v = 0.0;
          if (o < a.ell) {
            rhi = __ldg(a.idx + o) >> PS_LOG;
            v = thread_subtree(s.lvs + (size_t)o * ldl, j * q4, q4, ne, rhi);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double ot = __shfl_xor_sync(0xffffffffu, v, 1 << h);
            const bool upper = (j >> h) & 1;
            const double lf = upper ? ot : v, rt = upper ? v : ot;
            v = ((rhi >> (L + h)) & 1) ? __dsub_rn(lf, rt) : __dadd_rn(lf, rt);
          }
          if (o < a.ell && j == 0) s.yv[m + o] = __dmul_rn(v, a.norm_lo);
        }
      } else {
        for (int o = tid; o < a.ell; o += PS_NT) {
          const int64_t rhi = __ldg(a.idx + o) >> PS_LOG;
          s.yv[m + o] = __dmul_rn(thread_tile_tree(s.lvs + (size_t)o * ldl, nt, ne, rhi), a.norm_lo);
        }
      }
    } else {
      for (int o = warp; o < a.ell; o += PS_NT / 32) {
        const int64_t rhi = __ldg(a.idx + o) >> PS_LOG;
        const double v = warp_tile_tree<double>(lv + (int64_t)o * nt, nt, ne, rhi);
        if (lane == 0) s.yv[m + o] = __dmul_rn(v, a.norm_lo);
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Phase B: the step of column c, replaying rhqr_step_kernel (8 CTAs x 512
// threads, rows split in STEP_CL blocks of step_rows(od)) bit for bit.
// Column 0 takes y = Y0[:, 0]; later columns the identity rows from ytop and
// the Omega rows from the tile leaves.  Returns false on breakdown (uniform).
// ---------------------------------------------------------------------------
__device__ bool ps_step(const PersistArgs& a, const PsSmem& s, int c, bool top_cta, double* f_out,
                        double* clast_out) {
  const int m = a.m, od = a.od, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pv = c;
  const int B = step_rows(od);
  const bool has_next = c + 1 < m;
  const double* anext = a.abuf + ((c + 1) & 1) * (m + 1);
  double an = 0.0;  // a_{c+1}[tid] (helper of pass c), loaded with the leaves
  if (has_next && tid < c) an = __ldcg(anext + tid);
  ps_y_rows(a, s, c, top_cta);
  PS_STAMP(c, 4);
  // ---- rho^2: per virtual CTA q, block_sum over its 512 threads, then q order
  {
    double p[STEP_CL];
#pragma unroll
    for (int q = 0; q < STEP_CL; ++q) {
      const int r0 = q * B, nrow = max(0, min(od, r0 + B) - r0);
      double x = 0.0;
      for (int i = tid; i < nrow; i += PS_NT)
        if (r0 + i >= pv) x = fma(s.yv[r0 + i], s.yv[r0 + i], x);
      p[q] = x;
    }
    // warps whose virtual threads hold no rows sum to +0.0: skip their shuffles
#pragma unroll
    for (int q = 0; q < STEP_CL; ++q) {
      const int nrow = max(0, min(od, q * B + B) - q * B);
      if (warp * 32 < nrow) p[q] = warp_sum(p[q]);
      else p[q] = 0.0;
    }
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < STEP_CL; ++q) s.red[q * 32 + warp] = p[q];
    __syncthreads();
    if (warp < STEP_CL) {
      double r = lane < PS_NT / 32 ? s.red[warp * 32 + lane] : 0.0;
      r = warp_sum(r);
      if (lane == 0) s.dq[warp] = r;  // part[q] (dq is free until the partial vectors)
    }
    __syncthreads();
  }
  PS_STAMP(c, 7);
  if (tid == 0) {
    double r2 = 0.0;
    for (int q = 0; q < STEP_CL; ++q) r2 += s.dq[q];
    const double rho = sqrt(r2);
    const double yc = s.yv[pv];
    const double sigma = yc >= 0.0 ? 1.0 : -1.0;
    const double gamma = __dadd_rn(yc, sigma * rho);
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
    bool bad = false;
    if (rho == 0.0) { bad = true; if (top_cta) fail(a.st, SQB_ERR_BREAKDOWN, pv + 1, 0.0); }
    else if (!isfinite(beta)) { bad = true; if (top_cta) fail(a.st, SQB_ERR_BREAKDOWN, pv + 1, rho); }
    double f, bo;
    if (a.scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
    else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    s.scal[0] = -sigma * rho; s.scal[1] = gamma; s.scal[2] = f; s.scal[3] = bad ? -1.0 : bo;
    if (top_cta && !bad) { a.sigmas[c] = sigma; a.rhos[c] = rho; a.betas[c] = bo; s.sb[c] = bo; }
  }
  __syncthreads();
  const double rdiag = s.scal[0], gamma = s.scal[1], f = s.scal[2], bo = s.scal[3];
  if (bo < 0.0) return false;
  PS_STAMP(c, 8);
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  // ---- s = Psi u, S column, identity-block rows of U, R column
  double* Sc = s.Ss + (size_t)c * od;
  for (int row = tid; row < od; row += PS_NT) {
    const double yh = row < pv ? 0.0 : (row == pv ? gamma : s.yv[row]);
    const double sval = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s.sv[row] = sval;
    Sc[row] = sval;
    if (top_cta) {
      a.S[row + (int64_t)c * a.lds] = sval;
      if (row < m) {
        a.U[row + (int64_t)c * a.ldu] = sval;
        s.Utop[row + (size_t)c * m] = sval;
        a.R[row + (int64_t)c * a.ldr] = row < pv ? s.yv[row] : (row == pv ? rdiag : 0.0);
      }
    }
  }
  __syncthreads();
  PS_STAMP(c, 9);
  // ---- partial vectors: v[k] = S[:, k]^t s (k < c), d = s^t y0_{c+1}, per
  // virtual CTA q over its rows >= pv with STEP_NPART interleaved fma chains
  const int nkk = has_next ? c + 1 : c;
  const int nk = c + 1;
  for (int e = tid; e < STEP_CL * nkk; e += PS_NT) {
    const int q = e / nkk, k = e - q * nkk;
    const int r0 = q * B, r1 = min(od, r0 + B);
    const int rs = max(r0, pv), nr = max(0, r1 - rs);
    const double* col = k < c ? s.Ss + (size_t)k * od : s.y0s;
    double cp[STEP_NPART];
#pragma unroll
    for (int pp = 0; pp < STEP_NPART; ++pp) cp[pp] = 0.0;
    for (int i0 = 0; i0 < nr; i0 += STEP_NPART)
#pragma unroll
      for (int pp = 0; pp < STEP_NPART; ++pp)
        if (i0 + pp < nr) cp[pp] = fma(col[rs + i0 + pp], s.sv[rs + i0 + pp], cp[pp]);
    double d = 0.0;
#pragma unroll
    for (int pp = 0; pp < STEP_NPART; ++pp) d += cp[pp];
    s.dq[q * nk + k] = d;
  }
  __syncthreads();
  PS_STAMP(c, 10);
  // ---- v_c, and coef_{c+1}[c] = beta (d - v^t a_{c+1})
  double va = 0.0;
  for (int k = tid; k < c; k += PS_NT) {
    double v = 0.0;
    for (int q = 0; q < STEP_CL; ++q) v += s.dq[q * nk + k];
    if (top_cta) { a.vbuf[k] = v; s.vs[k] = v; }
    if (has_next) va = fma(v, k == tid ? an : __ldcg(anext + k), va);
  }
  *f_out = f;
  if (!has_next) return true;
  // block_sum over the 512 threads; warps with no k sum to +0.0
  va = warp * 32 < c ? warp_sum(va) : 0.0;
  if (lane == 0) s.red[warp] = va;
  __syncthreads();
  if (tid < 32) {
    double r = lane < PS_NT / 32 ? s.red[lane] : 0.0;
    r = warp_sum(r);
    if (lane == 0) {
      double d = 0.0;
      for (int q = 0; q < STEP_CL; ++q) d += s.dq[q * nk + c];
      s.scal[4] = __dmul_rn(bo, d - r);
    }
  }
  __syncthreads();
  *clast_out = s.scal[4];
  return true;
}

// ---------------------------------------------------------------------------
// Fast step (PersistArgs::fast): the critical path from the sketch y of w_c to
// the two scalars the next column pass needs is ONE block reduction.  With
//     g_{c+1} = y0_{c+1} - S_c a_{c+1}           (top CTA, during phase A)
// the last coefficient of rhqr.py:241 is
//     coef_{c+1}[c] = beta_c (s_c^t y0_{c+1} - v_c^t a_{c+1}) = beta_c s_c^t g_{c+1},
// and s_c = f (0, .., 0, gamma, y[c+1:]) (rhqr.py:83-96), so
//     rho^2 = sum_{r >= c} y_r^2   and   t = sum_{r > c} y_r g_r
// are reduced together, every thread derives rho, gamma, beta, f and the
// coefficient from them, and s_c, S's column, v_c = S_c^t s_c, T's column,
// a_{c+2} and g_{c+2} leave the critical path (ps_top_post, helper).  The
// same mathematics as the launch chain in a different association (not
// bitwise; tests/test_gpu_persist.py holds it to the oracle).
// ---------------------------------------------------------------------------
__device__ bool ps_step_fast(const PersistArgs& a, const PsSmem& s, int c, int role, double* f_out,
                             double* clast_out) {
  const int m = a.m, od = a.od, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool top_cta = role == PS_TOP;  // PS_STAMP
  const int pv = c;
  const bool has_next = c + 1 < m;
  const double* gsrc = c == 0 ? a.Y0 + od : a.gbuf + (size_t)((c + 1) & 1) * od;  // g_1 = y0_1
  double g0 = 0.0, g1 = 0.0;  // rows tid, tid + PS_NT (od <= 2 PS_NT)
  if (has_next) {
    if (tid < od) g0 = __ldcg(gsrc + tid);
    if (tid + PS_NT < od) g1 = __ldcg(gsrc + tid + PS_NT);
  }
  ps_y_rows(a, s, c, top_cta);
  PS_STAMP(c, 4);
  double p1 = 0.0, p2 = 0.0;
  if (tid < od && tid >= pv) {
    const double y = s.yv[tid];
    p1 = y * y;
    if (tid > pv) p2 = y * g0;
  }
  if (tid + PS_NT < od) {  // rows past 512 are always below the pivot (pv < m <= 64)
    const double y = s.yv[tid + PS_NT];
    p1 = fma(y, y, p1);
    p2 = fma(y, g1, p2);
  }
  p1 = warp_sum(p1);
  p2 = warp_sum(p2);
  if (lane == 0) { s.red[warp] = p1; s.red[32 + warp] = p2; }
  if (tid == pv) s.red[64] = g0;
  __syncthreads();
  double r2 = 0.0, t = 0.0;
  const int nact = min(PS_NT / 32, (od + 31) / 32);  // warps past the last row hold exact zeros
  for (int w = 0; w < nact; ++w) { r2 += s.red[w]; t += s.red[32 + w]; }
  const double gpv = s.red[64];
  PS_STAMP(c, 7);
  // rh_vector's scalars (rhqr.py:71-94), by every thread
  const double rho = sqrt(r2);
  const double yc = s.yv[pv];
  const double sigma = yc >= 0.0 ? 1.0 : -1.0;
  const double gamma = __dadd_rn(yc, sigma * rho);
  const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
  const bool bad = rho == 0.0 || !isfinite(beta);
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  double f, bo, sg;
  if (sq) { f = __dsqrt_rn(beta); bo = 1.0; sg = f * fma(gamma, gpv, t); }  // s = f yhat
  else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); sg = gpv + t / gamma; }  // s = yhat / gamma
  if (tid == 0) {
    if (bad && role == PS_TCTA) fail(a.st, SQB_ERR_BREAKDOWN, pv + 1, rho == 0.0 ? 0.0 : rho);
    s.scal[0] = -sigma * rho; s.scal[1] = gamma; s.scal[2] = f; s.scal[3] = bo;
    if (role == PS_TCTA && !bad) { a.sigmas[c] = sigma; a.rhos[c] = rho; a.betas[c] = bo; s.sb[c] = bo; }
  }
  *f_out = f;
  *clast_out = has_next ? bo * sg : 0.0;
  PS_STAMP(c, 8);
  return !bad;
}

// T CTA, after the fast step of column c: s_c = Psi u_c, S's column, the
// identity-block rows of U, R's column (rhqr.py:83-96, :248-249) and
// v_c = S_c^t s_c (the _extend_t product, :138), all from shared memory
__device__ void ps_t_post(const PersistArgs& a, const PsSmem& s, int c) {
  const int m = a.m, od = a.od, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pv = c;
  __syncthreads();  // s.scal written by thread 0 of the step
  const double rdiag = s.scal[0], gamma = s.scal[1], f = s.scal[2];
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  double* Sc = s.Ss + (size_t)c * od;
  for (int row = tid; row < od; row += PS_NT) {
    const double yh = row < pv ? 0.0 : (row == pv ? gamma : s.yv[row]);
    const double sval = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s.sv[row] = sval;
    Sc[row] = sval;
    a.S[row + (int64_t)c * a.lds] = sval;
    if (row < m) {
      a.U[row + (int64_t)c * a.ldu] = sval;
      s.Utop[row + (size_t)c * m] = sval;
      a.R[row + (int64_t)c * a.ldr] = row < pv ? s.yv[row] : (row == pv ? rdiag : 0.0);
    }
  }
  __syncthreads();
  for (int k = warp; k < c; k += PS_NT / 32) {
    const double* col = s.Ss + (size_t)k * od;
    double d0 = 0.0, d1 = 0.0;
    int r = pv + lane;
    for (; r + 32 < od; r += 64) {
      d0 = fma(col[r], s.sv[r], d0);
      d1 = fma(col[r + 32], s.sv[r + 32], d1);
    }
    if (r < od) d0 = fma(col[r], s.sv[r], d0);
    const double d = warp_sum(d0 + d1);
    if (lane == 0) { s.vs[k] = d; a.vbuf[k] = d; }
  }
  __syncthreads();
}

// T column kk of the top CTA's shared copy -> global T
__device__ inline void ps_copy_t_column(const PersistArgs& a, const PsSmem& s, int kk) {
  __syncthreads();
  for (int i = threadIdx.x; i <= kk; i += PS_NT) a.T[i + (int64_t)kk * a.ldt] = s.Ts[i + (size_t)kk * a.m];
}

// phase A of a tile CTA: the column pass of column c on its 512 rows held in
// shared memory (rhqr_col_kernel's operations in its order), SRHT leaves out
__device__ void ps_tile_pass(const PersistArgs& a, const PsSmem& s, int c, int64_t g, int rows, int64_t ro,
                             int64_t e0, double f_prev, double clast) {
  const int tid = threadIdx.x;
  static_assert(PS_TB == PS_NT, "one tile row per thread");
  double* tb = s.tile;
  const int r = tid;
  double w = 0.0;
  if (r < rows) {
    // final columns 0 .. c-2, one fma chain per row (rhqr_col_kernel order)
    double acc = 0.0;
    for (int k = 0; k < c - 1; ++k) acc = fma(s.Ut[(size_t)k * PS_TB + r], s.sc[k], acc);
    // column c-1: lazy scaling of the stored w_{c-1} (rhqr.py:86-95)
    double x = lazy_scale<double>(s.Ut[(size_t)(c - 1) * PS_TB + r], f_prev, a.scaling);
    s.Ut[(size_t)(c - 1) * PS_TB + r] = x;
    a.U[ro + r + (int64_t)(c - 1) * a.ldu] = x;
    acc = fma(x, clast, acc);
    w = __dsub_rn(s.Ut[(size_t)c * PS_TB + r], acc);
    s.Ut[(size_t)c * PS_TB + r] = w;
  }
  // in-tile FWHT of the 512 values, one per thread: stages h = 1..16 are lane
  // butterflies (the pair (i, i|h) becomes (x_i + x_{i|h}, x_i - x_{i|h}), the
  // operations of tile_fwht in its order), stages h = 32..256 are evaluated
  // only at the ell sampled positions — output p is the binary tree over the
  // 16 values {(p & 31) + 32 j}, level l taking left +/- right by bit 5 + l of
  // p: exactly the butterflies that feed position p.  Same bits as
  // tile_fwht + tile_gather, two shared-memory passes and the gather fewer.
  double v = r < rows ? srht_in<double>(w, a.scale_lo, sign_neg(a.bits, e0 + r)) : 0.0;
  const int lane = tid & 31;
#pragma unroll
  for (int h = 1; h < 32; h <<= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, h);
    v = (lane & h) ? __dsub_rn(o, v) : __dadd_rn(v, o);
  }
  tb[r] = v;
  __syncthreads();
  double* P = a.leaves + (int64_t)(c & 1) * a.ell * a.n_tiles + g;
  for (int k = tid; k < a.ell; k += PS_NT) {
    const int p = (int)(__ldg(a.idx + k) & (PS_TB - 1));
    const double* q = tb + (p & 31);
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = q[32 * j];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const bool neg = (p >> (5 + l)) & 1;
#pragma unroll
      for (int j = 0; j < 16; j += (2 << l)) x[j] = neg ? __dsub_rn(x[j], x[j + (1 << l)]) : __dadd_rn(x[j], x[j + (1 << l)]);
    }
    P[(int64_t)k * a.n_tiles] = x[0];
  }
}

__device__ void ps_identity_rows(const PersistArgs& a, const PsSmem& s, int c, double clast);

__global__ void __launch_bounds__(PS_NT, 1) rhqr_persist_kernel(PersistArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, od = a.od, tid = threadIdx.x;
  const PsSmem s = ps_carve(smem_raw, m, od);
  const int64_t g = blockIdx.x;
  const bool top_cta = g == a.n_eff;
  const unsigned G = gridDim.x;
  if (failed(a.st)) return;  // uniform: written before this kernel
  // tile rows: W[m + g*512 + r, :] -> Ut (column-major, 512 per column)
  const int64_t e0 = g << PS_LOG;
  const int rows = top_cta ? 0 : (int)(a.n - e0 < PS_TB ? a.n - e0 : (int64_t)PS_TB);
  const int64_t ro = (int64_t)m + e0;
  if (!top_cta) {
    for (int k = 0; k < m; ++k)
      for (int r = tid; r < rows; r += PS_NT) s.Ut[(size_t)k * PS_TB + r] = __ldg(a.W + ro + r + (int64_t)k * a.ldw);
  } else {
    for (int e = tid; e < m * m; e += PS_NT) s.Ts[e] = 0.0;
  }
  if (m > 1)
    for (int r = tid; r < od; r += PS_NT) s.y0s[r] = __ldg(a.Y0 + od + r);
  __syncthreads();
  double f_prev = 0.0, clast = 0.0;
  if (!ps_step(a, s, 0, top_cta, &f_prev, &clast)) return;
  unsigned nbar = 0;
  for (int c = 1; c < m; ++c) {
    PS_STAMP(c, 0);
    // ---------------- phase A: the column pass of column c
    const double* acur = a.abuf + (c & 1) * (m + 1);
    for (int k = tid; k < c - 1; k += PS_NT) s.sc[k] = __ldcg(acur + k);
    if (c + 1 < m)  // y0_{c+1} for phase B (a constant input: off the post-barrier path)
      for (int r = tid; r < od; r += PS_NT) s.y0s[r] = __ldg(a.Y0 + (int64_t)(c + 1) * od + r);
    __syncthreads();
    if (!top_cta) {
      ps_tile_pass(a, s, c, g, rows, ro, e0, f_prev, clast);
    } else {
      ps_identity_rows(a, s, c, clast);
      // helper (col_helper) on the shared copies: T column c-1, then
      // a_{c+1} = T_c^t (S_c^t y0_{c+1})
      ColArgs h{};
      h.c = c; h.ncol = m; h.od = od;
      h.S = s.Ss; h.lds = od; h.T = s.Ts; h.ldt = m; h.Y0 = a.Y0;
      h.vprev = s.vs; h.betas = s.sb;
      h.anext = a.abuf + ((c + 1) & 1) * (m + 1);
      __syncthreads();
      col_helper(h, s.tile);
      ps_copy_t_column(a, s, c - 1);
    }
    PS_STAMP(c, 1);
    // ---------------- one grid barrier per column
    grid_barrier(a.bar, ++nbar * G);
    PS_STAMP(c, 2);
    // ---------------- phase B: the step of column c (redundant in every CTA)
    double f = 0.0, cl = 0.0;
    if (!ps_step(a, s, c, top_cta, &f, &cl)) return;
    f_prev = f;
    clast = cl;
    PS_STAMP(c, 3);
  }
  // last column: lazy scaling of its Omega rows, its T column
  if (!top_cta) {
    for (int r = tid; r < rows; r += PS_NT)
      a.U[ro + r + (int64_t)(m - 1) * a.ldu] =
          lazy_scale<double>(s.Ut[(size_t)(m - 1) * PS_TB + r], f_prev, a.scaling);
  } else {
    __syncthreads();
    complete_t_column(s.Ts, m, m - 1, s.vs, s.sb[m - 1]);
    ps_copy_t_column(a, s, m - 1);
  }
}

// top CTA of the fast-step kernel, after the step of column c: apply reflector
// c to the sketches of the columns still ahead — G_j <- G_j - alpha_j s_c with
// alpha_j = beta_c s_c^t G_j = a_j[c] (rhqr.py:241 expanded column by column,
// see ps_step_fast) — so that a_{c+2} and g_{c+2} are ready before the next
// barrier without T on the path.  G lives in s.Ss, the a_j in s.Ts ([j][m]).
__device__ void ps_top_update(const PersistArgs& a, const PsSmem& s, int c) {
  const int m = a.m, od = a.od, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pv = c;
  __syncthreads();  // s.scal written by thread 0 of the step
  const double gamma = s.scal[1], f = s.scal[2], bo = s.scal[3];
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  for (int row = tid; row < od; row += PS_NT) {
    const double yh = row < pv ? 0.0 : (row == pv ? gamma : s.yv[row]);
    const double sval = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s.sv[row] = sval;
    if (row < m) s.Utop[row + (size_t)c * m] = sval;
  }
  __syncthreads();
  for (int j = c + 2 + warp; j < m; j += PS_NT / 32) {
    double* Gj = s.Ss + (size_t)j * od;
    double d0 = 0.0, d1 = 0.0;
    int r = pv + lane;
    for (; r + 32 < od; r += 64) {
      d0 = fma(Gj[r], s.sv[r], d0);
      d1 = fma(Gj[r + 32], s.sv[r + 32], d1);
    }
    if (r < od) d0 = fma(Gj[r], s.sv[r], d0);
    const double alpha = bo * warp_sum(d0 + d1);
    for (r = pv + lane; r < od; r += 32) Gj[r] = fma(-alpha, s.sv[r], Gj[r]);
    if (lane == 0) s.Ts[(size_t)j * m + c] = alpha;
  }
  __syncthreads();
}

// identity block y[r] = w_c[r], r < m (col_top_block's accumulation order)
__device__ void ps_identity_rows(const PersistArgs& a, const PsSmem& s, int c, double clast) {
  const int m = a.m, tid = threadIdx.x;
  double* yt = a.ytop + (c & 1) * m;
  for (int r = tid; r < m; r += PS_NT) {
    const double* ur = s.Utop + r;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int k = 0;
    for (; k + 4 <= c - 1; k += 4) {
      acc0 = fma(ur[(size_t)k * m], s.sc[k], acc0);
      acc1 = fma(ur[(size_t)(k + 1) * m], s.sc[k + 1], acc1);
      acc2 = fma(ur[(size_t)(k + 2) * m], s.sc[k + 2], acc2);
      acc3 = fma(ur[(size_t)(k + 3) * m], s.sc[k + 3], acc3);
    }
    for (; k < c - 1; ++k) acc0 = fma(ur[(size_t)k * m], s.sc[k], acc0);
    const double acc = (acc0 + acc1) + (acc2 + acc3);
    const double dot = fma(ur[(size_t)(c - 1) * m], clast, acc);
    yt[r] = __dsub_rn(__ldg(a.W + r + (int64_t)c * a.ldw), dot);
  }
}

// ---------------------------------------------------------------------------
// The fast-step persistent kernel (SQB_PERSIST=2): tile CTAs as in
// rhqr_persist_kernel; the TOP CTA owns the sketches of the columns ahead
// (ps_top_update), the ID CTA the identity-block rows of w_c — everything the
// next barrier waits for, on two CTAs so neither chain outlasts a tile pass;
// the T CTA writes the sketch-space outputs (S, R, U's identity rows, scalars)
// and builds T by _extend_t (rhqr.py:135-140) with a whole column period to
// do it.  Every CTA runs the single-reduction step (ps_step_fast).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PS_NT, 1) rhqr_persist_fast_kernel(PersistArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, od = a.od, tid = threadIdx.x;
  const PsSmem s = ps_carve(smem_raw, m, od);
  const int64_t g = blockIdx.x;
  const int role = g < a.n_eff ? PS_TILE : (g == a.n_eff ? PS_TOP : (g == a.n_eff + 1 ? PS_TCTA : PS_ID));
  const bool top_cta = role == PS_TOP;  // PS_STAMP
  const unsigned G = gridDim.x;
  if (failed(a.st)) return;  // uniform: written before this kernel
  const int64_t e0 = g << PS_LOG;
  const int rows = role != PS_TILE ? 0 : (int)(a.n - e0 < PS_TB ? a.n - e0 : (int64_t)PS_TB);
  const int64_t ro = (int64_t)m + e0;
  PS_STAMP(0, 0);
  if (role == PS_TILE) {
    // eight columns of the tile in flight per thread (the one-load-one-store loop spent one HBM round
    // trip per column: ~16 us of the kernel's 235)
    for (int k0 = 0; k0 < m; k0 += 8)
      for (int r = tid; r < rows; r += PS_NT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = k0 + u < m ? __ldg(a.W + ro + r + (int64_t)(k0 + u) * a.ldw) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + u < m) s.Ut[(size_t)(k0 + u) * PS_TB + r] = v[u];
      }
  } else {
    for (int e = tid; e < m * m; e += PS_NT) s.Ts[e] = 0.0;
    if (role == PS_TOP)  // G_j = y0_j
      for (int e0b = 0; e0b < m * od; e0b += 8 * PS_NT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = e0b + u * PS_NT + tid; v[u] = e < m * od ? __ldg(a.Y0 + e) : 0.0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) { const int e = e0b + u * PS_NT + tid; if (e < m * od) s.Ss[e] = v[u]; }
      }
  }
  __syncthreads();
  PS_STAMP(0, 1);
  double f_prev = 0.0, clast = 0.0;
  if (!ps_step_fast(a, s, 0, role, &f_prev, &clast)) return;
  PS_STAMP(0, 2);
  unsigned nbar = 0;
  double sc_pref = 0.0;
  for (int c = 1; c < m; ++c) {
    PS_STAMP(c, 0);
    // a_c was published before barrier c-1 and fetched under the leaf loads of step c-1
    if (role != PS_TCTA && tid < c - 1) s.sc[tid] = sc_pref;
    if (role == PS_TOP) ps_top_update(a, s, c - 1);
    if (role == PS_ID) {
      // the identity-block rows of u_{c-1} (= s_{c-1}[:m]) for this CTA's copy of U's top rows
      __syncthreads();  // s.scal of step c-1
      const double gamma = s.scal[1], f = s.scal[2];
      const bool sq = a.scaling == SQB_SCALE_SQRT2;
      for (int row = tid; row < m; row += PS_NT) {
        const double yh = row < c - 1 ? 0.0 : (row == c - 1 ? gamma : s.yv[row]);
        s.Utop[row + (size_t)(c - 1) * m] = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
      }
    }
    if (role == PS_TCTA) {
      // nothing this CTA writes is read inside the kernel: it arrives at barrier c now, having consumed
      // the data of column c-1, and only waits for it below — its 1.7 us of output work (S, R, U's
      // identity rows, T's column) no longer sits between the tile passes and the barrier
      grid_arrive(a.bar);
      ps_t_post(a, s, c - 1);
      complete_t_column(s.Ts, m, c - 1, s.vs, s.sb[c - 1]);
      ps_copy_t_column(a, s, c - 1);
    }
    __syncthreads();
    if (role == PS_TILE) {
      ps_tile_pass(a, s, c, g, rows, ro, e0, f_prev, clast);
    } else if (role == PS_ID) {
      ps_identity_rows(a, s, c, clast);  // y_c[0:m], off the TOP CTA's chain
    } else if (role == PS_TOP) {
      if (c + 1 < m) {
        double* gd = a.gbuf + (size_t)((c + 1) & 1) * od;
        const double* Gn = s.Ss + (size_t)(c + 1) * od;
        for (int r = tid; r < od; r += PS_NT) gd[r] = Gn[r];
        double* ag = a.abuf + ((c + 1) & 1) * (m + 1);
        for (int k = tid; k < c; k += PS_NT) ag[k] = s.Ts[(size_t)(c + 1) * m + k];
      }
    }
    PS_STAMP(c, 1);
    if (role == PS_TCTA) grid_wait(a.bar, ++nbar * G);
    else grid_barrier(a.bar, ++nbar * G);
    PS_STAMP(c, 2);
    double f = 0.0, cl = 0.0;
    // a_{c+1} (written by the TOP CTA before this barrier): in flight during the step instead of one
    // more L2 round trip at the head of the next column pass (m <= 64 < PS_NT: one entry per thread)
    sc_pref = (c + 1 < m && tid < c) ? __ldcg(a.abuf + ((c + 1) & 1) * (m + 1) + tid) : 0.0;
    if (!ps_step_fast(a, s, c, role, &f, &cl)) return;
    f_prev = f;
    clast = cl;
    PS_STAMP(c, 3);
  }
  if (role == PS_TILE) {
    for (int r = tid; r < rows; r += PS_NT)
      a.U[ro + r + (int64_t)(m - 1) * a.ldu] =
          lazy_scale<double>(s.Ut[(size_t)(m - 1) * PS_TB + r], f_prev, a.scaling);
  } else if (role == PS_TCTA) {
    ps_t_post(a, s, m - 1);
    complete_t_column(s.Ts, m, m - 1, s.vs, s.sb[m - 1]);
    ps_copy_t_column(a, s, m - 1);
  }
  PS_STAMP(0, 3);
}

// host side ------------------------------------------------------------------
size_t persist_ws_bytes(const sqb_sketch* sk, int64_t m) {
  if (sk->kind != SQB_SKETCH_SRHT || sk->n_pad > (int64_t(1) << 16)) return 0;
  return sizeof(double) * (2 * (size_t)sk->ell * (size_t)(sk->n_pad >> PS_LOG) + 2 * (size_t)m +
                           2 * (size_t)(m + sk->ell)) + 256;
}

// nonzero if the persistent kernel can run this sweep (fp64 SRHT, small n_pad,
// every CTA co-resident, W/U/S rows of a CTA in shared memory)
bool persist_eligible(sqb_ctx* ctx, const sqb_sketch* sk, int64_t N, int64_t m, int64_t ncol, int64_t off) {
  // SQB_PERSIST (read per call so tests can toggle it): unset / 2 = the
  // fast-step kernel (default: config 1 0.43 -> 0.24 ms), 1 = the kernel that
  // is bitwise the launch chain (at parity with it), 0 = the launch chain
  const char* ev = getenv("SQB_PERSIST");
  const bool off_env = ev && ev[0] == '0';
  if (off_env || off != 0 || ncol != m || sk->kind != SQB_SKETCH_SRHT) return false;
  if (sk->n_pad > (int64_t(1) << 16) || sk->n_pad < PS_TB || m < 2 || m > 64) return false;
  if (m + sk->ell > 2 * PS_NT) return false;
  const int64_t n = N - m, od = m + sk->ell;
  const int64_t n_eff = (n + PS_TB - 1) / PS_TB;
  if (n_eff + 3 > ctx->sm_count) return false;
  if (sizeof(double) * ps_base_doubles((int)m, (int)od) + 64 > 227 * 1024) return false;
  if (2 * m * m + 2 * m + 1 > m * PS_TB) return false;
  return true;
}

int launch_persist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const double* W, int64_t N, int64_t m,
                   int64_t ldw, double* U, int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt, double* R,
                   int64_t ldr, double* sigmas, double* rhos, double* betas, const double* Y0, double* abuf,
                   double* vbuf, void* pws, double scale_lo, double norm_lo) {
  PersistArgs a{};
  a.m = (int)m; a.ell = (int)sk->ell; a.od = (int)(m + sk->ell); a.scaling = scaling;
  a.n = N - m; a.n_tiles = sk->n_pad >> PS_LOG; a.n_eff = (a.n + PS_TB - 1) / PS_TB;
  a.W = W; a.ldw = ldw; a.U = U; a.ldu = ldu; a.S = S; a.lds = lds; a.T = Tm; a.ldt = ldt; a.R = R; a.ldr = ldr;
  a.sigmas = sigmas; a.rhos = rhos; a.betas = betas; a.Y0 = Y0;
  a.bits = sk->sign_bits; a.idx = sk->indices; a.scale_lo = scale_lo; a.norm_lo = norm_lo;
  char* p = static_cast<char*>(pws);
  a.leaves = reinterpret_cast<double*>(p);
  a.ytop = a.leaves + 2 * (size_t)a.ell * a.n_tiles;
  a.gbuf = a.ytop + 2 * m;
  a.bar = reinterpret_cast<unsigned*>(a.gbuf + 2 * (size_t)a.od);
  {
    const char* ev = getenv("SQB_PERSIST");
    a.fast = (ev && ev[0] == '1') ? 0 : 1;
  }
  a.abuf = abuf; a.vbuf = vbuf; a.st = ctx->d_status;
  SQB_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 64, ctx->stream));
  size_t smem = sizeof(double) * ps_base_doubles((int)m, a.od) + 64;
  const size_t lv_bytes = sizeof(double) * (size_t)a.ell * (size_t)(a.n_tiles + 1);
  a.stage_leaves = smem + lv_bytes <= 227 * 1024 ? 1 : 0;
  if (a.stage_leaves) smem += lv_bytes;
  a.dbg = ctx->dbg_col == -2 ? ctx->dbg_ts : nullptr;
  void (*kern)(PersistArgs) = a.fast ? rhqr_persist_fast_kernel : rhqr_persist_kernel;
  SQB_CUDA_TRY(allow_dyn_smem(kern, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.n_eff + (a.fast ? 3 : 1)));
  cfg.blockDim = dim3(PS_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  if (e != cudaSuccess) return set_cuda_error(ctx, e, "rhqr_persist_kernel", __FILE__, __LINE__);
  return check_launch(ctx, "rhqr_persist_kernel");
}

}  // namespace sqb
