#include <cstdlib>
#include <type_traits>
// recRHQR on the device (rec_rhqr, rhqr.py:368-395):
//   Z = Psi W (one sketch of all columns; K2 DMMA for a Gaussian Omega),
//   K5  householder_qr(Z) in the high precision (baselines.py:33-89), one CTA,
//   Mfac = triu(T^t S^t Z), zero-diagonal check (rhqr.py:387-391),
//   K6  U2 = W2 Mfac^{-1} by row-wise forward substitution (right_tri_solve,
//       linalg.py:119-129), streamed over the n-m rows,
//   U = [S[:m]; round_to(U2, low)].
#include <algorithm>
#include <cfloat>

#include "pdl.cuh"
#include "sketch.cuh"
#include "vec.cuh"

namespace sqb {

constexpr int HQR_NT = 1024;

// K5: left-looking Householder QR with compact T of Z (od x m), fp64 throughout.
// Writes S = U_z (od x m), T, R (m x m), sigmas/rhos/betas.
// RES: S and T live in shared memory for the whole factorization (every
// column re-reads all previous reflectors and T: shared-memory latency instead
// of L2 latency on the dependent chain) and are written out at the end.
template <bool RES>
__global__ void __launch_bounds__(HQR_NT)
hqr_kernel(const double* __restrict__ Z, int64_t ldz, int od, int m, int scaling, double* Sg,
           int64_t ldsg, double* Tg, int64_t ldtg, double* R, int64_t ldr, double* sig, double* rhos,
           double* bets, Status* st) {
  extern __shared__ double sm[];
  double* w = sm;          // [od]
  double* g = w + od;      // [m]
  double* cf = g + m;      // [m]
  double* red = cf + m;    // [32]
  __shared__ double scal[4];
  if (failed(st)) return;
  double* S = RES ? red + 32 : Sg;
  const int64_t lds = RES ? od : ldsg;
  double* T = RES ? S + (int64_t)od * m : Tg;
  const int64_t ldt = RES ? m : ldtg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = HQR_NT / 32;
  for (int e = tid; e < m * m; e += HQR_NT) {
    T[(e % m) + (int64_t)(e / m) * ldt] = 0.0;
    R[(e % m) + (int64_t)(e / m) * ldr] = 0.0;
  }
  // Z[:, c+1] is fetched while column c is processed (od <= HQR_NT: one
  // entry per thread), so the global load is off the per-column chain
  const bool pre = od <= HQR_NT;
  double zpre = (pre && tid < od) ? Z[tid] : 0.0;
  for (int c = 0; c < m; ++c) {
    if (pre) {
      if (tid < od) w[tid] = zpre;
      if (tid < od && c + 1 < m) zpre = Z[tid + (int64_t)(c + 1) * ldz];
    } else {
      for (int r = tid; r < od; r += HQR_NT) w[r] = Z[r + (int64_t)c * ldz];
    }
    __syncthreads();
    if (c > 0) {
      // coef = T[:c,:c]^t (U[:, :c]^t w); w = w - U[:, :c] coef   (baselines.py:57-59)
      for (int k = warp; k < c; k += nw) {
        const double* uk = S + (int64_t)k * lds;
        double d = 0.0;
        for (int r = k + lane; r < od; r += 32) d = fma(uk[r], w[r], d);
        d = warp_sum(d);
        if (lane == 0) g[k] = d;
      }
      __syncthreads();
      for (int j = warp; j < c; j += nw) {
        double d = 0.0;
        for (int k = lane; k <= j; k += 32) d = fma(T[k + (int64_t)j * ldt], g[k], d);
        d = warp_sum(d);
        if (lane == 0) cf[j] = d;
      }
      __syncthreads();
      for (int r = tid; r < od; r += HQR_NT) {
        double d = 0.0;
        const int kmax = min(c, r + 1);  // U[r, k] = 0 for k > r
        for (int k = 0; k < kmax; ++k) d = fma(S[r + (int64_t)k * lds], cf[k], d);
        w[r] = w[r] - d;
      }
      __syncthreads();
    }
    double p = 0.0;
    for (int r = c + tid; r < od; r += HQR_NT) p = fma(w[r], w[r], p);
    const double rho = sqrt(block_sum(p, red));
    if (tid == 0) {
      const double sigma = w[c] >= 0.0 ? 1.0 : -1.0;
      const double gamma = __dadd_rn(w[c], sigma * rho);
      const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
      double f, bo;
      if (scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
      else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
      scal[0] = sigma; scal[1] = gamma; scal[2] = f; scal[3] = bo;
      if (rho == 0.0) fail(st, SQB_ERR_BREAKDOWN, c + 1, 0.0);
      sig[c] = sigma; rhos[c] = rho; bets[c] = bo;
      R[c + (int64_t)c * ldr] = -sigma * rho;
    }
    __syncthreads();
    if (rho == 0.0) return;
    const double gamma = scal[1], f = scal[2], bo = scal[3];
    const bool sq = scaling == SQB_SCALE_SQRT2;
    for (int r = tid; r < od; r += HQR_NT) {
      const double uh = r < c ? 0.0 : (r == c ? gamma : w[r]);
      S[r + (int64_t)c * lds] = sq ? __dmul_rn(uh, f) : __ddiv_rn(uh, f);
      if (r < c) R[r + (int64_t)c * ldr] = w[r];
    }
    __syncthreads();
    if (c > 0) {
      // T[:c, c] = -beta T[:c,:c] (U[:, :c]^t u)   (baselines.py:78-81)
      const double* uc = S + (int64_t)c * lds;
      for (int k = warp; k < c; k += nw) {
        const double* uk = S + (int64_t)k * lds;
        double d = 0.0;
        for (int r = c + lane; r < od; r += 32) d = fma(uk[r], uc[r], d);  // u[r] = 0 for r < c
        d = warp_sum(d);
        if (lane == 0) g[k] = d;
      }
      __syncthreads();
      for (int i = warp; i < c; i += nw) {
        double d = 0.0;
        for (int k = i + lane; k < c; k += 32) d = fma(T[i + (int64_t)k * ldt], g[k], d);
        d = warp_sum(d);
        if (lane == 0) T[i + (int64_t)c * ldt] = __dmul_rn(-bo, d);
      }
    }
    if (tid == 0) T[c + (int64_t)c * ldt] = bo;
    __syncthreads();
  }
  if (RES) {
    for (int e = tid; e < od * m; e += HQR_NT) Sg[(e % od) + (int64_t)(e / od) * ldsg] = S[e];
    for (int e = tid; e < m * m; e += HQR_NT) Tg[(e % m) + (int64_t)(e / m) * ldtg] = T[e];
  }
}

// Mfac[:, j] = triu(T^t (S^t Z[:, j]))  — one CTA per column j
__global__ void __launch_bounds__(256)
mfac_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ T, int64_t ldt,
            const double* __restrict__ Z, int64_t ldz, int od, int m, double* M, const Status* st) {
  extern __shared__ double g[];  // [m]
  if (failed(st)) return;
  const int j = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* zj = Z + (int64_t)j * ldz;
  for (int k = warp; k < m; k += 8) {
    const double* sk = S + (int64_t)k * lds;
    double d = 0.0;
    for (int r = k + lane; r < od; r += 32) d = fma(sk[r], zj[r], d);
    d = warp_sum(d);
    if (lane == 0) g[k] = d;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += 256) {
    double d = 0.0;
    if (i <= j)
      for (int k = 0; k <= i; ++k) d = fma(T[k + (int64_t)i * ldt], g[k], d);
    M[i + (int64_t)j * m] = d;
  }
}

// zero-diagonal check (rhqr.py:388-391): argmin |diag| < DBL_MIN -> breakdown
__global__ void mfac_check_kernel(const double* M, int m, Status* st) {
  if (failed(st)) return;
  // the reference hands Mfac to scipy's solve_triangular (linalg.py:128), which rejects non-finite entries
  // (a sketch that overflowed its storage format) with a ValueError before any arithmetic
  for (int e = threadIdx.x; e < m * m; e += blockDim.x)
    if (e % m <= e / m && !isfinite(M[e])) fail(st, SQB_ERR_NONFINITE, e / m + 1, M[e]);
  __syncthreads();
  if (threadIdx.x != 0 || failed(st)) return;
  int k = 0;
  double dmin = fabs(M[0]);
  for (int j = 1; j < m; ++j) {
    const double d = fabs(M[j + (int64_t)j * m]);
    if (d < dmin) { dmin = d; k = j; }
  }
  if (dmin < DBL_MIN) fail(st, SQB_ERR_BREAKDOWN, k + 1, -1.0);
}

// K6: U2 = W2 Mfac^{-1}: per row x, x Mfac = w by forward substitution in fp64
// (x_j = (w_j - sum_{i<j} x_i M_ij) / M_jj), x kept in registers (m <= MAXM).
template <typename T, int MAXM>
__global__ void __launch_bounds__(128)
trsm_rows_kernel(const T* __restrict__ W2, int64_t ldw, int64_t n, int m, const double* __restrict__ M,
                 T* __restrict__ U2, int64_t ldu, const Status* st) {
  extern __shared__ double sM[];  // m x m, column-major
  if (failed(st)) return;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sM[e] = M[e];
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double x[MAXM];
#pragma unroll
    for (int j = 0; j < MAXM; ++j)
      if (j < m) x[j] = (double)Lo<T>::load(W2[r + (int64_t)j * ldw]);
#pragma unroll
    for (int j = 0; j < MAXM; ++j) {
      if (j < m) {
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < j; ++i) s = fma(x[i], sM[i + j * m], s);
        x[j] = __ddiv_rn(x[j] - s, sM[j + j * m]);
      }
    }
#pragma unroll
    for (int j = 0; j < MAXM; ++j)
      if (j < m) U2[r + (int64_t)j * ldu] = Lo<T>::store(Lo<T>::from_double(x[j]));
  }
}

// generic fallback for wide m: x in global scratch (the output itself)
template <typename T>
__global__ void __launch_bounds__(128)
trsm_rows_generic_kernel(const T* __restrict__ W2, int64_t ldw, int64_t n, int m,
                         const double* __restrict__ M, T* __restrict__ U2, int64_t ldu, double* X,
                         const Status* st) {
  if (failed(st)) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < m; ++j) {
      double s = 0.0;
      for (int i = 0; i < j; ++i) s = fma(X[r + (int64_t)i * n], M[i + (int64_t)j * m], s);
      const double xj = __ddiv_rn((double)Lo<T>::load(W2[r + (int64_t)j * ldw]) - s, M[j + (int64_t)j * m]);
      X[r + (int64_t)j * n] = xj;
      U2[r + (int64_t)j * ldu] = Lo<T>::store(Lo<T>::from_double(xj));
    }
  }
}

// K6 on the tensor pipe: blocked forward substitution X Mfac = W2 (the
// LAPACK dtrsm blocking): per 64-row tile and 16-column block b,
//   X_b -= X_{<b} M_{<b,b}          (DMMA m16n8k16, one warp per 16 rows)
//   X_b  = X_b M_bb^{-1}            (16-step substitution per row, division by M_jj)
// M (padded to a multiple of 16 with an identity tail) lives in shared memory.
constexpr int TR_ROWS = 128, TR_NT = 256;

__device__ __forceinline__ void dmma16x8x16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
        "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <typename T>
__global__ void __launch_bounds__(TR_NT)
trsm_dmma_kernel(const T* __restrict__ W2, int64_t ldw, int64_t n, int m, int mp, const double* __restrict__ M,
                 T* __restrict__ U2, int64_t ldu, const Status* st) {
  extern __shared__ __align__(16) double tsm[];
  const int ld = mp + 4;            // Ms: 2-way B-fragment loads
  const int lx = mp + 1;            // Xs: odd stride -> conflict-free column-wise access
  double* Ms = tsm;                 // [mp][ld] column-major: Ms[col * ld + row]
  double* Xs = tsm + mp * ld;       // [TR_ROWS][lx] row-major
  if (failed(st)) return;
  for (int e = threadIdx.x; e < mp * mp; e += TR_NT) {
    const int r = e % mp, c = e / mp;
    Ms[c * ld + r] = (r < m && c < m) ? M[r + (int64_t)c * m] : (r == c ? 1.0 : 0.0);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nb = mp / 16;
  for (int64_t r0 = (int64_t)blockIdx.x * TR_ROWS; r0 < n; r0 += (int64_t)gridDim.x * TR_ROWS) {
    __syncthreads();
    if constexpr (sizeof(T) == 8) {
      // all of the tile's loads in flight at once (cp.async, 8-byte granules)
      for (int e = threadIdx.x; e < TR_ROWS * mp; e += TR_NT) {
        const int row = e % TR_ROWS, col = e / TR_ROWS;
        double* d = &Xs[row * lx + col];
        if (r0 + row < n && col < m) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(d);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(W2 + r0 + row + (int64_t)col * ldw));
        } else {
          *d = 0.0;
        }
      }
      asm volatile("cp.async.commit_group;\n" ::);
      asm volatile("cp.async.wait_group 0;\n" ::);
    } else {
#pragma unroll 8
      for (int e = threadIdx.x; e < TR_ROWS * mp; e += TR_NT) {
        const int row = e % TR_ROWS, col = e / TR_ROWS;
        Xs[row * lx + col] = (r0 + row < n && col < m) ? (double)Lo<T>::load(W2[r0 + row + (int64_t)col * ldw]) : 0.0;
      }
    }
    __syncthreads();
    const int wr = warp * 16;  // this warp's 16 rows in the DMMA phase
    for (int b = 0; b < nb; ++b) {
      if (b > 0) {
        double acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
        for (int kk = 0; kk < b; ++kk) {
          double a[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) a[v] = Xs[(wr + g + 8 * (v & 1)) * lx + 16 * kk + t + 4 * (v >> 1)];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            double bb[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) bb[v] = Ms[(16 * b + 8 * nt + g) * ld + 16 * kk + t + 4 * v];
            dmma16x8x16(acc[nt], a, bb);
          }
        }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              double* p = &Xs[(wr + g + 8 * h) * lx + 16 * b + 8 * nt + 2 * t + q];
              *p = *p - acc[nt][2 * h + q];
            }
      }
      __syncthreads();
      // diagonal block: one thread per row, 16-step substitution
      if (threadIdx.x < TR_ROWS) {
        double* xr = &Xs[threadIdx.x * lx + 16 * b];
        double x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = xr[j];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double* mj = &Ms[(16 * b + j) * ld + 16 * b];
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < j; ++i) s = fma(x[i], mj[i], s);
          x[j] = __ddiv_rn(x[j] - s, mj[j]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) xr[j] = x[j];
      }
      __syncthreads();
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TR_ROWS * m; e += TR_NT) {
      const int row = e % TR_ROWS, col = e / TR_ROWS;
      if (r0 + row < n) U2[r0 + row + (int64_t)col * ldu] = Lo<T>::store(Lo<T>::from_double(Xs[row * lx + col]));
    }
  }
}

// K6, fp64 storage, m <= 64: the same blocked substitution as a software
// pipeline — 64-row tiles, two shared-memory tile buffers per CTA filled by
// 16-byte cp.async (the next tile streams in while this one is solved), two
// CTAs per SM.  Tiles are column-major in shared memory (ld 72 = 8 mod 16:
// conflict-free DMMA A fragments and row-per-thread substitution); the
// diagonal blocks are solved right-looking (x_j *= 1/M_jj, then x_k -= x_j
// M_jk for k > j), the reference BLAS dtrsm order (multiply by the
// reciprocal of the diagonal).  Measured (config 3, ncu): 2.17 -> 1.56 ms.
// With the solve removed the same kernel moves its 4.3 GB in 0.68 ms
// (6.25 TB/s), so what remains is the latency of the per-tile solve chain
// (two warps run the 16-step diagonal substitutions while six wait).
constexpr int TP_ROWS = 64, TP_NT = 256, TP_LDX = 68, TP_MP = 64, TP_LDM = 68;
// + the diagonal blocks transposed (row j of block b contiguous: pairs of
// M[j, k] for the substitution, loaded two at a time)
constexpr size_t TP_SMEM = sizeof(double) * ((size_t)2 * TP_MP * TP_LDX + (size_t)TP_MP * TP_LDM + TP_MP + (size_t)TP_MP * 16);

__global__ void __launch_bounds__(TP_NT, 2)
trsm_pipe_kernel(const double* __restrict__ W2, int64_t ldw, int64_t n, int m, int mp,
                 const double* __restrict__ M, double* __restrict__ U2, int64_t ldu, const Status* st) {
  extern __shared__ __align__(16) double tps[];
  double* Ms = tps + 2 * TP_MP * TP_LDX;  // column-major, ld TP_LDM
  double* rinv = Ms + TP_MP * TP_LDM;
  double* DT = rinv + TP_MP;  // [mp/16][16][16]: DT[b][j][k] = M[16b + j, 16b + k] for k > j
  if (failed(st)) return;
  const int tid = threadIdx.x;
  for (int e = tid; e < mp * mp; e += TP_NT) {
    const int r = e % mp, c = e / mp;
    Ms[c * TP_LDM + r] = (r < m && c < m) ? M[r + (int64_t)c * m] : (r == c ? 1.0 : 0.0);
  }
  for (int e = tid; e < mp; e += TP_NT) rinv[e] = e < m ? 1.0 / M[e + (int64_t)e * m] : 1.0;
  for (int e = tid; e < mp * 16; e += TP_NT) {
    const int b = e >> 8, j = (e >> 4) & 15, k = e & 15;
    const int r = 16 * b + j, c = 16 * b + k;
    DT[e] = (k > j && r < m && c < m) ? M[r + (int64_t)c * m] : 0.0;
  }
  // padding columns m..mp-1 stay zero in both buffers (never loaded)
  for (int e = tid; e < 2 * TP_MP * TP_LDX; e += TP_NT) {
    const int c = (e % (TP_MP * TP_LDX)) / TP_LDX;
    if (c >= m) tps[e] = 0.0;
  }
  const int64_t ntiles = (n + TP_ROWS - 1) / TP_ROWS;
  auto issue = [&](int64_t tile, double* X) {  // 16-byte granules (2 rows) per cp.async
    if (tile >= ntiles) return;
    const int64_t r0 = tile * TP_ROWS;
    for (int e = tid; e < (TP_ROWS / 2) * m; e += TP_NT) {
      const int g2 = e % (TP_ROWS / 2), c = e / (TP_ROWS / 2);
      const int64_t row = r0 + 2 * g2;
      const int64_t rem = n - row;
      const int bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
      cp_async16(X + c * TP_LDX + 2 * g2, bytes ? W2 + row + (int64_t)c * ldw : W2, bytes);
    }
  };
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int rg = warp & 3, nt = warp >> 2;  // DMMA: 16-row group, 8-column half of the block
  const int nb = mp / 16;
  int it = 0;
  issue(blockIdx.x, tps);
  cp_async_commit_group();
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    double* X = tps + (it & 1) * (TP_MP * TP_LDX);
    cp_async_wait_group<0>();
    __syncthreads();  // tile landed; every thread is done with the other buffer
    issue(tile + gridDim.x, tps + ((it + 1) & 1) * (TP_MP * TP_LDX));
    cp_async_commit_group();
    for (int b = 0; b < nb; ++b) {
      if (b > 0) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int kk = 0; kk < b; ++kk) {
          double a[8], bb[4];
#pragma unroll
          for (int v = 0; v < 8; ++v) a[v] = X[(16 * kk + t + 4 * (v >> 1)) * TP_LDX + 16 * rg + g + 8 * (v & 1)];
#pragma unroll
          for (int v = 0; v < 4; ++v) bb[v] = Ms[(16 * b + 8 * nt + g) * TP_LDM + 16 * kk + t + 4 * v];
          dmma16x8x16(acc, a, bb);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double* p = &X[(16 * b + 8 * nt + 2 * t + q) * TP_LDX + 16 * rg + g + 8 * h];
            *p = *p - acc[2 * h + q];
          }
        __syncthreads();
      }
      if (tid < TP_ROWS) {
        double x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = X[(16 * b + j) * TP_LDX + tid];
        const double2* dt2 = reinterpret_cast<const double2*>(DT + 256 * b);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          x[j] = x[j] * rinv[16 * b + j];
#pragma unroll
          for (int p2 = (j + 1) / 2; p2 < 8; ++p2) {  // same ops, same order: k = j+1 .. 15
            const double2 mm = dt2[8 * j + p2];
            if (2 * p2 > j) x[2 * p2] = fma(-x[j], mm.x, x[2 * p2]);
            x[2 * p2 + 1] = fma(-x[j], mm.y, x[2 * p2 + 1]);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) X[(16 * b + j) * TP_LDX + tid] = x[j];
      }
      __syncthreads();
    }
    // store the solved tile (16-byte stores, rows beyond n skipped)
    const int64_t r0 = tile * TP_ROWS;
    for (int e = tid; e < (TP_ROWS / 2) * m; e += TP_NT) {
      const int g2 = e % (TP_ROWS / 2), c = e / (TP_ROWS / 2);
      const int64_t row = r0 + 2 * g2;
      const double2 v = *reinterpret_cast<const double2*>(X + c * TP_LDX + 2 * g2);
      double* dst = U2 + row + (int64_t)c * ldu;
      if (row + 1 < n) *reinterpret_cast<double2*>(dst) = v;
      else if (row < n) dst[0] = v.x;
    }
  }
  cp_async_wait_group<0>();
}

template <typename T>
__global__ void top_from_s_kernel(const double* S, int64_t lds, int m, T* U, int64_t ldu, const Status* st) {
  if (failed(st)) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * m; e += gridDim.x * blockDim.x)
    U[(e % m) + (int64_t)(e / m) * ldu] = Lo<T>::store(Lo<T>::from_double(S[(e % m) + (int64_t)(e / m) * lds]));
}

// Everything of rec_rhqr after the sketch (rhqr.py:383-395): householder_qr
// of Z (od x m, fp64, overwritten by nothing), Mfac = triu(T^t S^t Z) and its
// diagonal check, U2 = W2 Mfac^{-1} over the n2 rows of W2 given, and — when
// Utop is set — the identity-block rows U[:m] = S[:m].  Shared by the single-
// GPU path and the row-partitioned one (rhqr_dist.cu), where every rank solves
// its own rows.  M: m x m fp64 scratch; X: n2 x m fp64 scratch when m > 64.
template <typename T>
int rec_finish_t(sqb_ctx* ctx, int scaling, const double* Z, int64_t od, int64_t m, const T* W2, int64_t n2,
                 int64_t ldw, T* U2, int64_t ldu, T* Utop, int64_t ldutop, double* S, int64_t lds, double* Tm,
                 int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* M,
                 double* X) {
  Status* st = ctx->d_status;
  // K5: householder_qr(Z) (rhqr.py:383)
  const size_t hsm = sizeof(double) * (od + 2 * m + 32);
  const size_t hsm_res = hsm + sizeof(double) * ((size_t)od * m + (size_t)m * m);
  if (hsm_res <= 227 * 1024) {
    allow_dyn_smem(hqr_kernel<true>, (size_t)(hsm_res));
    hqr_kernel<true><<<1, HQR_NT, hsm_res, ctx->stream>>>(Z, od, (int)od, (int)m, scaling, S, lds, Tm, ldt, R, ldr,
                                                          sigmas, rhos, betas, st);
  } else {
    allow_dyn_smem(hqr_kernel<false>, (size_t)(std::max<size_t>(hsm, 48 << 10)));
    hqr_kernel<false><<<1, HQR_NT, hsm, ctx->stream>>>(Z, od, (int)od, (int)m, scaling, S, lds, Tm, ldt, R, ldr,
                                                       sigmas, rhos, betas, st);
  }
  SQB_TRY(check_launch(ctx, "hqr_kernel"));
  // Mfac = triu(T^t S^t Z) and its diagonal check (rhqr.py:387-391)
  mfac_kernel<<<(unsigned)m, 256, sizeof(double) * m, ctx->stream>>>(S, lds, Tm, ldt, Z, od, (int)od, (int)m, M, st);
  SQB_TRY(check_launch(ctx, "mfac_kernel"));
  mfac_check_kernel<<<1, 256, 0, ctx->stream>>>(M, (int)m, st);
  SQB_TRY(check_launch(ctx, "mfac_check_kernel"));
  // K6: U2 = W2 Mfac^{-1}
  const int64_t n = n2;
  if (n > 0) {
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 8 * 148));
    const size_t msm = sizeof(double) * m * m;
    const int mp = (int)((m + 15) / 16 * 16);
    const size_t tsm = sizeof(double) * ((size_t)mp * (mp + 4) + (size_t)TR_ROWS * (mp + 1));
    const bool pipe_ok = std::is_same<T, double>::value && m > 16 && m <= TP_MP &&
                         ((reinterpret_cast<uintptr_t>(W2) & 15) == 0) && ((reinterpret_cast<uintptr_t>(U2) & 15) == 0) &&
                         (ldw % 2 == 0) && (ldu % 2 == 0) && !getenv("SQB_TRSM_BASE");
    if (pipe_ok) {
      allow_dyn_smem(trsm_pipe_kernel, (size_t)(TP_SMEM));
      const unsigned gt = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + TP_ROWS - 1) / TP_ROWS, 2 * (int64_t)ctx->sm_count));
      trsm_pipe_kernel<<<gt, TP_NT, TP_SMEM, ctx->stream>>>((const double*)W2, ldw, n, (int)m, mp, M, (double*)U2, ldu, st);
    } else if (m > 16 && tsm <= 200 * 1024) {
      allow_dyn_smem(trsm_dmma_kernel<T>, (size_t)(tsm));
      const unsigned gt = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + TR_ROWS - 1) / TR_ROWS, 2 * (int64_t)ctx->sm_count));
      trsm_dmma_kernel<T><<<gt, TR_NT, tsm, ctx->stream>>>(W2, ldw, n, (int)m, mp, M, U2, ldu, st);
    } else if (m <= 16) {
      trsm_rows_kernel<T, 16><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
    } else if (m <= 32) {
      trsm_rows_kernel<T, 32><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
    } else if (m <= 64) {
      trsm_rows_kernel<T, 64><<<grid, 128, msm, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, st);
    } else {
      trsm_rows_generic_kernel<T><<<grid, 128, 0, ctx->stream>>>(W2, ldw, n, (int)m, M, U2, ldu, X, st);
    }
    SQB_TRY(check_launch(ctx, "trsm_rows_kernel"));
  }
  if (Utop) {
    top_from_s_kernel<T><<<(unsigned)std::max<int64_t>(1, (m * m + 255) / 256), 256, 0, ctx->stream>>>(
        S, lds, (int)m, Utop, ldutop, st);
    SQB_TRY(check_launch(ctx, "top_from_s_kernel"));
  }
  return SQB_OK;
}

#define SQB_REC_FINISH_INST(T)                                                                              \
  template int rec_finish_t<T>(sqb_ctx*, int, const double*, int64_t, int64_t, const T*, int64_t, int64_t, T*, \
                               int64_t, T*, int64_t, double*, int64_t, double*, int64_t, double*, int64_t,   \
                               double*, double*, double*, double*, double*);
SQB_REC_FINISH_INST(double)
SQB_REC_FINISH_INST(float)
SQB_REC_FINISH_INST(__half)
SQB_REC_FINISH_INST(__nv_bfloat16)
#undef SQB_REC_FINISH_INST

template <typename T>
static int rec_rhqr_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                      int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt,
                      double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  const int64_t n = N - m, od = m + sk->ell;
  WsPlan plan;
  const size_t iZ = plan.add(sizeof(double) * od * m);
  const size_t iM = plan.add(sizeof(double) * m * m);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, m));
  const size_t iX = plan.add(m > 64 ? sizeof(double) * n * m : 8);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* Z = ws_ptr<double>(ctx, plan, iZ);
  Status* st = ctx->d_status;
  const size_t esz = sizeof(T);
  // Z = Psi W  (rhqr.py:382)
  SQB_TRY(launch_copy_top(ctx, Lo<T>::code, W, ldw, m, m, Z, od, st));
  SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)W + m * esz, ldw, m, Z, od, m,
                        ws_ptr<void>(ctx, plan, iP), st));
  return rec_finish_t<T>(ctx, scaling, Z, od, m, (const T*)W + m, n, ldw, (T*)U + m, ldu, (T*)U, ldu, S, lds, Tm,
                         ldt, R, ldr, sigmas, rhos, betas, ws_ptr<double>(ctx, plan, iM), ws_ptr<double>(ctx, plan, iX));
}

int rec_rhqr_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                      int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                      double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                      double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rec_rhqr_t<double>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rec_rhqr_t<float>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rec_rhqr_t<__half>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rec_rhqr_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb

namespace sqb {

// R X = B by back substitution, one CTA per right-hand side (upper_tri_solve,
// linalg.py:102-116); a zero/subnormal diagonal raises SingularFactorError
__global__ void __launch_bounds__(256)
upper_tri_solve_kernel(const double* __restrict__ R, int64_t ldr, int m, const double* __restrict__ B, int64_t ldb,
                       double* __restrict__ X, int64_t ldx, Status* st) {
  __shared__ double red[32];
  extern __shared__ double x[];
  if (failed(st)) return;
  const int col = blockIdx.x;
  if (threadIdx.x == 0 && col == 0)
    for (int i = 0; i < m; ++i)
      if (fabs(R[i + (int64_t)i * ldr]) < DBL_MIN) { fail(st, SQB_ERR_SINGULAR, i + 1, R[i + (int64_t)i * ldr]); break; }
  // scipy's check_finite (linalg.py:115): non-finite operands are a ValueError, after the diagonal check
  __syncthreads();
  if (!failed(st)) {
    bool bad = false;
    for (int i = threadIdx.x; i < m; i += blockDim.x) bad = bad || !isfinite(B[i + (int64_t)col * ldb]);
    if (col == 0)
      for (int e = threadIdx.x; e < m * m; e += blockDim.x)
        if (e % m <= e / m) bad = bad || !isfinite(R[e % m + (int64_t)(e / m) * ldr]);
    if (bad) fail(st, SQB_ERR_NONFINITE, col + 1, 0.0);
  }
  for (int i = m - 1; i >= 0; --i) {
    double part = 0.0;
    for (int j = i + 1 + threadIdx.x; j < m; j += blockDim.x) part = fma(R[i + (int64_t)j * ldr], x[j], part);
    const double d = block_sum(part, red);
    if (threadIdx.x == 0) x[i] = (B[i + (int64_t)col * ldb] - d) / R[i + (int64_t)i * ldr];
    __syncthreads();
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) X[i + (int64_t)col * ldx] = x[i];
}

}  // namespace sqb

namespace sqb {
// the solve inside a running call chain (no status reset: a breakdown recorded
// by an earlier kernel of the chain must survive to the caller's status read)
int upper_tri_solve_impl(sqb_ctx* ctx, const double* R, int64_t ldr, int64_t m, const double* B, int64_t ldb,
                         int64_t k, double* X, int64_t ldx) {
  if (m < 1 || k < 1) return SQB_OK;
  upper_tri_solve_kernel<<<(unsigned)k, 256, sizeof(double) * m, ctx->stream>>>(R, ldr, (int)m, B, ldb, X, ldx,
                                                                               ctx->d_status);
  return check_launch(ctx, "upper_tri_solve_kernel");
}
}  // namespace sqb

extern "C" int sqb_upper_tri_solve(sqb_ctx* ctx, const double* R, int64_t ldr, int64_t m, const double* B,
                                   int64_t ldb, int64_t k, double* X, int64_t ldx) {
  using namespace sqb;
  SQB_TRY(begin_entry(ctx));
  return upper_tri_solve_impl(ctx, R, ldr, m, B, ldb, k, X, ldx);
}

namespace sqb {
int hqr_tall(sqb_ctx* ctx, int scaling, const double* A, int64_t lda, int64_t p, int64_t m, double* U, int64_t ldu,
             double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas);
}

extern "C" int sqb_householder_qr(sqb_ctx* ctx, int scaling, const double* A, int64_t lda, int64_t p, int64_t m,
                                  double* U, int64_t ldu, double* T, int64_t ldt, double* R, int64_t ldr,
                                  double* sigmas, double* rhos, double* betas) {
  using namespace sqb;
  SQB_TRY(begin_entry(ctx));
  if (p < m) return set_error(ctx, SQB_ERR_ARG, "need p >= m, got %lld x %lld", (long long)p, (long long)m);
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  const size_t hsm = sizeof(double) * (p + 2 * m + 32);
  if (hsm > 200 * 1024) {  // tall matrix: the multi-CTA path (hqr_tall.cu)
    if ((reinterpret_cast<uintptr_t>(U) & 15) != 0 || ldu % 2 != 0)
      return set_error(ctx, SQB_ERR_ARG, "householder_qr: U must be 16-byte aligned with an even leading dimension");
    return hqr_tall(ctx, scaling, A, lda, p, m, U, ldu, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  const size_t hsm_res = hsm + sizeof(double) * ((size_t)p * m + (size_t)m * m);
  if (hsm_res <= 227 * 1024) {
    allow_dyn_smem(hqr_kernel<true>, (size_t)(hsm_res));
    hqr_kernel<true><<<1, HQR_NT, hsm_res, ctx->stream>>>(A, lda, (int)p, (int)m, scaling, U, ldu, T, ldt, R, ldr,
                                                          sigmas, rhos, betas, ctx->d_status);
  } else {
    allow_dyn_smem(hqr_kernel<false>, (size_t)(std::max<size_t>(hsm, 48 << 10)));
    hqr_kernel<false><<<1, HQR_NT, hsm, ctx->stream>>>(A, lda, (int)p, (int)m, scaling, U, ldu, T, ldt, R, ldr,
                                                       sigmas, rhos, betas, ctx->d_status);
  }
  return check_launch(ctx, "hqr_kernel");
}
