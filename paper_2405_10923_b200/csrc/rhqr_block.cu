// Blocked left-looking RHQR (rhqr_block, rhqr.py:334-365) and the compact-form
// T recovered from the sketches alone (t_factor_from_sketches, rhqr.py:122-132).
//
// Per panel [j0, j1):   X = W[:, j0:j1]
//   for every earlier panel p (in order, each one re-sketching X, rhqr.py:357-360):
//       Y = Psi X                      (K1, b columns at once)
//       C = T_p^t (S_p^t Y)            (coef_kernel, high precision)
//       X = fl(X - fl(U_p C))          (panel_update_kernel: one HBM pass, b_p x b FMAs per row)
//   the left-looking sweep over X with pivot offset j0 (left_sweep_t, the
//   rhqr_left machinery with StepArgs::off).
// The per-panel T blocks are returned on the diagonal of an m x m array
// (BlockRHQRFactors.panels[k].T); the stacked global T comes from
// t_factor_from_sketches(S).
#include <algorithm>
#include <type_traits>

#include "mma.cuh"
#include "rhqr_kernels.cuh"

namespace sqb {

template <typename T>
int left_sweep_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                 int64_t ldw, int64_t ncol, int64_t off, void* U, int64_t ldu, double* S, int64_t lds,
                 double* Tm, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                 double* betas, void* ws_base);
size_t left_sweep_ws_bytes(const sqb_sketch* sk, int code, int64_t m, int64_t ncol);
__global__ void coef_kernel(const double* __restrict__ S, int64_t lds, const double* __restrict__ Tm, int64_t ldt,
                            int transpose_t, const double* __restrict__ Y, int64_t ldy, int od, int r,
                            double* __restrict__ C, int64_t ldc, const Status* st);
__global__ void upper_tri_solve_kernel(const double* __restrict__ R, int64_t ldr, int m,
                                       const double* __restrict__ B, int64_t ldb, double* __restrict__ X,
                                       int64_t ldx, Status* st);

// X[:, :b] = fl(X - fl(U[:, :bp] C)), C (bp x b) in the high precision rounded
// to low once (rhqr.py:360).  A CTA owns PU_RB rows; U rows are staged through
// shared memory KC columns at a time, the two thread halves own 16 output
// columns each.
constexpr int PU_RB = 128, PU_KC = 32, PU_JC = 16;

template <typename T>
__global__ void __launch_bounds__(256)
panel_update_kernel(const T* __restrict__ U, int64_t ldu, int64_t N, int bp, const double* __restrict__ C,
                    int64_t ldc, T* X, int64_t ldx, int b, const Status* st) {
  using A = typename Lo<T>::acc;
  __shared__ T Us[PU_KC][PU_RB];
  __shared__ A Cs[PU_KC][2 * PU_JC];
  if (failed(st)) return;
  const int row = threadIdx.x % PU_RB, h = threadIdx.x / PU_RB;
  for (int64_t r0 = (int64_t)blockIdx.x * PU_RB; r0 < N; r0 += (int64_t)gridDim.x * PU_RB) {
    const int64_t i = r0 + row;
    for (int jb = 0; jb < b; jb += 2 * PU_JC) {
      // this thread's X entries first: their latency overlaps the U staging
      // and the FMAs (loads batched ahead of the stores)
      A xv[PU_JC];
#pragma unroll
      for (int j = 0; j < PU_JC; ++j) {
        const int col = jb + h * PU_JC + j;
        xv[j] = (i < N && col < b) ? Lo<T>::load(X[i + (int64_t)col * ldx]) : A(0);
      }
      A acc[PU_JC];
#pragma unroll
      for (int j = 0; j < PU_JC; ++j) acc[j] = A(0);
      for (int kb = 0; kb < bp; kb += PU_KC) {
        __syncthreads();
        T v[PU_KC * PU_RB / 256];
#pragma unroll
        for (int q = 0; q < PU_KC * PU_RB / 256; ++q) {
          const int e = threadIdx.x + q * 256, k = e / PU_RB, r = e % PU_RB;
          v[q] = (kb + k < bp && r0 + r < N) ? U[(r0 + r) + (int64_t)(kb + k) * ldu] : Lo<T>::store(A(0));
        }
#pragma unroll
        for (int q = 0; q < PU_KC * PU_RB / 256; ++q) {
          const int e = threadIdx.x + q * 256;
          Us[e / PU_RB][e % PU_RB] = v[q];
        }
        for (int e = threadIdx.x; e < PU_KC * 2 * PU_JC; e += 256) {
          const int k = e / (2 * PU_JC), j = e % (2 * PU_JC);
          Cs[k][j] = (kb + k < bp && jb + j < b) ? Lo<T>::from_double(C[(kb + k) + (int64_t)(jb + j) * ldc]) : A(0);
        }
        __syncthreads();
        const int kn = min(PU_KC, bp - kb);
        for (int k = 0; k < kn; ++k) {
          const A u = Lo<T>::load(Us[k][row]);
#pragma unroll
          for (int j = 0; j < PU_JC; ++j) acc[j] = fma(u, Cs[k][h * PU_JC + j], acc[j]);
        }
      }
      if (i < N) {
#pragma unroll
        for (int j = 0; j < PU_JC; ++j) {
          const int col = jb + h * PU_JC + j;
          if (col < b) X[i + (int64_t)col * ldx] = Lo<T>::store(Lo<T>::sub(xv[j], Lo<T>::rnd(acc[j])));
        }
      }
    }
  }
}

// fp64: the same update on the tensor pipe.  A CTA owns 128 rows x 32 output
// columns; warp w the rows [16w, 16w+16) as four m16n8 DMMA tiles.  U is
// staged by cp.async (8 B per element, any alignment) while the thread's X
// entries are loaded; shared strides padded to 2-wavefront fragment loads.
constexpr int PD_RB = 128, PD_KC = 32, PD_NC = 32, PD_US = PD_RB + 4, PD_CS = PD_NC + 4;

__global__ void __launch_bounds__(256, 3)
panel_update_dmma_kernel(const double* __restrict__ U, int64_t ldu, int64_t N, int bp,
                         const double* __restrict__ C, int64_t ldc, double* X, int64_t ldx, int b,
                         const Status* st) {
  __shared__ __align__(16) double Us[PD_KC * PD_US];
  __shared__ double Cs[PD_KC * PD_CS];
  if (failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wr = warp * 16;
  for (int64_t r0 = (int64_t)blockIdx.x * PD_RB; r0 < N; r0 += (int64_t)gridDim.x * PD_RB) {
    for (int jb = 0; jb < b; jb += PD_NC) {
      double acc[4][4], xv[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[nt][v] = 0.0;
      for (int kb = 0; kb < bp; kb += PD_KC) {
        __syncthreads();
#pragma unroll
        for (int q = 0; q < PD_KC * PD_RB / 256; ++q) {
          const int e = threadIdx.x + q * 256, k = e / PD_RB, r = e % PD_RB;
          double* dst = Us + k * PD_US + r;
          if (kb + k < bp && r0 + r < N) {
            const double* src = U + (r0 + r) + (int64_t)(kb + k) * ldu;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
          } else {
            *dst = 0.0;
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        for (int e = threadIdx.x; e < PD_KC * PD_NC; e += 256) {
          const int k = e / PD_NC, n = e % PD_NC;
          Cs[k * PD_CS + n] = (kb + k < bp && jb + n < b) ? C[(kb + k) + (int64_t)(jb + n) * ldc] : 0.0;
        }
        if (kb == 0) {
          // X fragment entries (rows g, g+8; columns 2t, 2t+1 of each n-tile)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const int64_t i = r0 + wr + g + 8 * (v >> 1);
              const int col = jb + nt * 8 + 2 * t + (v & 1);
              xv[nt][v] = (i < N && col < b) ? X[i + (int64_t)col * ldx] : 0.0;
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
#pragma unroll
        for (int k16 = 0; k16 < PD_KC / 16; ++k16) {
          double a[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) a[v] = Us[(k16 * 16 + t + 4 * (v >> 1)) * PD_US + wr + g + 8 * (v & 1)];
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            double bf[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) bf[v] = Cs[(k16 * 16 + t + 4 * v) * PD_CS + nt * 8 + g];
            dmma_16x8x16(acc[nt], a, bf);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int64_t i = r0 + wr + g + 8 * (v >> 1);
          const int col = jb + nt * 8 + 2 * t + (v & 1);
          if (i < N && col < b) X[i + (int64_t)col * ldx] = __dsub_rn(xv[nt][v], acc[nt][v]);
        }
    }
  }
}

// The block_size <= 32 case (the default): C staged once per CTA, U double-
// buffered across the CTA's row blocks and X prefetched one block ahead, so
// the HBM stream of block i+1 overlaps the DMMAs and stores of block i.
__device__ __forceinline__ void pd_stage_u(double* Us, const double* __restrict__ U, int64_t ldu, int64_t N,
                                           int bp, int64_t r0) {
#pragma unroll
  for (int q = 0; q < PD_KC * PD_RB / 256; ++q) {
    const int e = threadIdx.x + q * 256, k = e / PD_RB, r = e % PD_RB;
    double* dst = Us + k * PD_US + r;
    if (k < bp && r0 + r < N)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n"
                   ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(U + (r0 + r) + (int64_t)k * ldu) : "memory");
    else
      *dst = 0.0;
  }
}

__device__ __forceinline__ void pd_load_x(double (&xv)[4][4], const double* X, int64_t ldx, int64_t N, int b,
                                          int64_t rbase, int g, int t) {
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = rbase + g + 8 * (v >> 1);
      const int col = nt * 8 + 2 * t + (v & 1);
      xv[nt][v] = (i < N && col < b) ? X[i + (int64_t)col * ldx] : 0.0;
    }
}

__global__ void __launch_bounds__(256, 2)
panel_update_dmma32_kernel(const double* __restrict__ U, int64_t ldu, int64_t N, int bp,
                           const double* __restrict__ C, int64_t ldc, double* X, int64_t ldx, int b,
                           const Status* st) {
  extern __shared__ __align__(16) double pd_smem[];
  double* Us0 = pd_smem;
  double* Us1 = pd_smem + PD_KC * PD_US;
  double* Cs = pd_smem + 2 * PD_KC * PD_US;
  if (failed(st)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wr = warp * 16;
  const int64_t nblk = (N + PD_RB - 1) / PD_RB;
  for (int e = threadIdx.x; e < PD_KC * PD_NC; e += 256) {
    const int k = e / PD_NC, n = e % PD_NC;
    Cs[k * PD_CS + n] = (k < bp && n < b) ? C[k + (int64_t)n * ldc] : 0.0;
  }
  int64_t blk = blockIdx.x;
  double xv[4][4], xn[4][4];
  if (blk < nblk) {
    pd_stage_u(Us0, U, ldu, N, bp, blk * PD_RB);
    pd_load_x(xv, X, ldx, N, b, blk * PD_RB + wr, g, t);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int it = 0; blk < nblk; blk += gridDim.x, ++it) {
    double* Uc = (it & 1) ? Us1 : Us0;
    double* Un = (it & 1) ? Us0 : Us1;
    const int64_t nxt = blk + gridDim.x;
    if (nxt < nblk) {
      pd_stage_u(Un, U, ldu, N, bp, nxt * PD_RB);
      pd_load_x(xn, X, ldx, N, b, nxt * PD_RB + wr, g, t);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[nt][v] = 0.0;
#pragma unroll
    for (int k16 = 0; k16 < PD_KC / 16; ++k16) {
      double a[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) a[v] = Uc[(k16 * 16 + t + 4 * (v >> 1)) * PD_US + wr + g + 8 * (v & 1)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double bf[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) bf[v] = Cs[(k16 * 16 + t + 4 * v) * PD_CS + nt * 8 + g];
        dmma_16x8x16(acc[nt], a, bf);
      }
    }
    const int64_t rb = blk * PD_RB + wr;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int64_t i = rb + g + 8 * (v >> 1);
        const int col = nt * 8 + 2 * t + (v & 1);
        if (i < N && col < b) X[i + (int64_t)col * ldx] = __dsub_rn(xv[nt][v], acc[nt][v]);
      }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) xv[nt][v] = xn[nt][v];
    __syncthreads();  // Uc is refilled next iteration
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

template <typename T>
static int panel_update(sqb_ctx* ctx, const T* U, int64_t ldu, int64_t N, int64_t bp, const double* C, int64_t ldc,
                        T* X, int64_t ldx, int64_t b) {
  const int64_t blocks = (N + PU_RB - 1) / PU_RB;
  if constexpr (std::is_same<T, double>::value) {
    if (bp <= PD_KC && b <= PD_NC) {
      const size_t smem = sizeof(double) * (2 * PD_KC * PD_US + PD_KC * PD_CS);
      allow_dyn_smem(panel_update_dmma32_kernel, (size_t)(smem));
      const unsigned grid = (unsigned)std::min<int64_t>(blocks, 2 * (int64_t)ctx->sm_count);
      panel_update_dmma32_kernel<<<grid, 256, smem, ctx->stream>>>(U, ldu, N, (int)bp, C, ldc, X, ldx, (int)b,
                                                                   ctx->d_status);
      return check_launch(ctx, "panel_update_dmma32_kernel");
    }
    const unsigned grid = (unsigned)std::min<int64_t>(blocks, 3 * (int64_t)ctx->sm_count);
    panel_update_dmma_kernel<<<grid, 256, 0, ctx->stream>>>(U, ldu, N, (int)bp, C, ldc, X, ldx, (int)b,
                                                            ctx->d_status);
    return check_launch(ctx, "panel_update_dmma_kernel");
  }
  const unsigned grid = (unsigned)std::min<int64_t>(blocks, 8 * (int64_t)ctx->sm_count);
  panel_update_kernel<T><<<grid, 256, 0, ctx->stream>>>(U, ldu, N, (int)bp, C, ldc, X, ldx, (int)b, ctx->d_status);
  return check_launch(ctx, "panel_update_kernel");
}

template <typename T>
static int rhqr_block_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                        int64_t ldw, int64_t bs, void* U, int64_t ldu, double* S, int64_t lds, double* Tm,
                        int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas) {
  const int64_t od = m + sk->ell;
  const int64_t b0 = std::min(bs, m);
  constexpr int VN = VecN<T>::n;
  // panel buffer: row m of every column 16-byte aligned (vector path of the sweep)
  const int64_t ldx = (N + VN - 1) / VN * VN;
  const int64_t shift = (VN - m % VN) % VN;
  WsPlan plan;
  const size_t iX = plan.add(sizeof(T) * (ldx * b0 + shift));
  const size_t iY = plan.add(sizeof(double) * od * b0);
  const size_t iC = plan.add(sizeof(double) * m * b0);
  const size_t iP = plan.add(sketch_partials_bytes(sk, Lo<T>::code, b0));
  const size_t iSw = plan.add(left_sweep_ws_bytes(sk, Lo<T>::code, m, b0));
  SQB_TRY(ws_reserve(ctx, plan.total));
  T* X = ws_ptr<T>(ctx, plan, iX) + shift;
  double* Y = ws_ptr<double>(ctx, plan, iY);
  double* C = ws_ptr<double>(ctx, plan, iC);
  void* P = ws_ptr<void>(ctx, plan, iP);
  void* sw = ws_ptr<void>(ctx, plan, iSw);
  Status* st = ctx->d_status;
  const size_t esz = sizeof(T);
  // T holds the panel triangles on its diagonal blocks; the rest is zero
  SQB_CUDA_TRY(cudaMemset2DAsync(Tm, ldt * sizeof(double), 0, m * sizeof(double), m, ctx->stream));
  for (int64_t j0 = 0; j0 < m; j0 += bs) {
    const int64_t b = std::min(bs, m - j0);
    SQB_CUDA_TRY(cudaMemcpy2DAsync(X, ldx * esz, (const T*)W + j0 * ldw, ldw * esz, N * esz, b,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    for (int64_t p0 = 0; p0 < j0; p0 += bs) {
      const int64_t bp = std::min(bs, j0 - p0);
      SQB_TRY(launch_copy_top(ctx, Lo<T>::code, X, ldx, m, b, Y, od, st));
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, X + m, ldx, b, Y, od, m, P, st));
      coef_kernel<<<(unsigned)b, 256, sizeof(double) * bp, ctx->stream>>>(
          S + p0 * lds, lds, Tm + p0 + p0 * ldt, ldt, 1, Y, od, (int)od, (int)bp, C, bp, st);
      SQB_TRY(check_launch(ctx, "coef_kernel"));
      SQB_TRY(panel_update<T>(ctx, (const T*)U + p0 * ldu, ldu, N, bp, C, bp, X, ldx, b));
    }
    SQB_TRY(left_sweep_t<T>(ctx, sk, scaling, X, N, m, ldx, b, j0, (T*)U + j0 * ldu, ldu, S + j0 * lds, lds,
                            Tm + j0 + j0 * ldt, ldt, R + j0 * ldr, ldr, sigmas + j0, rhos + j0, betas + j0, sw));
  }
  return SQB_OK;
}

int rhqr_block_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W, int64_t N,
                        int64_t m, int64_t ldw, int64_t bs, void* U, int64_t ldu, double* S, int64_t lds,
                        double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                        double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return rhqr_block_t<double>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F32: return rhqr_block_t<float>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_F16: return rhqr_block_t<__half>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
    case SQB_BF16: return rhqr_block_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, bs, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

// Tinv = strict upper triangle of S^t S plus half its diagonal, and B = I
// (rhqr.py:129-131); one warp per entry (i <= j)
__global__ void tinv_kernel(const double* __restrict__ S, int64_t lds, int od, int k, double* __restrict__ Tinv,
                            double* __restrict__ B) {
  const int i = blockIdx.x, j = blockIdx.y, lane = threadIdx.x;
  if (i > j) {
    if (lane == 0) { Tinv[i + (int64_t)j * k] = 0.0; B[i + (int64_t)j * k] = 0.0; }
    return;
  }
  double d = 0.0;
  for (int r = lane; r < od; r += 32) d = fma(S[r + (int64_t)i * lds], S[r + (int64_t)j * lds], d);
  d = warp_sum(d);
  if (lane == 0) {
    Tinv[i + (int64_t)j * k] = i == j ? d / 2.0 : d;
    B[i + (int64_t)j * k] = i == j ? 1.0 : 0.0;
  }
}

}  // namespace sqb

namespace sqb {
int t_factor_impl(sqb_ctx* ctx, const double* S, int64_t lds, int64_t od, int64_t k, double* T, int64_t ldt);
}

extern "C" int sqb_t_factor(sqb_ctx* ctx, const double* S, int64_t lds, int64_t od, int64_t k, double* T,
                            int64_t ldt) {
  using namespace sqb;
  SQB_TRY(begin_entry(ctx));
  return t_factor_impl(ctx, S, lds, od, k, T, ldt);
}

// T from S inside a running call chain (no status reset: a breakdown recorded
// by the sweep must survive to the caller's status read)
int sqb::t_factor_impl(sqb_ctx* ctx, const double* S, int64_t lds, int64_t od, int64_t k, double* T, int64_t ldt) {
  using namespace sqb;
  if (k < 1) return SQB_OK;
  if (lds < od || ldt < k) return set_error(ctx, SQB_ERR_ARG, "bad leading dimensions");
  WsPlan plan;
  const size_t iA = plan.add(sizeof(double) * k * k);
  const size_t iB = plan.add(sizeof(double) * k * k);
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* Tinv = ws_ptr<double>(ctx, plan, iA);
  double* B = ws_ptr<double>(ctx, plan, iB);
  tinv_kernel<<<dim3((unsigned)k, (unsigned)k), 32, 0, ctx->stream>>>(S, lds, (int)od, (int)k, Tinv, B);
  SQB_TRY(check_launch(ctx, "tinv_kernel"));
  upper_tri_solve_kernel<<<(unsigned)k, 256, sizeof(double) * k, ctx->stream>>>(Tinv, k, (int)k, B, k, T, ldt,
                                                                               ctx->d_status);
  return check_launch(ctx, "upper_tri_solve_kernel");
}
