// K2 — dense sketch Y = G X on the FP64 tensor pipe (DMMA, mma.sync m16n8k16 f64).
//
// Reference: GaussianSketch._apply (sketching.py:109-125): Y = G @ X with G the
// (ell x n) N(0, 1/ell) matrix (row i from Philox(key=[seed, i]), :100-107;
// generated on the host with the same numpy calls and uploaded once).  For
// BASELINE config 3 the shape is 256 x 4,194,240 times 4,194,240 x 64: a
// split-K GEMM with a huge K.  Both operands are K-contiguous (G row-major,
// X column-major), so tiles stream straight into shared memory with cp.async
// and feed DMMA fragments; the split-K partials are summed in slab order by a
// second kernel (deterministic).
//
// Arithmetic type follows the reference: fp64 -> DMMA; fp32 / fp16 (fp32
// accumulation, sketching.py:111) / bf16 (ml_dtypes matmul, fp32
// accumulation) use a CUDA-core kernel — they are off the BASELINE configs.
#include <algorithm>

#include "dense.cuh"
#include "mma.cuh"
#include "sketch.cuh"
#include "vec.cuh"
#include "tma.cuh"

namespace sqb {

// Double-buffered 32-deep k tiles (2 x 55 KB) at 2 CTAs/SM (128 registers):
// the two CTAs' DMMA streams cover each other's block barriers and cp.async
// waits.  Config 3 (round 1 session 4): 3-stage 1-CTA 6.87 ms, 64-deep
// 2-stage 1-CTA 6.43 ms, this 6.34 ms (30.4 TFLOP/s in the sketch GEMM).
constexpr int DBM = 128, DBN = 64, DBK = 32, DSTR = DBK + 4, DSTAGES = 2, DNT = 256;
constexpr size_t DSMEM = sizeof(double) * DSTAGES * (size_t)(DBM + DBN) * DSTR;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// one CTA: a 128 x 64 tile of the partial product over K-range [k0, k1)
__global__ void __launch_bounds__(DNT, 2)
dense_dmma_kernel(const double* __restrict__ G, int64_t ldg, const double* __restrict__ X,
                  int64_t ldx, int64_t M, int64_t N, int64_t K, int64_t kslab,
                  double* __restrict__ P, const Status* st, int z_off) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sG = reinterpret_cast<double*>(smem_raw);
  double* sX = sG + DSTAGES * DBM * DSTR;
  if (st && failed(st)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * DBM, n0 = (int64_t)blockIdx.y * DBN;
  const int64_t z = (int64_t)blockIdx.z + z_off;  // slab (a streamed upload launches a range of slabs)
  const int64_t k0 = z * kslab;
  const int64_t k1 = std::min<int64_t>(K, k0 + kslab);
  const int nk = (int)((k1 - k0 + DBK - 1) / DBK);

  const bool v16 = ((reinterpret_cast<uintptr_t>(G) | reinterpret_cast<uintptr_t>(X)) & 15) == 0 &&
                   (ldg % 2 == 0) && (ldx % 2 == 0) && (k0 % 2 == 0) && (k1 % 2 == 0);
  auto load_stage = [&](int s, int kt) {
    const int64_t kb = k0 + (int64_t)kt * DBK;
    double* g = sG + s * DBM * DSTR;
    double* x = sX + s * DBN * DSTR;
    if (v16) {  // 16-byte chunks (k1 even, so a pair never straddles the slab end)
      for (int e = tid; e < DBM * DBK / 2; e += DNT) {
        const int r = e / (DBK / 2), kk = 2 * (e % (DBK / 2));
        const int64_t gr = m0 + r, gk = kb + kk;
        double* d = g + r * DSTR + kk;
        if (gr < M && gk < k1) cp_async16(d, G + gr * ldg + gk, 16);
        else { d[0] = 0.0; d[1] = 0.0; }
      }
      for (int e = tid; e < DBN * DBK / 2; e += DNT) {
        const int cidx = e / (DBK / 2), kk = 2 * (e % (DBK / 2));
        const int64_t gc = n0 + cidx, gk = kb + kk;
        double* d = x + cidx * DSTR + kk;
        if (gc < N && gk < k1) cp_async16(d, X + gc * ldx + gk, 16);
        else { d[0] = 0.0; d[1] = 0.0; }
      }
      return;
    }
    for (int e = tid; e < DBM * DBK; e += DNT) {
      const int r = e / DBK, kk = e % DBK;
      const int64_t gr = m0 + r, gk = kb + kk;
      double* d = g + r * DSTR + kk;
      if (gr < M && gk < k1) cp_async8(d, G + gr * ldg + gk);
      else *d = 0.0;
    }
    for (int e = tid; e < DBN * DBK; e += DNT) {
      const int cidx = e / DBK, kk = e % DBK;
      const int64_t gc = n0 + cidx, gk = kb + kk;
      double* d = x + cidx * DSTR + kk;
      if (gc < N && gk < k1) cp_async8(d, X + gc * ldx + gk);
      else *d = 0.0;
    }
  };

  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps of 32 x 32
  const int g = lane >> 2, t = lane & 3;

#pragma unroll
  for (int s = 0; s < DSTAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<DSTAGES - 2>();
    __syncthreads();
    const int nxt = kt + DSTAGES - 1;
    if (nxt < nk) load_stage(nxt % DSTAGES, nxt);
    cp_async_commit();
    const double* gs = sG + (kt % DSTAGES) * DBM * DSTR + (wm * 32) * DSTR;
    const double* xs = sX + (kt % DSTAGES) * DBN * DSTR + (wn * 32) * DSTR;
#pragma unroll
    for (int k16 = 0; k16 < DBK / 16; ++k16) {
      double a[2][8], b[4][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int v = 0; v < 8; ++v)
          a[mt][v] = gs[(mt * 16 + g + 8 * (v & 1)) * DSTR + k16 * 16 + t + 4 * (v >> 1)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) b[nt][v] = xs[(nt * 8 + g) * DSTR + k16 * 16 + t + 4 * v];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_16x8x16(acc[mt][nt], a[mt], b[nt]);
    }
  }
  cp_async_wait<0>();
  // epilogue: partial tile -> P[slab] (M x N column-major)
  double* p = P + z * M * N;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t r = m0 + wm * 32 + mt * 16 + g + h * 8;
          const int64_t c = n0 + wn * 32 + nt * 8 + 2 * t + q;
          if (r < M && c < N) p[r + c * M] = acc[mt][nt][h * 2 + q];
        }
}

// ---------------------------------------------------------------------------
// K2 on TMA + mbarriers (round 2 session 4).  One CTA per SM owns a
// 256 x 64 output tile of one K slab (config 3: the whole 256 x 64 sketch, so
// X is streamed once, not once per 128-row half): a producer warp issues one
// 2-D tensor-map box per operand and stage (16 doubles = 128 bytes of k times
// 256 / 64 rows, SWIZZLE_128B) on a 5-stage ring of full/empty mbarriers, 16
// consumer warps (8 x 2 of 32 x 32) wait per stage and issue DMMA m16n8k16 —
// no block-wide barrier in the main loop.  Under the 128-byte swizzle a
// fragment load of rows g = 0..7 would put rows g and g ^ 1 on the same banks;
// the kernel therefore maps fragment row g to tile row pr(g) = 2 (g & 3) +
// (g >> 2) inside every 8-row group (the MMA does not care which matrix row
// sits in which fragment row, the epilogue applies the same map), which makes
// every LDS.64 conflict-free.  Same slab partition and the same ascending-k
// DMMA sequence per accumulator as dense_dmma_kernel: Z is bitwise the same.
// ---------------------------------------------------------------------------
constexpr int TM_BM = 256, TM_BN = 64, TM_BK = 16, TM_STAGES = 5, TM_CW = 16, TM_NT = (TM_CW + 1) * 32;
constexpr uint32_t TM_G_BYTES = TM_BM * TM_BK * 8, TM_X_BYTES = TM_BN * TM_BK * 8;
constexpr size_t TM_SMEM = 1024 + (size_t)TM_STAGES * (TM_G_BYTES + TM_X_BYTES) + 2 * TM_STAGES * 8;

__device__ __forceinline__ int tm_pr(int g) { return ((g & 3) << 1) | (g >> 2); }

__global__ void __launch_bounds__(TM_NT, 1)
dense_tma_kernel(const __grid_constant__ CUtensorMap mapG, const __grid_constant__ CUtensorMap mapX, int64_t M,
                 int64_t N, int64_t K, int64_t kslab, double* __restrict__ P, const Status* st) {
  extern __shared__ __align__(1024) unsigned char tm_raw[];
  if (st && failed(st)) return;
  unsigned char* base = tm_raw + ((1024u - (smem_u32(tm_raw) & 1023u)) & 1023u);
  unsigned char* sG = base;                                     // [stage][256 rows][128 B]
  unsigned char* sX = base + (size_t)TM_STAGES * TM_G_BYTES;    // [stage][64 rows][128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + (size_t)TM_STAGES * (TM_G_BYTES + TM_X_BYTES));
  uint64_t* empty = full + TM_STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t m0 = (int64_t)blockIdx.x * TM_BM, n0 = (int64_t)blockIdx.y * TM_BN;
  const int64_t z = blockIdx.z;
  const int64_t k0 = z * kslab, k1 = min(K, k0 + kslab);
  const int nk = (int)((k1 - k0 + TM_BK - 1) / TM_BK);
  if (tid == 0) {
    for (int s = 0; s < TM_STAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, TM_CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == TM_CW) {
    // ---- producer: one elected lane feeds the ring
    if (lane == 0) {
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % TM_STAGES;
        if (kt >= TM_STAGES) mbar_wait(empty + s, ((kt / TM_STAGES) - 1) & 1);
        mbar_expect_tx(full + s, TM_G_BYTES + TM_X_BYTES);
        const int kc = (int)(k0 + (int64_t)kt * TM_BK);
        tma_load_2d(sG + (size_t)s * TM_G_BYTES, &mapG, kc, (int)m0, full + s);
        tma_load_2d(sX + (size_t)s * TM_X_BYTES, &mapX, kc, (int)n0, full + s);
      }
    }
    return;
  }
  // ---- consumers
  double acc[2][4][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;
  const int wm = warp & 7, wn = warp >> 3;  // 8 x 2 warps of 32 x 32
  const int g = lane >> 2, t = lane & 3, pg = tm_pr(g);
  // byte offsets inside a stage: row * 128 + ((chunk ^ (row & 7)) << 4) + (t & 1) * 8 with row & 7 = pg;
  // the k chunk of fragment element v is (t >> 1) + 2 (v >> 1) for A and (t >> 1) + 2 v for B: four
  // swizzled column offsets serve both, the row parts are compile-time multiples of 1024
  uint32_t cx[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) cx[c] = (uint32_t)(((((t >> 1) + 2 * c) ^ pg) << 4) + (t & 1) * 8);
  const uint32_t arow = (uint32_t)((wm * 32 + pg) * 128), brow = (uint32_t)((wn * 32 + pg) * 128);
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % TM_STAGES;
    mbar_wait(full + s, (kt / TM_STAGES) & 1);
    const unsigned char* gs = sG + (size_t)s * TM_G_BYTES + arow;
    const unsigned char* xs = sX + (size_t)s * TM_X_BYTES + brow;
    double b[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) b[nt][v] = *reinterpret_cast<const double*>(xs + nt * 1024 + cx[v]);
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      double a[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) a[v] = *reinterpret_cast<const double*>(gs + mt * 2048 + (v & 1) * 1024 + cx[v >> 1]);
      if (mt == 1) {  // every operand of the stage is in registers: the slot can be refilled
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_16x8x16(acc[mt][nt], a, b[nt]);
    }
  }
  // epilogue: partial tile -> P[slab] (M x N column-major), fragment rows / columns through pr()
  double* p = P + z * M * N;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int64_t r = m0 + wm * 32 + mt * 16 + h * 8 + pg;
          const int64_t c = n0 + wn * 32 + nt * 8 + tm_pr(2 * t + q);
          if (r < M && c < N) p[r + c * M] = acc[mt][nt][h * 2 + q];
        }
}

typedef CUresult (*TmEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TmEncodeFn tm_encode() {
  static TmEncodeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<TmEncodeFn>(p);
  }
  return fn;
}

// rows x K fp64 matrix with K contiguous (ld doubles between rows), box 16 x box_rows, 128-byte swizzle
static bool tm_make_map(CUtensorMap* map, const double* A, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  TmEncodeFn enc = tm_encode();
  if (!enc) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)TM_BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void dense_reduce_kernel(const double* __restrict__ P, int64_t M, int64_t N, int S,
                                    double* __restrict__ Y, int64_t ldy, int64_t row_off,
                                    const Status* st) {
  if (st && failed(st)) return;
  const int64_t MN = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < MN; e += (int64_t)gridDim.x * blockDim.x) {
    // slab order (deterministic); eight slab loads in flight ahead of the adds
    double s = 0.0;
    int z = 0;
    for (; z + 8 <= S; z += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = P[(int64_t)(z + u) * MN + e];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; z < S; ++z) s += P[(int64_t)z * MN + e];
    const int64_t r = e % M, c = e / M;
    Y[row_off + r + c * ldy] = s;
  }
}

// CUDA-core path for the reduced-precision dense sketches (fp32 accumulate)
template <typename T>
__device__ __forceinline__ float dense_g(double g);
template <> __device__ __forceinline__ float dense_g<float>(double g) { return __double2float_rn(g); }
template <> __device__ __forceinline__ float dense_g<__half>(double g) { return __double2float_rn(g); }
template <> __device__ __forceinline__ float dense_g<__nv_bfloat16>(double g) {
  return __bfloat162float(__float2bfloat16_rn(__double2float_rn(g)));
}

template <typename T>
__global__ void __launch_bounds__(256)
dense_lowp_kernel(const double* __restrict__ G, int64_t ldg, const T* __restrict__ X, int64_t ldx,
                  int64_t M, int64_t K, double* __restrict__ Y, int64_t ldy, int64_t row_off,
                  const Status* st) {
  __shared__ double red[32];
  if (st && failed(st)) return;
  const int64_t i = blockIdx.x, c = blockIdx.y;
  float acc = 0.f;
  for (int64_t r = threadIdx.x; r < K; r += blockDim.x)
    acc = fmaf(dense_g<T>(G[i * ldg + r]), Lo<T>::load(X[r + c * ldx]), acc);
  const double tot = block_sum((double)acc, red);
  if (threadIdx.x == 0) Y[row_off + i + c * ldy] = (double)Lo<T>::rnd((float)tot);
}

static int dense_slabs(int64_t M, int64_t N, int64_t K, int sms, int64_t* kslab) {
  const int64_t tiles = ((M + DBM - 1) / DBM) * ((N + DBN - 1) / DBN);
  int64_t want = std::max<int64_t>(1, (2 * (int64_t)sms + tiles - 1) / tiles);
  int64_t ks = (K + want - 1) / want;
  ks = std::max<int64_t>(DBK, ((ks + DBK - 1) / DBK) * DBK);
  *kslab = ks;
  return (int)((K + ks - 1) / ks);
}

size_t dense_ws_bytes(const sqb_sketch* sk, int dtype, int64_t k) {
  if (dtype != SQB_F64) return 0;
  int64_t ks;
  const int S = dense_slabs(sk->ell, k, sk->n, 148, &ks);
  return sizeof(double) * (size_t)S * (size_t)sk->ell * (size_t)k;
}

template <>
int launch_dense<double>(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                         double* Y, int64_t ldy, int64_t row_off, void* ws, const Status* st) {
  int64_t ks;
  const int S = dense_slabs(sk->ell, k, sk->n, 148, &ks);
  static bool attr = false;
  if (!attr) {
    allow_dyn_smem(dense_dmma_kernel, (size_t)(DSMEM));
    attr = true;
  }
  dim3 grid((unsigned)((sk->ell + DBM - 1) / DBM), (unsigned)((k + DBN - 1) / DBN), (unsigned)S);
  prof_begin(ctx);
  // TMA + mbarrier kernel (256-row tiles): same slabs, same bits.  Needs 16-byte aligned operands with
  // 16-byte row strides; SQB_DENSE_CPASYNC=1 keeps the cp.async kernel (A/B)
  static const bool no_tma = [] { const char* e = getenv("SQB_DENSE_CPASYNC"); return e && e[0] == '1'; }();
  CUtensorMap mapG, mapX;
  const bool tma_ok = !no_tma && sk->ell > DBM && ks % TM_BK == 0 && (sk->ldg % 2 == 0) && (ldx % 2 == 0) &&
                      ((reinterpret_cast<uintptr_t>(sk->G) | reinterpret_cast<uintptr_t>(X)) & 15) == 0 &&
                      tm_make_map(&mapG, sk->G, sk->ell, sk->n, sk->ldg, TM_BM) &&
                      tm_make_map(&mapX, (const double*)X, k, sk->n, ldx, TM_BN);
  if (tma_ok) {
    static bool attr_t = false;
    if (!attr_t) {
      allow_dyn_smem(dense_tma_kernel, (size_t)(TM_SMEM));
      attr_t = true;
    }
    dim3 gt((unsigned)((sk->ell + TM_BM - 1) / TM_BM), (unsigned)((k + TM_BN - 1) / TM_BN), (unsigned)S);
    dense_tma_kernel<<<gt, TM_NT, TM_SMEM, ctx->stream>>>(mapG, mapX, sk->ell, k, sk->n, ks, (double*)ws, st);
    SQB_TRY(check_launch(ctx, "dense_tma_kernel"));
  } else {
    dense_dmma_kernel<<<grid, DNT, DSMEM, ctx->stream>>>(sk->G, sk->ldg, (const double*)X, ldx, sk->ell,
                                                          k, sk->n, ks, (double*)ws, st, 0);
    SQB_TRY(check_launch(ctx, "dense_dmma_kernel"));
  }
  prof_end(ctx, 2.0 * (double)sk->ell * (double)sk->n * (double)k);  // flops (bench.py: tensor roofline)
  const int64_t MN = sk->ell * k;
  const unsigned rb = (unsigned)std::min<int64_t>((MN + 255) / 256, 4096);
  dense_reduce_kernel<<<rb, 256, 0, ctx->stream>>>((const double*)ws, sk->ell, k, S, Y, ldy, row_off, st);
  return check_launch(ctx, "dense_reduce_kernel");
}

// The same split-K product in pieces (host_pipe.cu, sqb_rec_rhqr_host): the
// slab partition of launch_dense<double>, slabs [z0, z1) launched on `stream`
// as soon as their rows of X are resident, then the slab-order reduction —
// bitwise the one-shot launch.
int dense_slab_plan(const sqb_sketch* sk, int64_t k, int64_t* kslab) {
  return dense_slabs(sk->ell, k, sk->n, 148, kslab);
}

int launch_dense_slabs(sqb_ctx* ctx, cudaStream_t stream, const sqb_sketch* sk, const double* X, int64_t ldx,
                       int64_t k, int z0, int z1, int64_t kslab, void* ws, const Status* st) {
  static bool attr = false;
  if (!attr) {
    allow_dyn_smem(dense_dmma_kernel, (size_t)(DSMEM));
    attr = true;
  }
  if (z1 <= z0) return SQB_OK;
  dim3 grid((unsigned)((sk->ell + DBM - 1) / DBM), (unsigned)((k + DBN - 1) / DBN), (unsigned)(z1 - z0));
  dense_dmma_kernel<<<grid, DNT, DSMEM, stream>>>(sk->G, sk->ldg, X, ldx, sk->ell, k, sk->n, kslab, (double*)ws,
                                                 st, z0);
  return check_launch(ctx, "dense_dmma_kernel");
}

int launch_dense_reduce(sqb_ctx* ctx, const sqb_sketch* sk, int64_t k, int S, const void* ws, double* Y,
                        int64_t ldy, int64_t row_off, const Status* st) {
  const int64_t MN = sk->ell * k;
  const unsigned rb = (unsigned)std::min<int64_t>((MN + 255) / 256, 4096);
  dense_reduce_kernel<<<rb, 256, 0, ctx->stream>>>((const double*)ws, sk->ell, k, S, Y, ldy, row_off, st);
  return check_launch(ctx, "dense_reduce_kernel");
}

template <typename T>
int launch_dense(sqb_ctx* ctx, const sqb_sketch* sk, const void* X, int64_t ldx, int64_t k,
                 double* Y, int64_t ldy, int64_t row_off, void*, const Status* st) {
  dim3 grid((unsigned)sk->ell, (unsigned)k);
  dense_lowp_kernel<T><<<grid, 256, 0, ctx->stream>>>(sk->G, sk->ldg, (const T*)X, ldx, sk->ell,
                                                      sk->n, Y, ldy, row_off, st);
  return check_launch(ctx, "dense_lowp_kernel");
}

template int launch_dense<float>(sqb_ctx*, const sqb_sketch*, const void*, int64_t, int64_t, double*,
                                 int64_t, int64_t, void*, const Status*);
template int launch_dense<__half>(sqb_ctx*, const sqb_sketch*, const void*, int64_t, int64_t, double*,
                                  int64_t, int64_t, void*, const Status*);
template int launch_dense<__nv_bfloat16>(sqb_ctx*, const sqb_sketch*, const void*, int64_t, int64_t,
                                         double*, int64_t, int64_t, void*, const Status*);

}  // namespace sqb
