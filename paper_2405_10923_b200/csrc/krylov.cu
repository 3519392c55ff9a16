// RHQR-Arnoldi and GMRES on the device (krylov.py:82-222).
//
// Per Arnoldi step j (krylov.py:113-143) the host enqueues, without any sync
// (the unscaled w of each step is written straight into its basis column):
//   arn_step_kernel   happy-breakdown test, rh_vector on z (rhqr.py:51-97),
//                     S/T columns (_extend_t), the Hessenberg column, and the
//                     q-coefficients T_j S_j[j-1, :]^t                (1 CTA)
//   arn_q_kernel      q = e_j - U_j coef (GEMV over U_j) with the lazy scaling
//                     of U[:, j-1] (u = f w on the Omega rows)
//   matvec            w = lo(A lo(q)): CSR SpMV kernel (row sums in CSR order,
//                     unfused mul/add like scipy's csr_matvec), dense DMMA, or
//                     a host callback that enqueues on the stream
//   compact apply     w = (I - U T^t S^t Psi) w   (rhqr.py:100-119, transpose_t)
//   z = Psi w
// A closed Krylov space is recorded in the device status word (SQB_CLOSED);
// every later kernel of the chain is then a no-op.  One sync at the end.
#include <algorithm>
#include <cfloat>
#include <cooperative_groups.h>

#include "pdl.cuh"
#include "sketch.cuh"
#include "vec.cuh"
#include "gemv.cuh"
#include "dense.cuh"
#include "dist_common.cuh"

namespace cg = cooperative_groups;

namespace sqb {

int apply_reflectors_dispatch(sqb_ctx*, const sqb_sketch*, int64_t, int, const void*, int64_t, int64_t,
                              int64_t, const double*, int64_t, const double*, int64_t, int, const void*,
                              int64_t, int64_t, void*, int64_t, void*);
size_t apply_reflectors_ws_bytes(const sqb_sketch* sk, int dtype, int64_t m, int64_t r, int64_t k);

template <typename T>
__global__ void scale_col_kernel(T* __restrict__ u, int64_t n, int mt, const double* fscale, int scaling,
                                 const Status* st) {
  if (st && failed(st) && st->code != SQB_CLOSED) return;
  const double f = *fscale;
  for (int64_t i = mt + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)Lo<T>::load(u[i]);
    u[i] = Lo<T>::store(Lo<T>::from_double(scaling == SQB_SCALE_SQRT2 ? __dmul_rn(v, f) : __ddiv_rn(v, f)));
  }
}

constexpr int ARN_NT = 512;

// ---------------------------------------------------------------------------
// CSR SpMV: y = lo(b - A x) or lo(A x); x in the low dtype, A in fp64.
// Row sums run in CSR order with separate mul/add roundings, as scipy's
// csr_matvec (sum += Ax[jj] * Xx[Aj[jj]]) does.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
csr_spmv_kernel(int64_t n, const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                const double* __restrict__ data, const T* __restrict__ x, const double* __restrict__ bsub,
                T* __restrict__ y, double* __restrict__ y64, const Status* st) {
  if (st && failed(st)) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = __ldg(indptr + r), p1 = __ldg(indptr + r + 1);
    double s = 0.0;
    for (int64_t p = p0; p < p1; ++p)
      s = __dadd_rn(s, __dmul_rn(__ldg(data + p), (double)Lo<T>::load(x[__ldg(indices + p)])));
    if (bsub) s = __dsub_rn(bsub[r], s);
    if (y64) y64[r] = s;
    y[r] = Lo<T>::store(Lo<T>::from_double(s));
  }
}

// y = lo(b - r64) (initial residual when the product came from a dense/callback operator)
template <typename T>
__global__ void resid_kernel(int64_t n, const double* __restrict__ b, const double* __restrict__ r64,
                             T* __restrict__ y, const Status* st) {
  if (st && failed(st)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = Lo<T>::store(Lo<T>::from_double(b[i] - r64[i]));
}

template <typename T>
__global__ void round_kernel(int64_t n, const double* __restrict__ src, T* __restrict__ dst, const Status* st) {
  if (st && failed(st)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = Lo<T>::store(Lo<T>::from_double(src[i]));
}

template <typename T>
__global__ void widen_kernel(int64_t n, const T* __restrict__ src, double* __restrict__ dst, const Status* st) {
  if (st && failed(st)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = (double)Lo<T>::load(src[i]);
}

// ---------------------------------------------------------------------------
// Arnoldi step j (1-based) on z = Psi w (krylov.py:114-139)
// ---------------------------------------------------------------------------
struct ArnArgs {
  int j, m, mt, od;        // mt = m + 1 identity-block rows; od = mt + ell
  int scaling;
  double happy_tol;
  const double* z;         // (od)
  double* S; int64_t lds;  // od x (m+1)
  double* T; int64_t ldt;  // (m+1) x (m+1)
  double* H; int64_t ldh;  // (m+1) x m
  void* U; int64_t ldu;    // identity-block rows of U[:, j-1]
  double* beta;            // [1]
  double* fscale;          // [1] f of U[:, j-1]
  double* coefq;           // [j] T_j S_j[j-1, :]^t
  Status* st;
};

template <typename T>
__global__ void __launch_bounds__(ARN_NT) arn_step_kernel(ArnArgs a) {
  extern __shared__ double sm[];
  double* s = sm;           // [od]
  double* v = s + a.od;     // [m+1]
  double* red = v + a.mt;   // [32]
  __shared__ double scal[4];
  if (failed(a.st)) return;
  const int j = a.j, jj = j - 1, od = a.od, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = ARN_NT / 32;
  // happy breakdown test: ||z[j-1:]|| <= tol ||z||  (krylov.py:115-125)
  double pt = 0.0, pf = 0.0;
  for (int r = tid; r < od; r += ARN_NT) {
    const double zz = a.z[r] * a.z[r];
    pf += zz;
    if (r >= jj) pt += zz;
  }
  const double tail = sqrt(block_sum(pt, red));
  const double full = sqrt(block_sum(pf, red));
  if (tail <= a.happy_tol * full) {
    if (j >= 2) {
      for (int r = tid; r < jj; r += ARN_NT) a.H[r + (int64_t)(j - 2) * a.ldh] = a.z[r];
      if (tid == 0) {
        const double sg = a.z[jj] >= 0.0 ? 1.0 : -1.0;
        a.H[jj + (int64_t)(j - 2) * a.ldh] = -sg * tail;
      }
    }
    if (tid == 0) fail(a.st, SQB_CLOSED, j - 1, tail);
    return;
  }
  // rh_vector (rhqr.py:71-96); rho == tail
  if (tid == 0) {
    const double rho = tail, yc = a.z[jj];
    const double sigma = yc >= 0.0 ? 1.0 : -1.0;
    const double gamma = __dadd_rn(yc, sigma * rho);
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
    bool bad = false;
    if (rho == 0.0) { bad = true; fail(a.st, SQB_ERR_BREAKDOWN, j, 0.0); }
    else if (!isfinite(beta)) { bad = true; fail(a.st, SQB_ERR_BREAKDOWN, j, rho); }
    double f, bo;
    if (a.scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
    else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    scal[0] = -sigma * rho; scal[1] = gamma; scal[2] = f; scal[3] = bad ? -1.0 : bo;
    *a.fscale = f;
    // Hessenberg column (krylov.py:130-134)
    if (j == 1) *a.beta = -sigma * rho;
    else a.H[jj + (int64_t)(j - 2) * a.ldh] = -sigma * rho;
  }
  __syncthreads();
  const double gamma = scal[1], f = scal[2], bo = scal[3];
  if (bo < 0.0) return;
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  T* U = (T*)a.U;
  for (int r = tid; r < od; r += ARN_NT) {
    const double yh = r < jj ? 0.0 : (r == jj ? gamma : a.z[r]);
    const double sv = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s[r] = sv;
    a.S[r + (int64_t)jj * a.lds] = sv;
    if (r < a.mt) U[r + (int64_t)jj * a.ldu] = Lo<T>::store(Lo<T>::from_double(sv));
    if (j >= 2 && r < jj) a.H[r + (int64_t)(j - 2) * a.ldh] = a.z[r];  // w[:j-1]
  }
  __syncthreads();
  // _extend_t (rhqr.py:135-140): T[:jj, jj] = -beta T[:jj,:jj] (S[:, :jj]^t s)
  // (warp per output, lanes over the reduction index: warp_dot)
  for (int k = warp; k < jj; k += nw) {
    const double d = warp_dot(a.S + (int64_t)k * a.lds, s, max(k, jj), od);
    if (lane == 0) v[k] = d;
  }
  // S[j-1, :j] for the q coefficients (row jj of S, gathered once)
  double* srow = red + 32;  // [m+1]
  for (int k = tid; k < j; k += ARN_NT) srow[k] = a.S[jj + (int64_t)k * a.lds];
  __syncthreads();
  for (int i = warp; i < jj; i += nw) {
    const double d = warp_dot_strided(a.T + i, a.ldt, v, i, jj);
    if (lane == 0) a.T[i + (int64_t)jj * a.ldt] = __dmul_rn(-bo, d);
  }
  if (tid == 0) a.T[jj + (int64_t)jj * a.ldt] = bo;
  if (j > a.m) return;
  __syncthreads();
  // coef = T[:j,:j] S[j-1, :j]^t  (krylov.py:136)
  for (int i = warp; i < j; i += nw) {
    const double d = warp_dot_strided(a.T + i, a.ldt, srow, i, j);
    if (lane == 0) a.coefq[i] = d;
  }
}

// The same step on an 8-CTA thread-block cluster: the sketch-space rows are
// split in 8 blocks, the _extend_t dots are partial sums over each CTA's rows
// combined through DSMEM in rank order, and the T column / q coefficients
// are spread over the cluster's 64 warps (the one-CTA kernel above is L2-
// latency bound: 37 us per step at m = 200).  Scalars are computed
// identically by every CTA; rank 0 writes them.
constexpr int ASC = 8, ASC_NT = 256;

template <typename T>
__global__ void __cluster_dims__(ASC, 1, 1) __launch_bounds__(ASC_NT) arn_step_cl_kernel(ArnArgs a) {
  extern __shared__ double sm[];
  double* s = sm;            // [od]
  double* vp = s + a.od;     // [m+1] this CTA's partial v
  double* v = vp + a.mt;     // [m+1] v
  double* srow = v + a.mt;   // [m+1] S[j-1, :j]
  double* red = srow + a.mt; // [32]
  __shared__ double scal[4];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int j = a.j, jj = j - 1, od = a.od, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = ASC_NT / 32;
  const bool dead = failed(a.st);  // uniform: every CTA takes part in the syncs
  // happy breakdown test: ||z[j-1:]|| <= tol ||z||  (krylov.py:115-125)
  double pt = 0.0, pf = 0.0;
  if (!dead)
    for (int r = tid; r < od; r += ASC_NT) {
      const double zz = a.z[r] * a.z[r];
      pf += zz;
      if (r >= jj) pt += zz;
    }
  const double tail = sqrt(block_sum(pt, red));
  const double full = sqrt(block_sum(pf, red));
  const bool closed = !dead && tail <= a.happy_tol * full;
  if (closed && rank == 0) {
    if (j >= 2) {
      for (int r = tid; r < jj; r += ASC_NT) a.H[r + (int64_t)(j - 2) * a.ldh] = a.z[r];
      if (tid == 0) {
        const double sg = a.z[jj] >= 0.0 ? 1.0 : -1.0;
        a.H[jj + (int64_t)(j - 2) * a.ldh] = -sg * tail;
      }
    }
    if (tid == 0) fail(a.st, SQB_CLOSED, j - 1, tail);
  }
  // rh_vector (rhqr.py:71-96); rho == tail
  if (tid == 0) {
    const double rho = tail, yc = dead ? 0.0 : a.z[jj];
    const double sigma = yc >= 0.0 ? 1.0 : -1.0;
    const double gamma = __dadd_rn(yc, sigma * rho);
    const double beta = __ddiv_rn(1.0, __dmul_rn(__dmul_rn(rho, sigma), gamma));
    bool bad = dead || closed;
    if (!bad && rho == 0.0) { bad = true; if (rank == 0) fail(a.st, SQB_ERR_BREAKDOWN, j, 0.0); }
    else if (!bad && !isfinite(beta)) { bad = true; if (rank == 0) fail(a.st, SQB_ERR_BREAKDOWN, j, rho); }
    double f, bo;
    if (a.scaling == SQB_SCALE_SQRT2) { f = __dsqrt_rn(beta); bo = 1.0; }
    else { f = gamma; bo = __ddiv_rn(__dmul_rn(sigma, gamma), rho); }
    scal[0] = -sigma * rho; scal[1] = gamma; scal[2] = f; scal[3] = bad ? -1.0 : bo;
    if (rank == 0 && !bad) {
      *a.fscale = f;
      // Hessenberg column (krylov.py:130-134)
      if (j == 1) *a.beta = -sigma * rho;
      else a.H[jj + (int64_t)(j - 2) * a.ldh] = -sigma * rho;
    }
  }
  __syncthreads();
  const double gamma = scal[1], f = scal[2], bo = scal[3];
  if (bo < 0.0) return;  // uniform across the cluster (no DSMEM access yet)
  const bool sq = a.scaling == SQB_SCALE_SQRT2;
  T* U = (T*)a.U;
  const int B = (od + ASC - 1) / ASC, r0 = rank * B, r1 = min(od, r0 + B);
  for (int r = tid; r < od; r += ASC_NT) {
    const double yh = r < jj ? 0.0 : (r == jj ? gamma : a.z[r]);
    const double sv = sq ? __dmul_rn(yh, f) : __ddiv_rn(yh, f);
    s[r] = sv;
    if (r >= r0 && r < r1) {  // each CTA writes its own rows
      a.S[r + (int64_t)jj * a.lds] = sv;
      if (r < a.mt) U[r + (int64_t)jj * a.ldu] = Lo<T>::store(Lo<T>::from_double(sv));
      if (j >= 2 && r < jj) a.H[r + (int64_t)(j - 2) * a.ldh] = a.z[r];  // w[:j-1]
    }
  }
  for (int k = tid; k < j; k += ASC_NT) srow[k] = k == jj ? s[jj] : a.S[jj + (int64_t)k * a.lds];
  __syncthreads();
  // _extend_t (rhqr.py:135-140): partial S[:, :jj]^t s over this CTA's rows
  for (int k = warp; k < jj; k += nw) {
    const double d = warp_dot(a.S + (int64_t)k * a.lds, s, max(max(k, jj), r0), max(max(k, jj), r1));
    if (lane == 0) vp[k] = d;
  }
  cluster.sync();
  for (int k = tid; k < jj; k += ASC_NT) {
    double d = 0.0;
    for (int q = 0; q < ASC; ++q) d += cluster.map_shared_rank(vp, q)[k];
    v[k] = d;
  }
  cluster.sync();  // remote reads done; T column below is global
  // T[:jj, jj] = -beta T[:jj,:jj] v   (outputs over the cluster's 64 warps)
  const int gw = rank * nw + warp, ngw = ASC * nw;
  for (int i = gw; i < jj; i += ngw) {
    const double d = warp_dot_strided(a.T + i, a.ldt, v, i, jj);
    if (lane == 0) a.T[i + (int64_t)jj * a.ldt] = __dmul_rn(-bo, d);
  }
  if (rank == 0 && tid == 0) a.T[jj + (int64_t)jj * a.ldt] = bo;
  if (j > a.m) return;
  cluster.sync();  // the new T column (global, other CTAs) is visible
  // coef = T[:j,:j] S[j-1, :j]^t  (krylov.py:136)
  for (int i = gw; i < j; i += ngw) {
    const int lo = i + lane;
    double d0 = 0.0;
    for (int k = lo; k < j; k += 32) d0 = fma(__ldcg(a.T + i + (int64_t)k * a.ldt), srow[k], d0);
    d0 = warp_sum(d0);
    if (lane == 0) a.coefq[i] = d0;
  }
}

// q = e_j - lo(U_j coef) (krylov.py:137-139); lazy scaling of U[:, j-1] rows >= mt
// (the local rows past the identity block; row0 = global index of local row 0);
// q_lo = round(q) feeds the matvec, Q[:, j-1] = q (fp64) when stored.
// Streaming GEMV core over the final columns 0..j-2 (gemv.cuh).
template <typename T>
__global__ void __launch_bounds__(GEMV_NT, 2)
arn_q_kernel(int64_t n, int mt, int j, T* U, int64_t ldu, const double* __restrict__ coefq,
             const double* __restrict__ fscale, int scaling, T* __restrict__ q, double* __restrict__ Q,
             const Status* st, int64_t row0 = 0) {
  using A = typename Lo<T>::acc;
  constexpr int VN = VecN<T>::n, NV = 4;
  extern __shared__ unsigned char smraw[];
  A* c = reinterpret_cast<A*>(smraw);
  if (failed(st)) return;
  for (int k = threadIdx.x; k < j; k += blockDim.x) c[k] = Lo<T>::from_double(coefq[k]);
  __syncthreads();
  const double f = *fscale;
  const int jj = j - 1;
  T* uj = U + (int64_t)jj * ldu;
  const int64_t rows_per = (int64_t)GEMV_NT * NV * VN;
  for (int64_t r0 = (int64_t)blockIdx.x * rows_per; r0 < n; r0 += (int64_t)gridDim.x * rows_per) {
    A acc[NV][VN];
    gemv_rows<T, NV>(U, ldu, r0, n, jj, c, acc);
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        const int64_t i = r0 + (v * GEMV_NT + threadIdx.x) * VN + e;
        if (i >= n) continue;
        A x = Lo<T>::load(uj[i]);
        if (i >= mt) {  // Omega rows hold the unscaled w: u = fl(f w) (rhqr.py:86-95)
          const double u = scaling == SQB_SCALE_SQRT2 ? __dmul_rn((double)x, f) : __ddiv_rn((double)x, f);
          x = Lo<T>::from_double(u);
          uj[i] = Lo<T>::store(x);
        }
        const A a = fma(x, c[jj], acc[v][e]);
        double qv = -(double)Lo<T>::rnd(a);
        if (row0 + i == jj) qv = qv + 1.0;  // e_j (global row j-1: rank 0's identity rows)
        q[i] = Lo<T>::store(Lo<T>::from_double(qv));
        if (Q) Q[i] = qv;
      }
  }
}

struct OpDesc {
  int kind;  // 0 csr, 1 dense, 2 callback
  int64_t n;
  const int64_t* indptr;
  const int32_t* indices;
  const double* data;
  sqb_sketch dense;  // G = A (row-major) for the dense matvec
  sqb_matvec_cb cb;
  void* user;
  void* xbuf;
  double* ybuf;
};

template <typename T>
static int matvec_t(sqb_ctx* ctx, const OpDesc& op, const T* x, const double* bsub, T* y, double* tmp64,
                    void* dense_ws, const Status* st) {
  const int64_t n = op.n;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16 * 148));
  if (op.kind == SQB_OP_CSR) {
    csr_spmv_kernel<T><<<grid, 256, 0, ctx->stream>>>(n, op.indptr, op.indices, op.data, x, bsub, y, nullptr, st);
    return check_launch(ctx, "csr_spmv_kernel");
  }
  // dense (K2 GEMM with k = 1) or callback: fp64 product into tmp64, then round
  if (op.kind == SQB_OP_DENSE) {
    // the reference multiplies in float64 (A @ round_to(q, low)): widen, then the K2 GEMM
    double* x64 = tmp64 + n;
    widen_kernel<T><<<grid, 256, 0, ctx->stream>>>(n, x, x64, st);
    SQB_TRY(check_launch(ctx, "widen_kernel"));
    SQB_TRY(launch_dense<double>(ctx, &op.dense, x64, n, 1, tmp64, n, 0, dense_ws, st));
  } else {
    SQB_CUDA_TRY(cudaMemcpyAsync(op.xbuf, x, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    int rc = op.cb(op.user, ctx->stream);
    if (rc != 0) return set_error(ctx, SQB_ERR_ARG, "matvec callback failed (%d)", rc);
    SQB_CUDA_TRY(cudaMemcpyAsync(tmp64, op.ybuf, sizeof(double) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (bsub) resid_kernel<T><<<grid, 256, 0, ctx->stream>>>(n, bsub, tmp64, y, st);
  else round_kernel<T><<<grid, 256, 0, ctx->stream>>>(n, tmp64, y, st);
  return check_launch(ctx, "matvec_round");
}

template <typename T>
static int arnoldi_t(sqb_ctx* ctx, const sqb_sketch* sk, const OpDesc& op, int m, int scaling, double happy_tol,
                     const double* b, const void* x0lo, void* U, int64_t ldu, double* S, int64_t lds, double* Tm,
                     int64_t ldt, double* H, int64_t ldh, double* Q, int64_t ldq, double* beta, int* attained) {
  const int64_t n = op.n;
  const int mt = m + 1;
  const int64_t od = mt + sk->ell;
  WsPlan plan;
  const size_t iz = plan.add(sizeof(double) * od);
  const size_t iY = plan.add(sizeof(double) * od);
  const size_t iC = plan.add(sizeof(double) * (mt + 1));
  const size_t icq = plan.add(sizeof(double) * (mt + 1));
  const size_t ifs = plan.add(sizeof(double) * 2);
  const size_t iw = plan.add(sizeof(T) * (n + 32));
  const size_t iq = plan.add(sizeof(T) * (n + 32));
  const size_t it64 = plan.add(op.kind == SQB_OP_CSR ? 8 : sizeof(double) * 2 * n);
  const size_t iAR = plan.add(apply_reflectors_ws_bytes(sk, Lo<T>::code, mt, mt, 1));
  const size_t iP = plan.add(std::max(sketch_partials_bytes(sk, Lo<T>::code, 1),
                                      op.kind == SQB_OP_DENSE ? dense_ws_bytes(&op.dense, SQB_F64, 1) : 0));
  SQB_TRY(ws_reserve(ctx, plan.total));
  double* z = ws_ptr<double>(ctx, plan, iz);
  double* fs = ws_ptr<double>(ctx, plan, ifs);
  double* cq = ws_ptr<double>(ctx, plan, icq);
  // w is sketched from row mt on (apply_reflectors): shift it so that w + mt is 16-byte aligned and the
  // sketch takes the TMA kernels instead of the scalar-load tile kernel (mt = m + 1 is odd for even m)
  T* w = ws_ptr<T>(ctx, plan, iw) + (VecN<T>::n - mt % VecN<T>::n) % VecN<T>::n;
  T* q = ws_ptr<T>(ctx, plan, iq);
  double* t64 = ws_ptr<double>(ctx, plan, it64);
  void* P = ws_ptr<void>(ctx, plan, iP);
  Status* st = ctx->d_status;
  // zero the outputs the steps fill column by column
  SQB_CUDA_TRY(cudaMemsetAsync(Tm, 0, sizeof(double) * ldt * mt, ctx->stream));
  SQB_CUDA_TRY(cudaMemsetAsync(H, 0, sizeof(double) * ldh * m, ctx->stream));
  SQB_CUDA_TRY(cudaMemsetAsync(beta, 0, sizeof(double), ctx->stream));
  // w = lo(b - A lo(x0)); z = Psi w   (krylov.py:111-112).  The unscaled w
  // of every step is written straight into its basis column U[:, j-1] (rows
  // >= mt; the step kernel writes the identity rows): no copy of w into U.
  SQB_TRY(matvec_t<T>(ctx, op, (const T*)x0lo, b, (T*)U, t64, P, st));
  defer_copy_top(ctx, Lo<T>::code, U, n, mt, 1, z, od);
  SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (T*)U + mt, n, 1, z, od, mt, P, st));
  SQB_TRY(flush_copy_top(ctx, st));
  const size_t step_smem = sizeof(double) * (od + 3 * mt + 32);
  allow_dyn_smem(arn_step_cl_kernel<T>, (size_t)(std::max<size_t>(step_smem, 48 << 10)));
  constexpr int VN = VecN<T>::n;
  if (!(((reinterpret_cast<uintptr_t>(U) & 15) == 0) && (ldu % VN == 0)))
    return set_error(ctx, SQB_ERR_ARG, "Arnoldi basis U must be 16-byte aligned with ldu %% %d == 0", VN);
  const unsigned gq = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n / VN + 255) / 256, 4 * 148));
  const unsigned gg = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((n + (int64_t)GEMV_NT * 4 * VN - 1) / ((int64_t)GEMV_NT * 4 * VN), 2 * (int64_t)ctx->sm_count));
  for (int j = 1; j <= mt; ++j) {
    T* uj = (T*)U + (int64_t)(j - 1) * ldu;
    ArnArgs aa{j, m, mt, (int)od, scaling, happy_tol, z, S, lds, Tm, ldt, H, ldh, U, ldu, beta, fs, cq, st};
    arn_step_cl_kernel<T><<<ASC, ASC_NT, step_smem, ctx->stream>>>(aa);
    SQB_TRY(check_launch(ctx, "arn_step_kernel"));
    if (j > m) {
      // lazy scaling of the last column's Omega rows
      scale_col_kernel<T><<<gq, 256, 0, ctx->stream>>>(uj, n, mt, fs, scaling, st);
      SQB_TRY(check_launch(ctx, "scale_col_kernel"));
      break;
    }
    double* Qj = Q ? Q + (int64_t)(j - 1) * ldq : nullptr;
    prof_begin(ctx);
    arn_q_kernel<T><<<gg, GEMV_NT, sizeof(double) * (mt + 1), ctx->stream>>>(n, mt, j, (T*)U, ldu, cq, fs,
                                                                             scaling, q, Qj, st);
    SQB_TRY(check_launch(ctx, "arn_q_kernel"));
    // algorithmic bytes of the GEMV q = e_j - U_j coef: read U[:, :j], write q
    prof_end(ctx, (double)sizeof(T) * (double)n * (double)(j + 1));
    // w = lo(A lo(q))  (krylov.py:140)
    SQB_TRY(matvec_t<T>(ctx, op, q, nullptr, w, t64, P, st));
    // U[:, j] = (I - U_j T_j^t S_j^t Psi) w  (krylov.py:141-142): the update
    // writes the next basis column in place
    static const bool via_w = [] { const char* e = getenv("SQB_ARN_COPY"); return e && e[0] == '1'; }();
    T* unext = via_w ? w : (T*)U + (int64_t)j * ldu;
    SQB_TRY(apply_reflectors_dispatch(ctx, sk, mt, Lo<T>::code, U, ldu, n, j, S, lds, Tm, ldt, 1, w, n, 1, unext,
                                      ldu, ws_ptr<void>(ctx, plan, iAR)));
    // z = Psi w  (krylov.py:143)
    defer_copy_top(ctx, Lo<T>::code, unext, n, mt, 1, z, od);
    SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, unext + mt, n, 1, z, od, mt, P, st));
    SQB_TRY(flush_copy_top(ctx, st));
    if (via_w)  // A/B: the unscaled w copied into its basis column
      SQB_CUDA_TRY(cudaMemcpyAsync((T*)U + (int64_t)j * ldu + mt, w + mt, sizeof(T) * (n - mt),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  }
  // read the outcome (the only sync of the whole Arnoldi run)
  SQB_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(Status), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  const Status hs = *ctx->h_status;
  if (hs.code == SQB_CLOSED) {
    // the space closed at step attained+1: every accepted reflector is final
    // (column attained-1 was scaled by the arn_q pass of step attained; the
    // unscaled w copied into column attained is past the returned factors)
    *attained = hs.col;
    SQB_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(Status), ctx->stream));
  } else {
    *attained = -1;
  }
  return SQB_OK;
}

// ---------------------------------------------------------------------------
// Hessenberg least squares by Givens rotations (krylov.py:153-190), one CTA
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
hess_lstsq_kernel(const double* __restrict__ H, int64_t ldh, int p, int k, double beta, double* R, double* g,
                  double* y, double* hist, double* resid) {
  __shared__ double red[32];
  __shared__ double cs_sn[2];
  const int tid = threadIdx.x;
  for (int e = tid; e < p * k; e += 256) R[(e % p) + (int64_t)(e / p) * p] = H[(e % p) + (int64_t)(e / p) * ldh];
  for (int i = tid; i < p; i += 256) g[i] = i == 0 ? beta : 0.0;
  if (tid == 0) hist[0] = fabs(beta);
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      const double a = R[j + (int64_t)j * p], t = R[j + 1 + (int64_t)j * p];
      const double r = hypot(a, t);
      double cs = 1.0, sn = 0.0;
      if (r != 0.0) { cs = a / r; sn = t / r; }
      cs_sn[0] = cs; cs_sn[1] = sn;
      const double g0 = g[j], g1 = g[j + 1];
      g[j] = cs * g0 + sn * g1;
      g[j + 1] = -sn * g0 + cs * g1;
      hist[j + 1] = fabs(g[j + 1]);
    }
    __syncthreads();
    const double cs = cs_sn[0], sn = cs_sn[1];
    for (int c = j + tid; c < k; c += 256) {
      const double r1 = R[j + (int64_t)c * p], r2 = R[j + 1 + (int64_t)c * p];
      R[j + (int64_t)c * p] = cs * r1 + sn * r2;
      R[j + 1 + (int64_t)c * p] = -sn * r1 + cs * r2;
    }
    __syncthreads();
  }
  for (int i = k - 1; i >= 0; --i) {
    double part = 0.0;
    for (int c = i + 1 + tid; c < k; c += 256) part = fma(R[i + (int64_t)c * p], y[c], part);
    const double dot = block_sum(part, red);
    if (tid == 0) {
      const double rii = R[i + (int64_t)i * p];
      y[i] = rii == 0.0 ? 0.0 : (g[i] - dot) / rii;
    }
    __syncthreads();
  }
  if (tid == 0) *resid = p > k ? fabs(g[k]) : 0.0;
}

template <typename T>
static int arnoldi_dispatch_t(sqb_ctx* ctx, const sqb_sketch* sk, const OpDesc& op, int m, int scaling,
                              double happy_tol, const double* b, const void* x0lo, void* U, int64_t ldu,
                              double* S, int64_t lds, double* Tm, int64_t ldt, double* H, int64_t ldh,
                              double* Q, int64_t ldq, double* beta, int* attained) {
  return arnoldi_t<T>(ctx, sk, op, m, scaling, happy_tol, b, x0lo, U, ldu, S, lds, Tm, ldt, H, ldh, Q, ldq,
                      beta, attained);
}

// ---------------------------------------------------------------------------
// Row-partitioned RHQR-Arnoldi.  Rank p owns the rows of the
// Omega coordinates [p n_pad/P, (p+1) n_pad/P) (whole SRHT tiles) and rank 0
// also the m+1 identity-block rows, so every rank's rows are one contiguous
// range.  Per step the exchanges are (a) the all-gather of q for the SpMV
// (each rank multiplies its own CSR rows, whose column indices the caller has
// remapped into the gathered [rank][seg] layout), and (b) two (ell+m+1)-vector
// all-gathers of the rank-local SRHT subtrees (the projection's sketch and
// z = Psi w), combined in rank order — the single-GPU tree, so z, H, S, T
// and beta are bitwise the single-GPU ones.  The sketch-space step runs
// redundantly on every rank; U, w, q and the Krylov rows never move.
// ---------------------------------------------------------------------------
int compact_update_dispatch(sqb_ctx* ctx, int lo_dtype, const double* Y, int64_t od, const double* S, int64_t lds,
                            const double* Tm, int64_t ldt, int transpose_t, int64_t r, const void* U, int64_t ldu,
                            int64_t N, const void* X, void* Out, double* C);

struct ArnRank {
  int64_t rows;     // local rows (identity block included on rank 0)
  int mrow;         // m+1 on rank 0, else 0
  int64_t row0;     // global row of local row 0
  int64_t e_base;   // first global Omega coordinate
  const int64_t* indptr; const int32_t* indices; const double* data;  // local CSR rows, remapped columns
  const double* b; const void* x0lo;                                  // local rows
  void* U; int64_t ldu; double* Q; int64_t ldq;
  double *S, *T, *H, *beta; int64_t lds, ldt, ldh;
  void* Utop; int64_t ldutop;                                         // identity rows of U (ranks > 0: scratch)
  // workspace
  double *z, *Y, *C, *cq, *fs, *pay;
  void *w, *q, *P;
};

template <typename T>
static int arnoldi_dist_t(sqb_ctx* ctx, const sqb_sketch* sk, int m, int scaling, double happy_tol,
                          std::vector<ArnRank>& rk, int nranks, bool virt, const std::vector<int>& ids, int64_t seg,
                          int* attained) {
  using A = typename Lo<T>::acc;
  const int mt = m + 1;
  const int64_t ell = sk->ell, od = mt + ell, pl = ell + mt;
  const SrhtGeom g = srht_geom_t<T>(sk);
  if (g.n_tiles % nranks != 0)
    return set_error(ctx, SQB_ERR_ARG, "n_pad=%lld too small for %d ranks", (long long)sk->n_pad, nranks);
  const int64_t tpr = g.n_tiles / nranks, tb = int64_t(1) << g.log_tb;
  int rank_level = 0;
  while ((int64_t(1) << rank_level) < tpr) ++rank_level;
  const int L = (int)rk.size();
  constexpr int VN = VecN<T>::n;
  WsPlan plan;
  std::vector<size_t> off(L * 9);
  for (int r = 0; r < L; ++r) {
    off[r * 9 + 0] = plan.add(sizeof(double) * od);             // z
    off[r * 9 + 1] = plan.add(sizeof(double) * od);             // Y (projection sketch)
    off[r * 9 + 2] = plan.add(sizeof(double) * (mt + 1));       // C
    off[r * 9 + 3] = plan.add(sizeof(double) * (mt + 1));       // cq
    off[r * 9 + 4] = plan.add(sizeof(double) * 2);              // fs
    off[r * 9 + 5] = plan.add(sizeof(double) * pl);             // payload
    off[r * 9 + 6] = plan.add(sizeof(T) * (seg + 2 * VN));      // w
    off[r * 9 + 7] = plan.add(sizeof(T) * (seg + 2 * VN));      // q
    off[r * 9 + 8] = plan.add(sizeof(A) * ell * tpr);           // leaves
  }
  const bool halo = ctx->halo.size() == (size_t)nranks * nranks * 2;
  // virtual ranks with halo ranges: one gathered buffer per rank (each holds
  // only what its own rows reference — a wrong range shows up as wrong bits)
  const size_t iGq = plan.add(sizeof(T) * nranks * seg * (halo && virt ? L : 1));
  const size_t iGs = plan.add(sizeof(double) * nranks * pl);
  SQB_TRY(ws_reserve(ctx, plan.total));
  char* base = static_cast<char*>(ctx->ws);
  for (int r = 0; r < L; ++r) {
    ArnRank& d = rk[r];
    d.z = (double*)(base + plan.offs[off[r * 9 + 0]]);
    d.Y = (double*)(base + plan.offs[off[r * 9 + 1]]);
    d.C = (double*)(base + plan.offs[off[r * 9 + 2]]);
    d.cq = (double*)(base + plan.offs[off[r * 9 + 3]]);
    d.fs = (double*)(base + plan.offs[off[r * 9 + 4]]);
    d.pay = (double*)(base + plan.offs[off[r * 9 + 5]]);
    // w, q: the Omega rows (local row mrow) start 16-byte aligned
    const int shift = (int)((VN - d.mrow % VN) % VN);
    d.w = (T*)(base + plan.offs[off[r * 9 + 6]]) + shift;
    d.q = (T*)(base + plan.offs[off[r * 9 + 7]]) + shift;
    d.P = base + plan.offs[off[r * 9 + 8]];
  }
  T* Gq = (T*)(base + plan.offs[iGq]);
  if (halo)
    SQB_CUDA_TRY(cudaMemsetAsync(Gq, 0, sizeof(T) * nranks * seg * (virt ? L : 1), ctx->stream));
  double* Gs = (double*)(base + plan.offs[iGs]);
  Status* st = ctx->d_status;
  double scale_lo = 0.0, norm_lo = 0.0;
  srht_constants(sk, Lo<T>::code, &scale_lo, &norm_lo);

  // Psi (local rows of) v for every rank -> out[r] (od): local subtrees, one
  // all-gather, rank-order combine
  auto sketch_all = [&](void* ArnRank::*vsel, double* ArnRank::*osel) -> int {
    std::vector<const void*> send(L);
    for (int r = 0; r < L; ++r) {
      ArnRank& d = rk[r];
      const T* v = (const T*)(d.*vsel);
      const int64_t n_local = d.rows - d.mrow;
      SrhtGeom gl{g.log_tb, tpr, (n_local + tb - 1) / tb};
      if (n_local > 0) SQB_TRY(launch_srht_tiles_geom(ctx, sk, Lo<T>::code, gl, n_local, d.e_base, v + d.mrow,
                                                      n_local, 1, d.P, st));
      else SQB_CUDA_TRY(cudaMemsetAsync(d.P, 0, sizeof(A) * ell * tpr, ctx->stream));
      SQB_TRY(launch_srht_tree_geom(ctx, sk, Lo<T>::code, gl, d.P, 1, d.pay, pl, 0, 0, st));
      if (d.mrow > 0) SQB_TRY(launch_copy_top(ctx, Lo<T>::code, v, d.rows, mt, 1, d.pay + ell, pl, st));
      send[r] = d.pay;
    }
    SQB_TRY(dist_allgather(ctx, virt, ids, send, sizeof(double) * pl, Gs));
    for (int r = 0; r < L; ++r) {
      rank_combine_kernel<T><<<dim3((unsigned)((od + 255) / 256), 1), 256, 0, ctx->stream>>>(
          Gs, nranks, (int)ell, mt, 1, rank_level, sk->indices, g.log_tb, norm_lo, rk[r].*osel, od, st);
      SQB_TRY(check_launch(ctx, "rank_combine_kernel"));
    }
    return SQB_OK;
  };
  // q for the SpMV: the halo exchange when the caller set the ranges
  // (sqb_ctx_set_halo), else the all-gather of the whole vector
  auto gather_T = [&](void* ArnRank::*sel) -> int {
    std::vector<const void*> send(L);
    for (int r = 0; r < L; ++r) send[r] = rk[r].*sel;
    if (halo) {
      std::vector<int64_t> rows(L);
      std::vector<void*> G(L);
      for (int r = 0; r < L; ++r) {
        rows[r] = rk[r].rows;
        G[r] = Gq + (virt ? (int64_t)r * nranks * seg : 0);
      }
      return dist_halo_exchange(ctx, virt, ids, nranks, send, rows, sizeof(T), seg, G);
    }
    return dist_allgather(ctx, virt, ids, send, sizeof(T) * seg, Gq);
  };
  auto spmv = [&](ArnRank& d, const double* bsub) -> int {
    const int r = (int)(&d - rk.data());
    const T* Gr = Gq + (halo && virt ? (int64_t)r * nranks * seg : 0);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((d.rows + 255) / 256, 16 * 148));
    csr_spmv_kernel<T><<<grid, 256, 0, ctx->stream>>>(d.rows, d.indptr, d.indices, d.data, Gr, bsub, (T*)d.w,
                                                      nullptr, st);
    return check_launch(ctx, "csr_spmv_kernel");
  };

  // w = lo(b - A lo(x0)); z = Psi w  (krylov.py:111-112)
  for (int r = 0; r < L; ++r) {
    ArnRank& d = rk[r];
    SQB_CUDA_TRY(cudaMemsetAsync(d.T, 0, sizeof(double) * d.ldt * mt, ctx->stream));
    SQB_CUDA_TRY(cudaMemsetAsync(d.H, 0, sizeof(double) * d.ldh * m, ctx->stream));
    SQB_CUDA_TRY(cudaMemsetAsync(d.beta, 0, sizeof(double), ctx->stream));
    SQB_CUDA_TRY(cudaMemcpyAsync(d.q, d.x0lo, sizeof(T) * d.rows, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  SQB_TRY(gather_T(&ArnRank::q));
  for (int r = 0; r < L; ++r) SQB_TRY(spmv(rk[r], rk[r].b));
  SQB_TRY(sketch_all(&ArnRank::w, &ArnRank::z));
  const size_t step_smem = sizeof(double) * (od + 3 * mt + 32);
  allow_dyn_smem(arn_step_cl_kernel<T>, (size_t)(std::max<size_t>(step_smem, 48 << 10)));
  for (int j = 1; j <= mt; ++j) {
    for (int r = 0; r < L; ++r) {
      ArnRank& d = rk[r];
      T* uj = (T*)d.U + (int64_t)(j - 1) * d.ldu;
      if (d.rows > d.mrow)
        SQB_CUDA_TRY(cudaMemcpyAsync(uj + d.mrow, (T*)d.w + d.mrow, sizeof(T) * (d.rows - d.mrow),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
      ArnArgs aa{j, m, mt, (int)od, scaling, happy_tol, d.z, d.S, d.lds, d.T, d.ldt, d.H, d.ldh, d.Utop, d.ldutop,
                 d.beta, d.fs, d.cq, st};
      arn_step_cl_kernel<T><<<ASC, ASC_NT, step_smem, ctx->stream>>>(aa);
      SQB_TRY(check_launch(ctx, "arn_step_kernel"));
      if (j > m) {
        const unsigned gq = (unsigned)std::max<int64_t>(1, std::min<int64_t>((d.rows / VN + 255) / 256, 4 * 148));
        scale_col_kernel<T><<<gq, 256, 0, ctx->stream>>>(uj, d.rows, d.mrow, d.fs, scaling, st);
        SQB_TRY(check_launch(ctx, "scale_col_kernel"));
      }
    }
    if (j > m) break;
    for (int r = 0; r < L; ++r) {
      ArnRank& d = rk[r];
      const unsigned gg = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>((d.rows + (int64_t)GEMV_NT * 4 * VN - 1) / ((int64_t)GEMV_NT * 4 * VN),
                               2 * (int64_t)ctx->sm_count));
      double* Qj = d.Q ? d.Q + (int64_t)(j - 1) * d.ldq : nullptr;
      arn_q_kernel<T><<<gg, GEMV_NT, sizeof(double) * (mt + 1), ctx->stream>>>(
          d.rows, d.mrow, j, (T*)d.U, d.ldu, d.cq, d.fs, scaling, (T*)d.q, Qj, st, d.row0);
      SQB_TRY(check_launch(ctx, "arn_q_kernel"));
    }
    // w = lo(A lo(q))  (krylov.py:140)
    SQB_TRY(gather_T(&ArnRank::q));
    for (int r = 0; r < L; ++r) SQB_TRY(spmv(rk[r], nullptr));
    // w = (I - U_j T_j^t S_j^t Psi) w  (krylov.py:141-142)
    SQB_TRY(sketch_all(&ArnRank::w, &ArnRank::Y));
    for (int r = 0; r < L; ++r) {
      ArnRank& d = rk[r];
      SQB_TRY(compact_update_dispatch(ctx, Lo<T>::code, d.Y, od, d.S, d.lds, d.T, d.ldt, 1, j, d.U, d.ldu, d.rows,
                                      d.w, d.w, d.C));
    }
    // z = Psi w  (krylov.py:143)
    SQB_TRY(sketch_all(&ArnRank::w, &ArnRank::z));
  }
  SQB_CUDA_TRY(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(Status), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  const Status hs = *ctx->h_status;
  if (hs.code == SQB_CLOSED) {
    *attained = hs.col;
    SQB_CUDA_TRY(cudaMemsetAsync(ctx->d_status, 0, sizeof(Status), ctx->stream));
  } else {
    *attained = -1;
  }
  return SQB_OK;
}

static int arnoldi_dist_entry(sqb_ctx* ctx, const sqb_sketch* sk, int m, int scaling, int lo_dtype, double happy_tol,
                              std::vector<ArnRank>& rk, int nranks, bool virt, const std::vector<int>& ids,
                              int64_t seg, int* attained) {
  SQB_TRY(validate_sketch(ctx, sk));
  if (sk->kind != SQB_SKETCH_SRHT) return set_error(ctx, SQB_ERR_ARG, "the row-partitioned Arnoldi needs an SRHT");
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need m >= 1");
  if (sk->ell < m + 1) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (nranks < 1 || nranks > 8 || (nranks & (nranks - 1)))
    return set_error(ctx, SQB_ERR_ARG, "nranks must be a power of two <= 8");
  const int64_t span = sk->n_pad / nranks;
  for (auto& d : rk) {
    if (d.rows > seg) return set_error(ctx, SQB_ERR_ARG, "local rows exceed the gather segment");
    if (d.mrow == 0 && d.rows > span) return set_error(ctx, SQB_ERR_ARG, "local rows exceed the Omega span");
  }
  switch (lo_dtype) {
    case SQB_F64: return arnoldi_dist_t<double>(ctx, sk, m, scaling, happy_tol, rk, nranks, virt, ids, seg, attained);
    case SQB_F32: return arnoldi_dist_t<float>(ctx, sk, m, scaling, happy_tol, rk, nranks, virt, ids, seg, attained);
    case SQB_F16: return arnoldi_dist_t<__half>(ctx, sk, m, scaling, happy_tol, rk, nranks, virt, ids, seg, attained);
    case SQB_BF16:
      return arnoldi_dist_t<__nv_bfloat16>(ctx, sk, m, scaling, happy_tol, rk, nranks, virt, ids, seg, attained);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb

using namespace sqb;

extern "C" int sqb_rhqr_arnoldi(sqb_ctx* ctx, const sqb_sketch* sk, const sqb_operator* A, int m, int scaling,
                                int lo_dtype, double happy_tol, const double* b, const void* x0lo, void* U,
                                int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt, double* H,
                                int64_t ldh, double* Q, int64_t ldq, double* beta, int* attained) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(validate_sketch(ctx, sk));
  if (!A || A->n < 1) return set_error(ctx, SQB_ERR_ARG, "missing operator");
  if (m < 1) return set_error(ctx, SQB_ERR_ARG, "need m >= 1");
  if (sk->n != A->n - m - 1)
    return set_error(ctx, SQB_ERR_ARG, "sketch takes %lld coordinates, expected n-m=%lld", (long long)sk->n,
                     (long long)(A->n - m - 1));
  if (sk->ell < m + 1) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  OpDesc op{};
  op.kind = A->kind;
  op.n = A->n;
  op.indptr = A->indptr;
  op.indices = A->indices;
  op.data = A->data;
  op.cb = A->cb;
  op.user = A->user;
  op.xbuf = A->xbuf;
  op.ybuf = A->ybuf;
  if (A->kind == SQB_OP_DENSE) {
    op.dense.kind = SQB_SKETCH_DENSE;
    op.dense.ell = A->n;
    op.dense.n = A->n;
    op.dense.G = A->A;
    op.dense.ldg = A->lda;
  } else if (A->kind == SQB_OP_CSR) {
    if (!A->indptr || !A->indices || !A->data) return set_error(ctx, SQB_ERR_ARG, "incomplete CSR operator");
  } else if (A->kind == SQB_OP_CALLBACK) {
    if (!A->cb || !A->xbuf || !A->ybuf) return set_error(ctx, SQB_ERR_ARG, "incomplete matvec callback");
  } else {
    return set_error(ctx, SQB_ERR_ARG, "unknown operator kind %d", A->kind);
  }
  switch (lo_dtype) {
    case SQB_F64: return arnoldi_dispatch_t<double>(ctx, sk, op, m, scaling, happy_tol, b, x0lo, U, ldu, S, lds, T, ldt, H, ldh, Q, ldq, beta, attained);
    case SQB_F32: return arnoldi_dispatch_t<float>(ctx, sk, op, m, scaling, happy_tol, b, x0lo, U, ldu, S, lds, T, ldt, H, ldh, Q, ldq, beta, attained);
    case SQB_F16: return arnoldi_dispatch_t<__half>(ctx, sk, op, m, scaling, happy_tol, b, x0lo, U, ldu, S, lds, T, ldt, H, ldh, Q, ldq, beta, attained);
    case SQB_BF16: return arnoldi_dispatch_t<__nv_bfloat16>(ctx, sk, op, m, scaling, happy_tol, b, x0lo, U, ldu, S, lds, T, ldt, H, ldh, Q, ldq, beta, attained);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

extern "C" int sqb_hessenberg_lstsq(sqb_ctx* ctx, const double* H, int64_t ldh, int64_t p, int64_t k, double beta,
                                    double* y, double* hist, double* resid, double* work) {
  SQB_TRY(begin_entry(ctx));
  if (p < k || k < 0) return set_error(ctx, SQB_ERR_ARG, "Hessenberg must be (k+1) x k");
  double* R = work;
  double* g = work + p * std::max<int64_t>(k, 1);
  hess_lstsq_kernel<<<1, 256, 0, ctx->stream>>>(H, ldh, (int)p, (int)k, beta, R, g, y, hist, resid);
  return check_launch(ctx, "hess_lstsq_kernel");
}

extern "C" int sqb_csr_spmv(sqb_ctx* ctx, int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
                            const double* data, const void* x, const double* bsub, void* y) {
  // no status clear: a matvec may run inside a caller's Arnoldi callback
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 16 * 148));
  switch (dtype) {
    case SQB_F64: csr_spmv_kernel<double><<<grid, 256, 0, ctx->stream>>>(n, indptr, indices, data, (const double*)x, bsub, (double*)y, nullptr, nullptr); break;
    case SQB_F32: csr_spmv_kernel<float><<<grid, 256, 0, ctx->stream>>>(n, indptr, indices, data, (const float*)x, bsub, (float*)y, nullptr, nullptr); break;
    case SQB_F16: csr_spmv_kernel<__half><<<grid, 256, 0, ctx->stream>>>(n, indptr, indices, data, (const __half*)x, bsub, (__half*)y, nullptr, nullptr); break;
    case SQB_BF16: csr_spmv_kernel<__nv_bfloat16><<<grid, 256, 0, ctx->stream>>>(n, indptr, indices, data, (const __nv_bfloat16*)x, bsub, (__nv_bfloat16*)y, nullptr, nullptr); break;
    default: return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", dtype);
  }
  return check_launch(ctx, "csr_spmv_kernel");
}

// Row-partitioned RHQR-Arnoldi, one process per GPU (NCCL communicator from
// sqb_ctx_init_comm).  This rank's rows: `rows` consecutive global rows
// starting at row0 (rank 0: the m+1 identity rows and its Omega rows; rank p:
// the Omega coordinates [p n_pad/P, ...)).  CSR: the local rows with column
// indices remapped to the gathered layout [rank][seg] (global row g of rank
// q at q*seg + (g - row0_q)).  Utop: (m+1) x (m+1) scratch on ranks > 0.
extern "C" int sqb_rhqr_arnoldi_dist(sqb_ctx* ctx, const sqb_sketch* sk, int m, int scaling, int lo_dtype,
                                     double happy_tol, int64_t rows, int64_t row0, int64_t seg,
                                     const int64_t* indptr, const int32_t* indices, const double* data,
                                     const double* b, const void* x0lo, void* U, int64_t ldu, double* S,
                                     int64_t lds, double* T, int64_t ldt, double* H, int64_t ldh, double* Q,
                                     int64_t ldq, double* beta, void* Utop, int* attained) {
  SQB_TRY(begin_entry(ctx));
  std::vector<ArnRank> rk(1);
  ArnRank& d = rk[0];
  d = ArnRank{};
  const int mt = m + 1;
  d.rows = rows; d.row0 = row0; d.mrow = ctx->rank == 0 ? mt : 0;
  d.e_base = ctx->rank == 0 ? 0 : row0 - mt;
  d.indptr = indptr; d.indices = indices; d.data = data; d.b = b; d.x0lo = x0lo;
  d.U = U; d.ldu = ldu; d.Q = Q; d.ldq = ldq; d.S = S; d.lds = lds; d.T = T; d.ldt = ldt; d.H = H; d.ldh = ldh;
  d.beta = beta;
  d.Utop = ctx->rank == 0 ? U : Utop;
  d.ldutop = ctx->rank == 0 ? ldu : mt;
  if (!d.Utop) return set_error(ctx, SQB_ERR_ARG, "ranks > 0 need an (m+1) x (m+1) Utop scratch");
  return arnoldi_dist_entry(ctx, sk, m, scaling, lo_dtype, happy_tol, rk, ctx->nranks, false,
                            std::vector<int>{ctx->rank}, seg, attained);
}

// Halo ranges for the row-partitioned SpMV of sqb_rhqr_arnoldi_dist /
// _virtual: table[(r P + p) 2 + {0, 1}] = [lo, hi) of rank p's segment that
// rank r's CSR rows reference.  table = NULL (or nranks = 0) clears it: the
// q exchange falls back to the all-gather.
extern "C" int sqb_ctx_set_halo(sqb_ctx* ctx, int nranks, const int64_t* table) {
  if (!ctx) return SQB_ERR_ARG;
  ctx->err[0] = 0;
  if (!table || nranks <= 0) {
    ctx->halo.clear();
    return SQB_OK;
  }
  if (nranks > 8) return set_error(ctx, SQB_ERR_ARG, "nranks must be <= 8");
  ctx->halo.assign(table, table + (size_t)nranks * nranks * 2);
  for (int r = 0; r < nranks; ++r)
    for (int p = 0; p < nranks; ++p) {
      const int64_t lo = ctx->halo[((size_t)r * nranks + p) * 2], hi = ctx->halo[((size_t)r * nranks + p) * 2 + 1];
      if (lo < 0 || hi < lo) {
        ctx->halo.clear();
        return set_error(ctx, SQB_ERR_ARG, "bad halo range [%lld, %lld) for ranks %d <- %d", (long long)lo,
                         (long long)hi, r, p);
      }
    }
  return SQB_OK;
}

// The same with P virtual ranks on one device (the all-gathers become device
// copies); per-rank arrays of length P; outputs S/T/H/beta of rank p in
// S_parts[p] etc. (every rank computes them redundantly).
extern "C" int sqb_rhqr_arnoldi_virtual(sqb_ctx* ctx, const sqb_sketch* sk, int m, int scaling, int lo_dtype,
                                        double happy_tol, int nranks, const int64_t* rows, const int64_t* row0,
                                        int64_t seg, const int64_t* const* indptr, const int32_t* const* indices,
                                        const double* const* data, const double* const* b,
                                        const void* const* x0lo, void* const* U, const int64_t* ldu,
                                        double* const* S, int64_t lds, double* const* T, int64_t ldt,
                                        double* const* H, int64_t ldh, double* const* beta,
                                        void* const* Utop, int* attained) {
  SQB_TRY(begin_entry(ctx));
  const int mt = m + 1;
  std::vector<ArnRank> rk(nranks);
  std::vector<int> ids(nranks);
  for (int r = 0; r < nranks; ++r) {
    ArnRank& d = rk[r];
    d = ArnRank{};
    ids[r] = r;
    d.rows = rows[r]; d.row0 = row0[r]; d.mrow = r == 0 ? mt : 0; d.e_base = r == 0 ? 0 : row0[r] - mt;
    d.indptr = indptr[r]; d.indices = indices[r]; d.data = data[r]; d.b = b[r]; d.x0lo = x0lo[r];
    d.U = U[r]; d.ldu = ldu[r]; d.Q = nullptr; d.ldq = 1;
    d.S = S[r]; d.lds = lds; d.T = T[r]; d.ldt = ldt; d.H = H[r]; d.ldh = ldh; d.beta = beta[r];
    d.Utop = r == 0 ? U[0] : Utop[r];
    d.ldutop = r == 0 ? ldu[0] : mt;
  }
  return arnoldi_dist_entry(ctx, sk, m, scaling, lo_dtype, happy_tol, rk, nranks, true, ids, seg, attained);
}
