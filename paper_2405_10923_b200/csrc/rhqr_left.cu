// Left-looking RHQR driver, single GPU (kernels in rhqr_kernels.cuh).
#include <cstdlib>

#include "rhqr_kernels.cuh"

namespace sqb {

__global__ void zero_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * cols; e += (int64_t)gridDim.x * blockDim.x)
    p[(e % rows) + (e / rows) * ld] = 0.0;
}

static int zero2d(sqb_ctx* ctx, double* p, int64_t rows, int64_t cols, int64_t ld) {
  if (rows * cols == 0) return SQB_OK;
  const unsigned g = (unsigned)std::min<int64_t>((rows * cols + 255) / 256, 2048);
  zero_kernel<<<g, 256, 0, ctx->stream>>>(p, rows, cols, ld);
  return check_launch(ctx, "zero_kernel");
}

// persistent single-kernel sweep for small fp64 problems (rhqr_persist.cu)
size_t persist_ws_bytes(const sqb_sketch* sk, int64_t m);
bool persist_eligible(sqb_ctx* ctx, const sqb_sketch* sk, int64_t N, int64_t m, int64_t ncol, int64_t off);
int launch_persist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const double* W, int64_t N, int64_t m,
                   int64_t ldw, double* U, int64_t ldu, double* S, int64_t lds, double* Tm, int64_t ldt, double* R,
                   int64_t ldr, double* sigmas, double* rhos, double* betas, const double* Y0, double* abuf,
                   double* vbuf, void* pws, double scale_lo, double norm_lo);

// workspace of one sweep
struct SweepWs {
  WsPlan plan;
  int64_t chunk;
  size_t iY0, iy, icoef, iabuf, ivbuf, ifs, iP, iPS, iflag;
};
static SweepWs sweep_ws(const sqb_sketch* sk, int code, int64_t m, int64_t ncol) {
  SweepWs w;
  const int64_t od = m + sk->ell;
  w.chunk = std::max<int64_t>(1, std::min<int64_t>(ncol, (int64_t)(64ll << 20) /
                              std::max<size_t>(1, sketch_partials_bytes(sk, code, 1))));
  w.iY0 = w.plan.add(sizeof(double) * od * ncol);
  w.iy = w.plan.add(sizeof(double) * od);
  w.icoef = w.plan.add(sizeof(double) * (m + 1));
  w.iabuf = w.plan.add(sizeof(double) * 2 * (m + 1));
  w.ivbuf = w.plan.add(sizeof(double) * (m + 1));
  w.ifs = w.plan.add(sizeof(double) * 2);
  w.iP = w.plan.add(std::max(sketch_partials_bytes(sk, code, w.chunk), sketch_partials_bytes(sk, code, 1)));
  w.iPS = w.plan.add(code == SQB_F64 ? persist_ws_bytes(sk, m) : 0);
  // per-block pass-completion flags of the column pass (tiles of >= 512 rows + identity block + helper)
  w.iflag = w.plan.add(sizeof(int) * (size_t)((std::max<int64_t>(sk->n, 1) >> 9) + 8));
  return w;
}
size_t left_sweep_ws_bytes(const sqb_sketch* sk, int code, int64_t m, int64_t ncol) {
  return sweep_ws(sk, code, m, ncol).plan.total + 256;
}

// ---------------------------------------------------------------------------
// driver: the left-looking sweep (_left_sweep, rhqr.py:219-251) over the ncol
// columns of W, eliminating column c at global index off + c + 1.  m is the
// identity-block size of Psi (the column count of the whole matrix).  U, S, R,
// sigmas, rhos and betas point at the sweep's first column; T is ncol x ncol.
// rhqr_left is the sweep with off = 0, ncol = m.
// ---------------------------------------------------------------------------
template <typename T>
int left_sweep_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, const void* W, int64_t N, int64_t m,
                 int64_t ldw, int64_t ncol, int64_t off, void* U, int64_t ldu, double* S, int64_t lds,
                 double* Tm, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                 double* betas, void* ws_base) {
  using A = typename Lo<T>::acc;
  const int64_t n = N - m, ell = sk->ell, od = m + ell;
  const bool srht = sk->kind == SQB_SKETCH_SRHT;
  const SrhtGeom g = srht ? srht_geom_t<T>(sk) : SrhtGeom{0, 1, 1};
  const SweepWs sw = sweep_ws(sk, Lo<T>::code, m, ncol);
  const int64_t chunk = sw.chunk;
  const WsPlan& plan = sw.plan;
  const size_t iY0 = sw.iY0, iy = sw.iy, icoef = sw.icoef, iabuf = sw.iabuf, ivbuf = sw.ivbuf, ifs = sw.ifs,
               iP = sw.iP;
  if (!ws_base) {
    SQB_TRY(ws_reserve(ctx, plan.total));
    ws_base = ctx->ws;
  }
  char* wb = static_cast<char*>(ws_base);
  double* Y0 = reinterpret_cast<double*>(wb + plan.offs[iY0]);
  double* y = reinterpret_cast<double*>(wb + plan.offs[iy]);
  double* coef = reinterpret_cast<double*>(wb + plan.offs[icoef]);
  double* abuf = reinterpret_cast<double*>(wb + plan.offs[iabuf]);
  double* vbuf = reinterpret_cast<double*>(wb + plan.offs[ivbuf]);
  double* fs = reinterpret_cast<double*>(wb + plan.offs[ifs]);
  void* P = wb + plan.offs[iP];
  Status* st = ctx->d_status;
  // cross-pass overlap (ColArgs::tflag): on for passes of many blocks; a small
  // sweep (config 1: 34 blocks) is a latency chain in which the extra fence +
  // flag store at every block's exit costs ~1 us per column (0.47 -> 0.50 ms)
  const int early = early_env();
  int* tflag = (early == 2 || (early == 1 && n >= (int64_t(1) << 19)))
                   ? reinterpret_cast<int*>(wb + plan.offs[sw.iflag]) : nullptr;

  SQB_TRY(zero2d(ctx, Tm, ncol, ncol, ldt));
  if (tflag)
    SQB_CUDA_TRY(cudaMemsetAsync(tflag, 0, sizeof(int) * (size_t)((std::max<int64_t>(sk->n, 1) >> 9) + 8), ctx->stream));
  // raw sketches y0 = Psi W (rhqr.py:240 for every column).  Pass c and step
  // c read y0_{c+1}; with a streamed input (host_pipe.cu) the columns arrive
  // in groups and each group is sketched as soon as it is resident.
  SweepHooks* hk = ctx->hooks;
  const bool streamed = hk && hk->streamed_input;
  const size_t esz = sizeof(T);
  int64_t y0_done = 0;
  auto ensure_y0 = [&](int64_t upto) -> int {  // y0 of columns [0, upto)
    upto = std::min(upto, ncol);
    if (upto <= y0_done) return SQB_OK;
    int64_t end = streamed ? std::min(ncol, hk->wait_cols(ctx, upto)) : ncol;
    SQB_TRY(launch_copy_top(ctx, Lo<T>::code, (const char*)W + y0_done * ldw * esz, ldw, m, end - y0_done,
                            Y0 + y0_done * od, od, st));
    for (int64_t c0 = y0_done; c0 < end; c0 += chunk) {
      const int64_t kc = std::min(chunk, end - c0);
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)W + (c0 * ldw + m) * esz, ldw, kc,
                            Y0 + c0 * od, od, m, P, st));
    }
    y0_done = end;
    return SQB_OK;
  };
  double scale_lo = 0.0, norm_lo = 0.0;
  if (srht) srht_constants(sk, Lo<T>::code, &scale_lo, &norm_lo);
  if constexpr (std::is_same<T, double>::value) {
    // small fp64 problems (config 1): one cooperative kernel runs every column
    constexpr int VN2 = VecN<T>::n;
    const bool vec2 = ((reinterpret_cast<uintptr_t>((const char*)W + m * esz) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>((const char*)U + m * esz) & 15) == 0) && (ldw % VN2 == 0) &&
                      (ldu % VN2 == 0);
    if (vec2 && persist_eligible(ctx, sk, N, m, ncol, off)) {
      SQB_TRY(ensure_y0(ncol));
      prof_begin(ctx);
      SQB_TRY(launch_persist(ctx, sk, scaling, (const double*)W, N, m, ldw, (double*)U, ldu, S, lds, Tm, ldt, R,
                             ldr, sigmas, rhos, betas, Y0, abuf, vbuf, wb + plan.offs[sw.iPS], scale_lo, norm_lo));
      // algorithmic bytes of the column passes it replaces: sum_c 8 N (c + 2)
      prof_end(ctx, 8.0 * (double)N * (double)((ncol - 1) * ncol / 2 + 2 * (ncol - 1)));
      if (hk)
        for (int64_t c = 0; c < ncol; ++c) SQB_TRY(hk->col_final(ctx, c));
      return SQB_OK;
    }
  }
  SQB_TRY(ensure_y0(2));

  const size_t step_smem = step_smem_bytes((int)od, (int)m);
  allow_dyn_smem(rhqr_step_kernel<T>, (size_t)(std::max<size_t>(step_smem, 48 * 1024)));
  // column 0: y = y0_0 (w = W[:, 0]); a_1 is empty
  StepArgs sa{};
  sa.c = 0; sa.m = (int)m; sa.ell = (int)ell; sa.od = (int)od; sa.scaling = scaling; sa.tree = 0;
  sa.off = (int)off; sa.ncol = (int)ncol;
  sa.gath = nullptr; sa.nranks = 1; sa.rank_level = 0;
  sa.P = P; sa.n_tiles = g.n_tiles; sa.n_eff = g.n_eff; sa.idx = srht ? sk->indices : nullptr;
  sa.log_tb = g.log_tb; sa.norm_lo = norm_lo; sa.y = Y0; sa.Y0 = Y0; sa.S = S; sa.lds = lds;
  sa.R = R; sa.ldr = ldr; sa.U = U; sa.ldu = ldu; sa.sigmas = sigmas; sa.rhos = rhos; sa.betas = betas;
  sa.fscale = fs; sa.vbuf = vbuf; sa.anext = abuf + (m + 1); sa.clast = coef; sa.st = st;
  sa.early = tflag ? 1 : 0;
  SQB_TRY(launch_pdl(ctx, "rhqr_step_kernel", rhqr_step_kernel<T>, dim3(STEP_CL), dim3(STEP_NT),
                     step_smem, sa));

  constexpr int VN = VecN<T>::n;
  const bool vec = ((reinterpret_cast<uintptr_t>((const char*)W + m * esz) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>((const char*)U + m * esz) & 15) == 0) &&
                   (ldw % VN == 0) && (ldu % VN == 0);
  const int tb_max = 1 << TileCfg<T>::LOG_TB;
  // small fp64 problems (config 1: 2^14 rows = 4 tiles of 4096): 512-row
  // tiles, 8x the CTAs per column pass; leaves and the step kernel's tree
  // follow the geometry
  constexpr int SMALL_LOG = 9;
  const bool small = std::is_same<T, double>::value && srht && vec && g.log_tb == TileCfg<T>::LOG_TB &&
                     sk->n_pad <= (int64_t(1) << 16) && ncol >= 8;
  SrhtGeom gc = g;
  if (small) {
    gc.log_tb = SMALL_LOG;
    gc.n_tiles = sk->n_pad >> SMALL_LOG;
    gc.n_eff = (n + (1 << SMALL_LOG) - 1) >> SMALL_LOG;
  }
  const int64_t n_eff_col = srht ? gc.n_eff : (n + tb_max - 1) / tb_max;
  const int log_tb_col = srht ? gc.log_tb : TileCfg<T>::LOG_TB;
  const size_t tile_bytes = srht ? tile_smem_bytes<A>(tb_max) : 0;
  const size_t col_smem_max = sizeof(A) * ((m + 3) & ~3) +
                              std::max(tile_bytes, sizeof(double) * (size_t)(m + 1));
  void (*colk)(ColArgs) = col_kernel_select<T, VN>(vec);
  if constexpr (std::is_same<T, double>::value) {
    if (small) colk = rhqr_col_kernel<T, VN, 0, 2, SMALL_LOG>;
  }
  allow_dyn_smem(colk, (size_t)(col_smem_max));
  for (int64_t c = 1; c < ncol; ++c) {
    SQB_TRY(ensure_y0(c + 2));
    double* a_cur = abuf + (c & 1) * (m + 1);
    double* a_nxt = abuf + ((c + 1) & 1) * (m + 1);
    ColArgs ca{};
    ca.c = (int)c; ca.m = (int)m; ca.ncol = (int)ncol; ca.mrow = (int)m; ca.e_base = 0; ca.n = n; ca.ell = (int)ell;
    ca.od = (int)od; ca.log_tb = log_tb_col; ca.n_tiles = gc.n_tiles; ca.n_eff = n_eff_col;
    ca.W = W; ca.ldw = ldw; ca.U = U; ca.ldu = ldu; ca.acur = a_cur; ca.clast = coef; ca.fscale = fs;
    ca.scaling = scaling; ca.srht = srht ? 1 : 0; ca.bits = srht ? sk->sign_bits : nullptr;
    ca.idx = srht ? sk->indices : nullptr; ca.scale_lo = scale_lo; ca.P = P; ca.y = y;
    ca.S = S; ca.lds = lds; ca.T = Tm; ca.ldt = ldt; ca.Y0 = Y0; ca.vprev = vbuf; ca.betas = betas;
    ca.anext = a_nxt; ca.st = st; ca.tflag = tflag;
    ca.dbg = (c == ctx->dbg_ccol) ? ctx->dbg_cts : nullptr;
    ca.helper_first = helper_first_default();
    ca.no_p16 = no_p16_env();
    ca.no_pre = no_pre_env();
    ca.no_part = no_part_env();
    const size_t smem = sizeof(A) * ((c + 3) & ~3) + std::max(tile_bytes, sizeof(double) * (size_t)(c + 1));
    prof_begin(ctx);
    SQB_TRY(launch_pdl(ctx, "rhqr_col_kernel", colk, dim3((unsigned)(n_eff_col + 2)), dim3(COL_NT), smem,
                       ca));
    // algorithmic bytes of this pass: read U[:, :c] and W[:, c], write U[:, c]
    prof_end(ctx, (double)esz * (double)N * (double)(c + 2));
    if (hk) SQB_TRY(hk->col_final(ctx, c - 1));  // pass c wrote the scaled U[:, c-1]
    if (!srht)
      SQB_TRY(launch_sketch(ctx, sk, Lo<T>::code, (const char*)U + (c * ldu + m) * esz, ldu, 1, y, od,
                            m, P, st));
    sa.c = (int)c;
    sa.y = y;
    sa.dbg = (c == ctx->dbg_col) ? ctx->dbg_ts : nullptr;
    sa.gdbg = (c == ctx->dbg_ccol && ctx->dbg_cts) ? ctx->dbg_cts + 8 * (n_eff_col + 2) : nullptr;
    sa.anext = a_nxt;
    sa.tree = srht ? 1 : 0;
    sa.n_tiles = gc.n_tiles; sa.n_eff = gc.n_eff; sa.log_tb = gc.log_tb;
    SQB_TRY(launch_pdl(ctx, "rhqr_step_kernel", rhqr_step_kernel<T>, dim3(STEP_CL), dim3(STEP_NT),
                       step_smem, sa));
  }
  // last column: lazy scaling of its Omega rows and its T column
  {
    const T* src = ncol == 1 ? (const T*)W + m : (const T*)U + (ncol - 1) * ldu + m;
    T* dst = (T*)U + (ncol - 1) * ldu + m;
    const unsigned gb = (unsigned)std::min<int64_t>((n + 255) / 256, 4 * 148);
    SQB_TRY(launch_pdl(ctx, "finish_kernel", finish_kernel<T>, dim3(gb + 1), dim3(256), 0, src, dst, n,
                       (const double*)fs, scaling, Tm, ldt, (int)ncol, (const double*)vbuf,
                       (const double*)betas, (const Status*)st));
  }
  if (hk) SQB_TRY(hk->col_final(ctx, ncol - 1));
  return SQB_OK;
}

#define SQB_SWEEP_INST(T)                                                                                  \
  template int left_sweep_t<T>(sqb_ctx*, const sqb_sketch*, int, const void*, int64_t, int64_t, int64_t, int64_t, \
                               int64_t, void*, int64_t, double*, int64_t, double*, int64_t, double*, int64_t,     \
                               double*, double*, double*, void*);
SQB_SWEEP_INST(double)
SQB_SWEEP_INST(float)
SQB_SWEEP_INST(__half)
SQB_SWEEP_INST(__nv_bfloat16)
#undef SQB_SWEEP_INST

int rhqr_left_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                       const void* W, int64_t N, int64_t m, int64_t ldw, void* U, int64_t ldu,
                       double* S, int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr,
                       double* sigmas, double* rhos, double* betas) {
  switch (lo_dtype) {
    case SQB_F64: return left_sweep_t<double>(ctx, sk, scaling, W, N, m, ldw, m, 0, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas, nullptr);
    case SQB_F32: return left_sweep_t<float>(ctx, sk, scaling, W, N, m, ldw, m, 0, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas, nullptr);
    case SQB_F16: return left_sweep_t<__half>(ctx, sk, scaling, W, N, m, ldw, m, 0, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas, nullptr);
    case SQB_BF16: return left_sweep_t<__nv_bfloat16>(ctx, sk, scaling, W, N, m, ldw, m, 0, U, ldu, S, lds, T, ldt, R, ldr, sigmas, rhos, betas, nullptr);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

}  // namespace sqb
