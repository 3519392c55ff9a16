// Row-partitioned left-looking RHQR over P GPUs.
//
// Rank p owns the Omega coordinates [p n_pad/P, (p+1) n_pad/P) — whole SRHT
// tiles — plus, on rank 0, the m identity-block rows.  Per column the only
// exchange is the (ell + m)-vector of rank-local partials: each rank finishes
// the SRHT tree over its own tiles (levels below log2(tiles per rank)), the
// vectors are all-gathered (NCCL over NVLink), and every rank completes the top
// log2(P) tree levels in rank order (lower rank = left operand) inside the
// step kernel — the same binary tree as on one GPU, so y, and with it S, T, R
// and the coefficients, are bitwise identical to the single-GPU factorization
// (and to the reference's Psi).  Every rank then runs the sketch-space step
// redundantly; U and W never move.
//
// The exchange is either NCCL (one process per GPU, sqb_ctx_init_comm) or, for
// testing on a single GPU, "virtual ranks": all ranks' row blocks on one device,
// the all-gather a set of device copies.
#include <vector>

#include "dist_common.cuh"
#include "rhqr_kernels.cuh"

namespace sqb {

struct DistRank {
  const void* W; int64_t ldw;
  void* U; int64_t ldu;
  int64_t n_local;  // Omega rows held
  int mrow;         // m on rank 0, else 0
  int64_t e_base;   // first global Omega coordinate
  double *S, *T, *R, *sig, *rho, *bet;
  int64_t lds, ldt, ldr;
  void* Utop; int64_t ldutop;  // where the step kernel writes the identity-block rows of u
  // workspace
  double *y, *coef, *abuf, *vbuf, *fs, *pay, *Y0pay;
  void* P;
};

// Y0 (od x m) = the rank-order combine of every rank's raw-sketch partials:
// from the gather buffer, or (p2p) from this process's first mailbox once
// the peers' release flags of exchange xseq are acquired
template <typename T>
static int combine_gathered(sqb_ctx* ctx, bool p2p, const double* G0, int nranks, int64_t ell, int64_t m,
                            int rank_level, const int64_t* idx, int log_tb, double norm_lo, double* Y0, int64_t od,
                            unsigned long long xseq) {
  dim3 grid((unsigned)((od + 255) / 256), (unsigned)m);
  const int par = (int)(xseq & 1);
  void* mb = p2p ? ctx->p2p_local[0] : nullptr;
  rank_combine_kernel<T><<<grid, 256, 0, ctx->stream>>>(
      p2p ? p2p_slot(mb, nranks, ctx->p2p_count, par, 0) : G0, nranks, (int)ell, (int)m, (int)m, rank_level, idx,
      log_tb, norm_lo, Y0, od, ctx->d_status, p2p ? ctx->p2p_count : -1,
      p2p ? reinterpret_cast<const unsigned long long*>(mb) : nullptr, par, xseq);
  return check_launch(ctx, "rank_combine_kernel");
}

template <typename T>
static int rhqr_dist_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int64_t m, std::vector<DistRank>& rk,
                       int nranks, bool virt, const std::vector<int>& rank_ids) {
  using A = typename Lo<T>::acc;
  const int64_t ell = sk->ell, od = m + ell;
  const SrhtGeom g = srht_geom_t<T>(sk);
  if (g.n_tiles % nranks != 0)
    return set_error(ctx, SQB_ERR_ARG, "n_pad=%lld too small for %d ranks (need n_pad/P >= %d)",
                     (long long)sk->n_pad, nranks, 1 << g.log_tb);
  const int64_t tpr = g.n_tiles / nranks;  // tiles per rank
  int rank_level = 0;
  while ((int64_t(1) << rank_level) < tpr) ++rank_level;
  const int64_t tb = int64_t(1) << g.log_tb;
  const size_t esz = sizeof(T);
  const int L = (int)rk.size();
  // workspace: per local rank + shared gather buffers
  WsPlan plan;
  std::vector<size_t> off(L * 8);
  for (int r = 0; r < L; ++r) {
    off[r * 8 + 0] = plan.add(sizeof(double) * od);            // y
    off[r * 8 + 1] = plan.add(sizeof(double) * (m + 1));       // coef (clast)
    off[r * 8 + 2] = plan.add(sizeof(double) * 2 * (m + 1));   // abuf
    off[r * 8 + 3] = plan.add(sizeof(double) * (m + 1));       // vbuf
    off[r * 8 + 4] = plan.add(sizeof(double) * 2);             // fs
    off[r * 8 + 5] = plan.add(sizeof(double) * od);            // payload (ell partials + m top)
    off[r * 8 + 6] = plan.add(sizeof(double) * m * od);        // raw-sketch payload
    off[r * 8 + 7] = plan.add(sizeof(A) * ell * tpr * m);      // leaves
  }
  int64_t nl_max = 0;
  for (auto& d : rk) nl_max = std::max(nl_max, d.n_local);
  const size_t flag_bytes = sizeof(int) * (size_t)((nl_max >> 9) + 8);
  const size_t iFlag = plan.add(flag_bytes);                       // column-pass block flags (fused exchange)
  const size_t iG = plan.add(sizeof(double) * nranks * od);        // per-column gather
  const size_t iG0 = plan.add(sizeof(double) * nranks * m * od);   // raw-sketch gather
  const size_t iY0 = plan.add(sizeof(double) * od * m);            // combined raw sketches (shared)
  SQB_TRY(ws_reserve(ctx, plan.total));
  char* base = static_cast<char*>(ctx->ws);
  for (int r = 0; r < L; ++r) {
    DistRank& d = rk[r];
    d.y = (double*)(base + plan.offs[off[r * 8 + 0]]);
    d.coef = (double*)(base + plan.offs[off[r * 8 + 1]]);
    d.abuf = (double*)(base + plan.offs[off[r * 8 + 2]]);
    d.vbuf = (double*)(base + plan.offs[off[r * 8 + 3]]);
    d.fs = (double*)(base + plan.offs[off[r * 8 + 4]]);
    d.pay = (double*)(base + plan.offs[off[r * 8 + 5]]);
    d.Y0pay = (double*)(base + plan.offs[off[r * 8 + 6]]);
    d.P = base + plan.offs[off[r * 8 + 7]];
  }
  double* Gc = (double*)(base + plan.offs[iG]);
  double* G0 = (double*)(base + plan.offs[iG0]);
  double* Y0 = (double*)(base + plan.offs[iY0]);
  Status* st = ctx->d_status;
  const bool p2p_ready = ctx->p2p_on && ctx->p2p_nranks == nranks && (int)ctx->p2p_local.size() == L &&
                         ctx->p2p_count >= m * od;
  NcclApi* nc = (virt || p2p_ready) ? nullptr : nccl_api();
  if (!virt && !p2p_ready && (!nc || !ctx->nccl))
    return set_error(ctx, SQB_ERR_NCCL, "no exchange: neither an NCCL communicator nor peer mailboxes (sqb_p2p_open)");

  // peer-memory exchange (sqb_p2p_*): every payload fits a mailbox slot
  const bool p2p = ctx->p2p_on && ctx->p2p_nranks == nranks && ctx->p2p_count >= (int64_t)m * od &&
                   (int)ctx->p2p_local.size() == L;
  unsigned long long xseq = 0;  // sequence number of the last exchange (p2p)
  // all-gather `count` doubles from every rank's send buffer into G ([rank][count]);
  // p2p: store them into every peer's mailbox instead (the consumer acquires)
  auto exchange = [&](double* (*sendp)(DistRank&), size_t count, double* G) -> int {
    if (p2p) {
      xseq = ++ctx->p2p_seq;
      for (int r = 0; r < L; ++r) SQB_TRY(p2p_push(ctx, sendp(rk[r]), (int64_t)count, r, rank_ids[r], xseq));
      return SQB_OK;
    }
    if (virt) {
      for (int r = 0; r < L; ++r)
        SQB_CUDA_TRY(cudaMemcpyAsync(G + (size_t)rank_ids[r] * count, sendp(rk[r]), sizeof(double) * count,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
      return SQB_OK;
    }
    ncclResult_t e = nc->allGather(sendp(rk[0]), G, count, ncclDouble, (ncclComm_t)ctx->nccl, ctx->stream);
    if (e != ncclSuccess)
      return set_error(ctx, SQB_ERR_NCCL, "ncclAllGather: %s", nc->getErrorString ? nc->getErrorString(e) : "?");
    return SQB_OK;
  };

  double scale_lo = 0.0, norm_lo = 0.0;
  srht_constants(sk, Lo<T>::code, &scale_lo, &norm_lo);
  // ---- raw sketches: rank-local subtrees, one all-gather, rank-level combine
  for (int r = 0; r < L; ++r) {
    DistRank& d = rk[r];
    SQB_CUDA_TRY(cudaMemsetAsync(d.T, 0, sizeof(double) * d.ldt * m, ctx->stream));
    SrhtGeom gl{g.log_tb, tpr, (d.n_local + tb - 1) / tb};
    const char* wo = (const char*)d.W + d.mrow * esz;
    if (d.n_local > 0) {
      SQB_TRY(launch_srht_tiles_geom(ctx, sk, Lo<T>::code, gl, d.n_local, d.e_base, wo, d.ldw, m, d.P, st));
    } else {
      SQB_CUDA_TRY(cudaMemsetAsync(d.P, 0, sizeof(A) * ell * tpr * m, ctx->stream));
    }
    SQB_TRY(launch_srht_tree_geom(ctx, sk, Lo<T>::code, gl, d.P, m, d.Y0pay, od, 0, 0, st));
    if (d.mrow > 0) SQB_TRY(launch_copy_top(ctx, Lo<T>::code, d.W, d.ldw, m, m, d.Y0pay + ell, od, st));
  }
  SQB_TRY(exchange([](DistRank& d) { return d.Y0pay; }, (size_t)m * od, G0));
  // every local rank combines from its own mailbox (p2p) or the shared gather buffer
  SQB_TRY(combine_gathered<T>(ctx, p2p, G0, nranks, ell, m, rank_level, sk->indices, g.log_tb, norm_lo, Y0, od,
                              xseq));
  const size_t step_smem = step_smem_bytes((int)od, (int)m);
  allow_dyn_smem(rhqr_step_kernel<T>, (size_t)(std::max<size_t>(step_smem, 48 * 1024)));
  // real ranks over peer memory: the step kernel itself folds the rank-local
  // subtree, stores it into the peers' mailboxes and waits for theirs (tree =
  // 3): two launches per column, as on one GPU.  Virtual ranks share one
  // stream, where a rank's step cannot wait for ranks that have not run yet:
  // they keep the separate subtree + push launches.
  static const bool no_fuse = [] { const char* e = getenv("SQB_P2P_NOFUSE"); return e && e[0] == '1'; }();
  const bool fused = p2p && !virt && L == 1 && !no_fuse;
  // with the exchange inside the step the chain is the single-GPU one (pass,
  // step), so the cross-pass overlap applies unchanged (ColArgs::tflag)
  int* tflag = (fused && early_env() && rk[0].n_local >= (int64_t(1) << 19))
                   ? reinterpret_cast<int*>(base + plan.offs[iFlag]) : nullptr;
  if (tflag) SQB_CUDA_TRY(cudaMemsetAsync(tflag, 0, flag_bytes, ctx->stream));
  auto step_args = [&](DistRank& d, int c) {
    StepArgs sa{};
    sa.c = c; sa.m = (int)m; sa.off = 0; sa.ncol = (int)m; sa.ell = (int)ell; sa.od = (int)od; sa.scaling = scaling;
    sa.tree = c == 0 ? 0 : 2;
    sa.gath = Gc; sa.gstride = od; sa.flags = nullptr; sa.seq = 0;
    if (p2p) {  // this rank's own mailbox: the peers stored their partials into it
      void* mb = ctx->p2p_local[&d - rk.data()];
      sa.gath = p2p_slot(mb, nranks, ctx->p2p_count, (int)(xseq & 1), 0);
      sa.gstride = ctx->p2p_count;
      sa.flags = reinterpret_cast<const unsigned long long*>(mb);
      sa.seq = xseq;
    }
    sa.nranks = nranks; sa.rank_level = rank_level;
    sa.early = tflag ? 1 : 0;
    sa.P = nullptr; sa.n_tiles = tpr; sa.n_eff = 0; sa.idx = sk->indices; sa.log_tb = g.log_tb; sa.norm_lo = norm_lo;
    if (fused && c > 0) {
      sa.tree = 3;
      sa.P = d.P; sa.n_eff = (d.n_local + tb - 1) / tb;
      sa.peers = ctx->p2p_table + (size_t)(&d - rk.data()) * nranks;
      sa.my_rank = rank_ids[&d - rk.data()];
      sa.slot_count = ctx->p2p_count;
      sa.toprows = d.mrow > 0 ? d.pay + ell : nullptr;
    }
    sa.y = c == 0 ? Y0 : d.y; sa.Y0 = Y0; sa.S = d.S; sa.lds = d.lds; sa.R = d.R; sa.ldr = d.ldr;
    sa.U = d.Utop; sa.ldu = d.ldutop; sa.sigmas = d.sig; sa.rhos = d.rho; sa.betas = d.bet;
    sa.fscale = d.fs; sa.vbuf = d.vbuf; sa.anext = d.abuf + ((c + 1) & 1) * (m + 1); sa.clast = d.coef;
    sa.st = st;
    return sa;
  };
  for (int r = 0; r < L; ++r)
    SQB_TRY(launch_pdl(ctx, "rhqr_step_kernel", rhqr_step_kernel<T>, dim3(STEP_CL), dim3(STEP_NT), step_smem,
                       step_args(rk[r], 0)));
  // ---- column loop
  constexpr int VN = VecN<T>::n;
  const size_t tile_bytes = tile_smem_bytes<A>(1 << TileCfg<T>::LOG_TB);
  const size_t col_smem_max = sizeof(A) * ((m + 3) & ~3) + std::max(tile_bytes, sizeof(double) * (size_t)(m + 1));
  allow_dyn_smem(col_kernel_select<T, VN>(true), (size_t)(col_smem_max));
  allow_dyn_smem(col_kernel_select<T, VN>(false), (size_t)(col_smem_max));
  for (int64_t c = 1; c < m; ++c) {
    for (int r = 0; r < L; ++r) {
      DistRank& d = rk[r];
      const int64_t n_eff = (d.n_local + tb - 1) / tb;
      ColArgs ca{};
      ca.c = (int)c; ca.m = (int)m; ca.ncol = (int)m; ca.mrow = d.mrow; ca.e_base = d.e_base; ca.n = d.n_local; ca.ell = (int)ell;
      ca.od = (int)od; ca.log_tb = g.log_tb; ca.n_tiles = tpr; ca.n_eff = n_eff;
      ca.W = d.W; ca.ldw = d.ldw; ca.U = d.U; ca.ldu = d.ldu; ca.acur = d.abuf + (c & 1) * (m + 1);
      ca.clast = d.coef; ca.fscale = d.fs; ca.scaling = scaling; ca.srht = 1; ca.bits = sk->sign_bits;
      ca.idx = sk->indices; ca.scale_lo = scale_lo; ca.P = d.P; ca.y = d.pay + ell;
      ca.S = d.S; ca.lds = d.lds; ca.T = d.T; ca.ldt = d.ldt; ca.Y0 = Y0; ca.vprev = d.vbuf; ca.betas = d.bet;
      ca.anext = d.abuf + ((c + 1) & 1) * (m + 1); ca.st = st;
      ca.tflag = tflag;
      ca.no_part = no_part_env();
      ca.helper_first = helper_first_default();
      ca.no_p16 = no_p16_env();
      ca.no_pre = no_pre_env();
      const bool vec = ((reinterpret_cast<uintptr_t>((const char*)d.W + d.mrow * esz) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>((const char*)d.U + d.mrow * esz) & 15) == 0) &&
                       (d.ldw % VN == 0) && (d.ldu % VN == 0);
      const size_t smem = sizeof(A) * ((c + 3) & ~3) + std::max(tile_bytes, sizeof(double) * (size_t)(c + 1));
      SQB_TRY(launch_pdl(ctx, "rhqr_col_kernel", col_kernel_select<T, VN>(vec), dim3((unsigned)(n_eff + 2)),
                         dim3(COL_NT), smem, ca));
      // rank-local subtree of w_c's sketch -> payload[0:ell]
      SrhtGeom gl{g.log_tb, tpr, n_eff};
      if (n_eff == 0) SQB_CUDA_TRY(cudaMemsetAsync(d.P, 0, sizeof(A) * ell * tpr, ctx->stream));
      if (!fused)
        SQB_TRY(launch_srht_tree_geom(ctx, sk, Lo<T>::code, gl, d.P, 1, d.pay, od, 0, 0, st, 1));  // column-kernel leaves
    }
    if (fused) xseq = ++ctx->p2p_seq;  // the step kernel is the exchange
    else SQB_TRY(exchange([](DistRank& d) { return d.pay; }, (size_t)od, Gc));
    for (int r = 0; r < L; ++r)
      SQB_TRY(launch_pdl(ctx, "rhqr_step_kernel", rhqr_step_kernel<T>, dim3(STEP_CL), dim3(STEP_NT), step_smem,
                         step_args(rk[r], (int)c)));
  }
  for (int r = 0; r < L; ++r) {
    DistRank& d = rk[r];
    const T* src = m == 1 ? (const T*)d.W + d.mrow : (const T*)d.U + (m - 1) * d.ldu + d.mrow;
    T* dst = (T*)d.U + (m - 1) * d.ldu + d.mrow;
    const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((d.n_local + 255) / 256, 4 * 148));
    SQB_TRY(launch_pdl(ctx, "finish_kernel", finish_kernel<T>, dim3(gb + 1), dim3(256), 0, src, dst, d.n_local,
                       (const double*)d.fs, scaling, d.T, d.ldt, (int)m, (const double*)d.vbuf, (const double*)d.bet,
                       (const Status*)st));
  }
  return SQB_OK;
}

// ---------------------------------------------------------------------------
// Row-partitioned recRHQR (rhqr.py:368-395): the rank-local
// SRHT subtrees of Psi W, ONE all-gather of the (ell+m) x m partials, the
// rank-order combine (the same binary tree as one GPU, so Z is bitwise the
// single-GPU sketch), then every rank runs the sketch-space QR and Mfac
// redundantly and solves its own rows U2 = W2 Mfac^{-1}; rank 0 also writes
// the identity-block rows U[:m] = S[:m].
// ---------------------------------------------------------------------------
template <typename T>
int rec_finish_t(sqb_ctx* ctx, int scaling, const double* Z, int64_t od, int64_t m, const T* W2, int64_t n2,
                 int64_t ldw, T* U2, int64_t ldu, T* Utop, int64_t ldutop, double* S, int64_t lds, double* Tm,
                 int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* M,
                 double* X);

template <typename T>
static int rec_dist_t(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int64_t m, std::vector<DistRank>& rk,
                      int nranks, bool virt, const std::vector<int>& rank_ids) {
  using A = typename Lo<T>::acc;
  const int64_t ell = sk->ell, od = m + ell;
  const SrhtGeom g = srht_geom_t<T>(sk);
  if (g.n_tiles % nranks != 0)
    return set_error(ctx, SQB_ERR_ARG, "n_pad=%lld too small for %d ranks (need n_pad/P >= %d)",
                     (long long)sk->n_pad, nranks, 1 << g.log_tb);
  const int64_t tpr = g.n_tiles / nranks;
  int rank_level = 0;
  while ((int64_t(1) << rank_level) < tpr) ++rank_level;
  const int64_t tb = int64_t(1) << g.log_tb;
  const size_t esz = sizeof(T);
  const int L = (int)rk.size();
  int64_t nmax = 0;
  for (auto& d : rk) nmax = std::max(nmax, d.n_local);
  WsPlan plan;
  std::vector<size_t> off(L * 2);
  for (int r = 0; r < L; ++r) {
    off[r * 2 + 0] = plan.add(sizeof(double) * m * od);    // partial payload
    off[r * 2 + 1] = plan.add(sizeof(A) * ell * tpr * m);  // leaves
  }
  const size_t iG0 = plan.add(sizeof(double) * nranks * m * od);
  const size_t iZ = plan.add(sizeof(double) * od * m);
  const size_t iM = plan.add(sizeof(double) * m * m);
  const size_t iX = plan.add(m > 64 ? sizeof(double) * nmax * m : 8);
  SQB_TRY(ws_reserve(ctx, plan.total));
  char* base = static_cast<char*>(ctx->ws);
  for (int r = 0; r < L; ++r) {
    rk[r].Y0pay = (double*)(base + plan.offs[off[r * 2 + 0]]);
    rk[r].P = base + plan.offs[off[r * 2 + 1]];
  }
  double* G0 = (double*)(base + plan.offs[iG0]);
  double* Z = (double*)(base + plan.offs[iZ]);
  Status* st = ctx->d_status;
  const bool p2p_ready = ctx->p2p_on && ctx->p2p_nranks == nranks && (int)ctx->p2p_local.size() == L &&
                         ctx->p2p_count >= m * od;
  NcclApi* nc = (virt || p2p_ready) ? nullptr : nccl_api();
  if (!virt && !p2p_ready && (!nc || !ctx->nccl))
    return set_error(ctx, SQB_ERR_NCCL, "no exchange: neither an NCCL communicator nor peer mailboxes (sqb_p2p_open)");
  double scale_lo = 0.0, norm_lo = 0.0;
  srht_constants(sk, Lo<T>::code, &scale_lo, &norm_lo);
  for (int r = 0; r < L; ++r) {
    DistRank& d = rk[r];
    SrhtGeom gl{g.log_tb, tpr, (d.n_local + tb - 1) / tb};
    if (d.n_local > 0) {
      SQB_TRY(launch_srht_tiles_geom(ctx, sk, Lo<T>::code, gl, d.n_local, d.e_base,
                                     (const char*)d.W + d.mrow * esz, d.ldw, m, d.P, st));
    } else {
      SQB_CUDA_TRY(cudaMemsetAsync(d.P, 0, sizeof(A) * ell * tpr * m, ctx->stream));
    }
    SQB_TRY(launch_srht_tree_geom(ctx, sk, Lo<T>::code, gl, d.P, m, d.Y0pay, od, 0, 0, st));
    if (d.mrow > 0) SQB_TRY(launch_copy_top(ctx, Lo<T>::code, d.W, d.ldw, m, m, d.Y0pay + ell, od, st));
  }
  const size_t count = (size_t)m * od;
  const bool p2p = ctx->p2p_on && ctx->p2p_nranks == nranks && ctx->p2p_count >= (int64_t)count &&
                   (int)ctx->p2p_local.size() == L;
  unsigned long long xseq = 0;
  if (p2p) {
    xseq = ++ctx->p2p_seq;
    for (int r = 0; r < L; ++r) SQB_TRY(p2p_push(ctx, rk[r].Y0pay, (int64_t)count, r, rank_ids[r], xseq));
  } else if (virt) {
    for (int r = 0; r < L; ++r)
      SQB_CUDA_TRY(cudaMemcpyAsync(G0 + (size_t)rank_ids[r] * count, rk[r].Y0pay, sizeof(double) * count,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    ncclResult_t e = nc->allGather(rk[0].Y0pay, G0, count, ncclDouble, (ncclComm_t)ctx->nccl, ctx->stream);
    if (e != ncclSuccess)
      return set_error(ctx, SQB_ERR_NCCL, "ncclAllGather: %s", nc->getErrorString ? nc->getErrorString(e) : "?");
  }
  SQB_TRY(combine_gathered<T>(ctx, p2p, G0, nranks, ell, m, rank_level, sk->indices, g.log_tb, norm_lo, Z, od, xseq));
  for (int r = 0; r < L; ++r) {
    DistRank& d = rk[r];
    SQB_TRY(rec_finish_t<T>(ctx, scaling, Z, od, m, (const T*)d.W + d.mrow, d.n_local, d.ldw, (T*)d.U + d.mrow,
                            d.ldu, d.mrow > 0 ? (T*)d.U : nullptr, d.ldu, d.S, d.lds, d.T, d.ldt, d.R, d.ldr, d.sig,
                            d.rho, d.bet, (double*)(base + plan.offs[iM]), (double*)(base + plan.offs[iX])));
  }
  return SQB_OK;
}

static int rec_dist_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, int64_t m,
                             std::vector<DistRank>& rk, int nranks, bool virt, const std::vector<int>& ids) {
  switch (lo_dtype) {
    case SQB_F64: return rec_dist_t<double>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_F32: return rec_dist_t<float>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_F16: return rec_dist_t<__half>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_BF16: return rec_dist_t<__nv_bfloat16>(ctx, sk, scaling, m, rk, nranks, virt, ids);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

static int dist_dispatch(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, int64_t m,
                         std::vector<DistRank>& rk, int nranks, bool virt, const std::vector<int>& ids) {
  switch (lo_dtype) {
    case SQB_F64: return rhqr_dist_t<double>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_F32: return rhqr_dist_t<float>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_F16: return rhqr_dist_t<__half>(ctx, sk, scaling, m, rk, nranks, virt, ids);
    case SQB_BF16: return rhqr_dist_t<__nv_bfloat16>(ctx, sk, scaling, m, rk, nranks, virt, ids);
  }
  return set_error(ctx, SQB_ERR_ARG, "unknown dtype %d", lo_dtype);
}

static int check_common(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int64_t m, int nranks) {
  SQB_TRY(validate_sketch(ctx, sk));
  if (sk->kind != SQB_SKETCH_SRHT) return set_error(ctx, SQB_ERR_ARG, "the row-partitioned sweep needs an SRHT");
  if (scaling != SQB_SCALE_SQRT2 && scaling != SQB_SCALE_UNIT)
    return set_error(ctx, SQB_ERR_ARG, "unknown scaling %d", scaling);
  if (m < 1 || m > 1024) return set_error(ctx, SQB_ERR_ARG, "need 1 <= m <= 1024");
  if (sk->ell < m) return set_error(ctx, SQB_ERR_ARG, "sampling size below column count");
  if (nranks < 1 || nranks > 8 || (nranks & (nranks - 1)))
    return set_error(ctx, SQB_ERR_ARG, "nranks must be a power of two <= 8");
  return SQB_OK;
}

}  // namespace sqb

using namespace sqb;

// ---- peer-memory exchange setup ------------------------------------------------
static int p2p_release(sqb_ctx* ctx) {
  for (void* p : ctx->p2p_opened) cudaIpcCloseMemHandle(p);
  for (void* p : ctx->p2p_local) cudaFree(p);
  for (void* p : ctx->p2p_absent) cudaFree(p);
  ctx->p2p_absent.clear();
  if (ctx->p2p_table) cudaFree(ctx->p2p_table);
  ctx->p2p_opened.clear();
  ctx->p2p_local.clear();
  ctx->p2p_table = nullptr;
  if (ctx->p2p_on && !ctx->nccl) {  // the partition sqb_p2p_open set goes with the mailboxes
    ctx->nranks = 1;
    ctx->rank = 0;
  }
  ctx->p2p_on = 0;
  ctx->p2p_nranks = 0;
  ctx->p2p_count = 0;
  ctx->p2p_seq = 0;  // fresh mailboxes have zero flags (every rank re-opens collectively)
  return SQB_OK;
}

static int p2p_alloc(sqb_ctx* ctx, int nranks, int64_t count, void** out) {
  const size_t bytes = p2p_mailbox_bytes(nranks, count);
  SQB_CUDA_TRY(cudaMalloc(out, bytes));
  SQB_CUDA_TRY(cudaMemset(*out, 0, p2p_flag_bytes(nranks)));
  return SQB_OK;
}

static int p2p_set_table(sqb_ctx* ctx, const std::vector<void*>& table) {
  SQB_CUDA_TRY(cudaMalloc(&ctx->p2p_table, sizeof(void*) * table.size()));
  SQB_CUDA_TRY(cudaMemcpy(ctx->p2p_table, table.data(), sizeof(void*) * table.size(), cudaMemcpyHostToDevice));
  return SQB_OK;
}


extern "C" {

int sqb_nccl_unique_id(char* out, int size) {
  NcclApi* nc = nccl_api();
  if (!nc || size < (int)sizeof(ncclUniqueId)) return SQB_ERR_NCCL;
  ncclUniqueId id;
  if (nc->getUniqueId(&id) != ncclSuccess) return SQB_ERR_NCCL;
  memcpy(out, &id, sizeof(id));
  return SQB_OK;
}

int sqb_p2p_mailbox(sqb_ctx* ctx, int nranks, int64_t count, void* handle_out) {
  if (!ctx || !handle_out || nranks < 1 || nranks > 8 || count < 1) return SQB_ERR_ARG;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  SQB_CUDA_TRY(cudaDeviceSynchronize());
  p2p_release(ctx);
  void* mb = nullptr;
  SQB_TRY(p2p_alloc(ctx, nranks, count, &mb));
  ctx->p2p_local.push_back(mb);
  ctx->p2p_nranks = nranks;
  ctx->p2p_count = count;
  cudaIpcMemHandle_t h;
  SQB_CUDA_TRY(cudaIpcGetMemHandle(&h, mb));
  memcpy(handle_out, &h, sizeof(h));
  return SQB_OK;
}

int sqb_p2p_open(sqb_ctx* ctx, int rank, const void* handles) {
  if (!ctx || !handles || ctx->p2p_local.size() != 1) return SQB_ERR_ARG;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  const int P = ctx->p2p_nranks;
  if (rank < 0 || rank >= P) return set_error(ctx, SQB_ERR_ARG, "rank %d outside %d", rank, P);
  std::vector<void*> table(P);
  for (int q = 0; q < P; ++q) {
    if (q == rank) {
      table[q] = ctx->p2p_local[0];
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, static_cast<const char*>(handles) + (size_t)q * sizeof(h), sizeof(h));
    bool absent = true;  // an all-zero handle: a peer that never answers (fault injection, tests)
    for (size_t b = 0; b < sizeof(h); ++b) absent = absent && reinterpret_cast<const char*>(&h)[b] == 0;
    void* p = nullptr;
    if (absent) {
      SQB_TRY(p2p_alloc(ctx, P, ctx->p2p_count, &p));
      ctx->p2p_absent.push_back(p);  // freed with the mailboxes
    } else {
      SQB_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      ctx->p2p_opened.push_back(p);
    }
    table[q] = p;
  }
  SQB_TRY(p2p_set_table(ctx, table));
  ctx->p2p_on = 1;
  ctx->nranks = P;  // the row partition of the *_dist entries (as sqb_ctx_init_comm sets it)
  ctx->rank = rank;
  return SQB_OK;
}

int sqb_p2p_virtual(sqb_ctx* ctx, int nranks, int64_t count) {
  if (!ctx || nranks < 1 || nranks > 8 || count < 1) return SQB_ERR_ARG;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  SQB_CUDA_TRY(cudaDeviceSynchronize());
  p2p_release(ctx);
  for (int q = 0; q < nranks; ++q) {
    void* mb = nullptr;
    SQB_TRY(p2p_alloc(ctx, nranks, count, &mb));
    ctx->p2p_local.push_back(mb);
  }
  std::vector<void*> table((size_t)nranks * nranks);
  for (int r = 0; r < nranks; ++r)
    for (int q = 0; q < nranks; ++q) table[(size_t)r * nranks + q] = ctx->p2p_local[q];
  ctx->p2p_nranks = nranks;
  ctx->p2p_count = count;
  SQB_TRY(p2p_set_table(ctx, table));
  ctx->p2p_on = 1;
  return SQB_OK;
}

int sqb_p2p_set_timeout_ms(sqb_ctx* ctx, int64_t ms) {
  if (!ctx || ms < 0 || ctx->p2p_local.empty()) return SQB_ERR_ARG;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  const unsigned long long ns = (unsigned long long)ms * 1000000ull;
  for (void* mb : ctx->p2p_local)
    SQB_CUDA_TRY(cudaMemcpy(reinterpret_cast<unsigned long long*>(mb) + 2 * ctx->p2p_nranks, &ns, sizeof(ns),
                            cudaMemcpyHostToDevice));
  return SQB_OK;
}

int sqb_p2p_close(sqb_ctx* ctx) {
  if (!ctx) return SQB_ERR_ARG;
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  SQB_CUDA_TRY(cudaDeviceSynchronize());
  return p2p_release(ctx);
}

int sqb_ctx_init_comm(sqb_ctx* ctx, const char* id, int nranks, int rank) {
  if (!ctx) return SQB_ERR_ARG;
  NcclApi* nc = nccl_api();
  if (!nc) return set_error(ctx, SQB_ERR_NCCL, "libnccl.so.2 not found");
  SQB_CUDA_TRY(cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  ncclResult_t e = nc->commInitRank(&comm, nranks, uid, rank);
  if (e != ncclSuccess) return set_error(ctx, SQB_ERR_NCCL, "ncclCommInitRank: %s", nc->getErrorString(e));
  ctx->nccl = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return SQB_OK;
}

static int left_dist_entry(bool rec, sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                       int64_t n_local, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                       double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                       double* betas, void* Utop_scratch) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_common(ctx, sk, scaling, m, ctx->nranks));
  const int64_t span = sk->n_pad / ctx->nranks;
  const int64_t e_base = span * ctx->rank;
  const int64_t want = std::max<int64_t>(0, std::min<int64_t>(span, sk->n - e_base));
  if (n_local != want)
    return set_error(ctx, SQB_ERR_ARG, "rank %d holds %lld Omega rows, expected %lld", ctx->rank,
                     (long long)n_local, (long long)want);
  std::vector<DistRank> rk(1);
  DistRank& d = rk[0];
  d.W = W; d.ldw = ldw; d.U = U; d.ldu = ldu; d.n_local = n_local; d.mrow = ctx->rank == 0 ? (int)m : 0;
  d.e_base = e_base; d.S = S; d.T = T; d.R = R; d.sig = sigmas; d.rho = rhos; d.bet = betas;
  d.lds = lds; d.ldt = ldt; d.ldr = ldr;
  d.Utop = ctx->rank == 0 ? U : Utop_scratch;
  d.ldutop = ctx->rank == 0 ? ldu : m;
  if (!d.Utop && !rec) return set_error(ctx, SQB_ERR_ARG, "ranks > 0 need an m x m Utop_scratch buffer");
  return rec ? rec_dist_dispatch(ctx, sk, scaling, lo_dtype, m, rk, ctx->nranks, false, std::vector<int>{ctx->rank})
             : dist_dispatch(ctx, sk, scaling, lo_dtype, m, rk, ctx->nranks, false, std::vector<int>{ctx->rank});
}

static int left_virtual_entry(bool rec, sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, int nranks,
                          const void* const* W_parts, const int64_t* ldw, void* const* U_parts,
                          const int64_t* ldu, int64_t m, double* S, int64_t lds, double* T, int64_t ldt,
                          double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* scratch) {
  SQB_TRY(begin_entry(ctx));
  SQB_TRY(check_common(ctx, sk, scaling, m, nranks));
  const int64_t span = sk->n_pad / nranks;
  const int64_t od = m + sk->ell;
  // scratch for ranks > 0: S, T, R, 3m scalars, m x m Utop  (per rank)
  const int64_t per = od * m + 2 * m * m + 3 * m + m * m;
  std::vector<DistRank> rk(nranks);
  std::vector<int> ids(nranks);
  for (int r = 0; r < nranks; ++r) {
    DistRank& d = rk[r];
    ids[r] = r;
    d.W = W_parts[r]; d.ldw = ldw[r]; d.U = U_parts[r]; d.ldu = ldu[r];
    d.e_base = span * r;
    d.n_local = std::max<int64_t>(0, std::min<int64_t>(span, sk->n - d.e_base));
    d.mrow = r == 0 ? (int)m : 0;
    if (r == 0) {
      d.S = S; d.T = T; d.R = R; d.sig = sigmas; d.rho = rhos; d.bet = betas;
      d.lds = lds; d.ldt = ldt; d.ldr = ldr; d.Utop = U_parts[0]; d.ldutop = ldu[0];
    } else {
      double* b = scratch + (r - 1) * per;
      d.S = b; d.lds = od; d.T = b + od * m; d.ldt = m; d.R = d.T + m * m; d.ldr = m;
      d.sig = d.R + m * m; d.rho = d.sig + m; d.bet = d.rho + m; d.Utop = d.bet + m; d.ldutop = m;
    }
  }
  // rank r > 0 writes its identity-block u rows as T; the scratch is double, large enough for any T
  return rec ? rec_dist_dispatch(ctx, sk, scaling, lo_dtype, m, rk, nranks, true, ids)
             : dist_dispatch(ctx, sk, scaling, lo_dtype, m, rk, nranks, true, ids);
}

int sqb_rhqr_left_dist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                       int64_t n_local, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                       double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                       double* betas, void* Utop_scratch) {
  return left_dist_entry(false, ctx, sk, scaling, lo_dtype, W, n_local, m, ldw, U, ldu, S, lds, T, ldt, R, ldr,
                         sigmas, rhos, betas, Utop_scratch);
}

int sqb_rec_rhqr_dist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, const void* W,
                      int64_t n_local, int64_t m, int64_t ldw, void* U, int64_t ldu, double* S, int64_t lds,
                      double* T, int64_t ldt, double* R, int64_t ldr, double* sigmas, double* rhos,
                      double* betas) {
  return left_dist_entry(true, ctx, sk, scaling, lo_dtype, W, n_local, m, ldw, U, ldu, S, lds, T, ldt, R, ldr,
                         sigmas, rhos, betas, nullptr);
}

int sqb_rhqr_left_virtual(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, int nranks,
                          const void* const* W_parts, const int64_t* ldw, void* const* U_parts,
                          const int64_t* ldu, int64_t m, double* S, int64_t lds, double* T, int64_t ldt,
                          double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* scratch) {
  return left_virtual_entry(false, ctx, sk, scaling, lo_dtype, nranks, W_parts, ldw, U_parts, ldu, m, S, lds, T,
                            ldt, R, ldr, sigmas, rhos, betas, scratch);
}

int sqb_rec_rhqr_virtual(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype, int nranks,
                         const void* const* W_parts, const int64_t* ldw, void* const* U_parts,
                         const int64_t* ldu, int64_t m, double* S, int64_t lds, double* T, int64_t ldt,
                         double* R, int64_t ldr, double* sigmas, double* rhos, double* betas, double* scratch) {
  return left_virtual_entry(true, ctx, sk, scaling, lo_dtype, nranks, W_parts, ldw, U_parts, ldu, m, S, lds, T,
                            ldt, R, ldr, sigmas, rhos, betas, scratch);
}

}  // extern "C"
