// Host-side launchers for the sketch operators (shared by the factorizations).
#pragma once

#include "ctx.cuh"
#include "srht.cuh"

namespace sqb {

struct SrhtGeom {
  int log_tb;       // tile = 2^log_tb Omega coordinates (min(TileCfg::LOG_TB, log2 n_pad))
  int64_t n_tiles;  // n_pad >> log_tb
  int64_t n_eff;    // tiles that hold at least one real (non-padding) coordinate
};

inline int ilog2_exact(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

template <typename T>
inline SrhtGeom srht_geom_t(const sqb_sketch* sk) {
  SrhtGeom g;
  const int lp = ilog2_exact(sk->n_pad);
  g.log_tb = lp < TileCfg<T>::LOG_TB ? lp : TileCfg<T>::LOG_TB;
  g.n_tiles = sk->n_pad >> g.log_tb;
  const int64_t tb = int64_t(1) << g.log_tb;
  g.n_eff = (sk->n + tb - 1) / tb;
  return g;
}

SrhtGeom srht_geom(const sqb_sketch* sk, int dtype);
size_t acc_bytes(int dtype);   // sizeof(Lo<T>::acc)
size_t elem_bytes(int dtype);  // sizeof(T)

int validate_sketch(sqb_ctx* ctx, const sqb_sketch* sk);
// Arguments shared by every left-looking sweep entry (sqb_rhqr_left,
// sqb_rhqr_left_host, sqb_rhqr_block): the sketch itself, the scaling, the
// column count (1..1024) and Omega taking exactly the N-m trailing rows with
// ell >= m (rhqr.py:202-216 `_embed`).
int validate_left_args(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int64_t N, int64_t m);

// Y[y_row_off + i + col*ldy] = (Omega X)[i, col], i < ell, col < k.
// `partials` must hold sketch_partials_bytes(sk, dtype, k) bytes (SRHT only).
size_t sketch_partials_bytes(const sqb_sketch* sk, int dtype, int64_t k);
int launch_sketch(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* X, int64_t ldx,
                  int64_t k, double* Y, int64_t ldy, int64_t y_row_off, void* partials,
                  const Status* st);

// Re-sketch of ONE vector after entries [0, upto) changed, when `partials`
// still holds the leaves of its previous launch_sketch (k = 1): only the
// first tile's leaves are recomputed (every other tile's in-tile FWHT sees the
// same inputs, so its leaves are bitwise the same), then the whole tree runs.
// Falls back to a full launch_sketch when the changed range leaves tile 0 or
// the sketch is not an SRHT.
int launch_sketch_resketch_head(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* X, int64_t ldx,
                                int64_t upto, double* Y, int64_t ldy, int64_t y_row_off, void* partials,
                                const Status* st);

// tree over the group-major leaves of the standalone tile kernels, P[(col*n_tiles + t)*ell + kk]
int launch_srht_tree(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const void* P, int64_t k,
                     double* Y, int64_t ldy, int64_t y_row_off, const Status* st);

// geometry-explicit SRHT pieces for the row-partitioned (multi-GPU) path: the
// tile kernel over n_local rows whose first global Omega coordinate is e_base,
// and the tree over g.n_tiles local tiles (without the final n_pad^-1/2 when
// apply_norm == 0, i.e. the rank-local subtree).
int launch_srht_tiles_geom(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const SrhtGeom& g, int64_t n_local,
                           int64_t e_base, const void* X, int64_t ldx, int64_t k, void* P, const Status* st);
int launch_srht_tree_geom(sqb_ctx* ctx, const sqb_sketch* sk, int dtype, const SrhtGeom& g, const void* P,
                          int64_t k, double* Y, int64_t ldy, int64_t row_off, int apply_norm, const Status* st,
                          int kmajor = 0);  // leaves: 0 = standalone tiles (group-major), 1 = rhqr_col_kernel

// Y[0:m, col] = X[0:m, col] as fp64 (identity block of Psi, sketching.py:257)
int launch_copy_top(sqb_ctx* ctx, int dtype, const void* X, int64_t ldx, int64_t m, int64_t k,
                    double* Y, int64_t ldy, const Status* st);
void defer_copy_top(sqb_ctx* ctx, int dtype, const void* X, int64_t ldx, int64_t m, int64_t k, double* Y, int64_t ldy);
int flush_copy_top(sqb_ctx* ctx, const Status* st);

// host rounding of the SRHT constants to the arithmetic dtype:
// c = dtype(scale) (sketching.py:150) and dtype(n_pad^-1/2) (sketching.py:42)
void srht_constants(const sqb_sketch* sk, int dtype, double* scale_lo, double* norm_lo);

}  // namespace sqb
