/*
 * sketchqr_b200 — C ABI of the B200-native randomized Householder QR library.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `sketchqr` (arXiv 2405.10923, /root/reference/pkg/src/sketchqr).  Every
 * entry point below names the reference function it replaces.  The Python
 * facade (paper_2405_10923_b200/) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Plain pointers and sizes; no torch types.  Device pointers are CUDA
 *    device addresses on the context's device.
 *  - n-dimensional operands (W, U, X, Q, Krylov vectors) are COLUMN-MAJOR:
 *    element (i, j) at ptr[i + j*ld].  Sketch-space operands (S, T, R, Y, H)
 *    are fp64, column-major as well.
 *  - Calls are asynchronous and ordered on the context's stream.  The
 *    library never allocates or frees caller buffers; scratch workspace is
 *    owned by the context.  A context is not thread-safe: one per device per
 *    thread.
 *  - Every call returns an sqb_status.  Numerical failures detected on the
 *    device (breakdowns, singular factors) are recorded in a device status
 *    word that makes the rest of the call chain a no-op; read it with
 *    sqb_ctx_status(), which synchronises the stream.
 */
#ifndef SKETCHQR_B200_H
#define SKETCHQR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (the facade maps them to the reference's exception types) */
enum sqb_status {
  SQB_OK = 0,
  SQB_ERR_ARG = 1,        /* ValueError (sketching.py:52, :143; rhqr.py:204-215) */
  SQB_ERR_BREAKDOWN = 2,  /* BreakdownError "... column {j} ..." (linalg.py:18, rhqr.py:73-79) */
  SQB_ERR_SINGULAR = 3,   /* SingularFactorError (linalg.py:35, :92-99) */
  SQB_ERR_CUDA = 4,
  SQB_ERR_NCCL = 5,
  SQB_ERR_RANGE = 6,      /* PrecisionRangeError (precision.py:25, :45-50) */
  SQB_ERR_NONFINITE = 7   /* ValueError "array must not contain infs or NaNs": what the reference's triangular
                             solves (scipy.linalg.solve_triangular, linalg.py:115, :128) raise on such operands */
};

/* storage / arithmetic formats (precision.py:12-19, plus bf16) */
enum sqb_dtype { SQB_F64 = 0, SQB_F32 = 1, SQB_F16 = 2, SQB_BF16 = 3 };

/* reflector scaling (linalg.py:25-32) */
enum sqb_scaling { SQB_SCALE_SQRT2 = 0, SQB_SCALE_UNIT = 1 };

/* sketch operator kinds */
enum sqb_sketch_kind {
  SQB_SKETCH_SRHT = 0,     /* SRHTSketch     sketching.py:128-155 */
  SQB_SKETCH_DENSE = 1,    /* GaussianSketch sketching.py:82-125 (and MatrixSketch :198-213) */
  SQB_SKETCH_IDENTITY = 2  /* IdentitySketch sketching.py:186-195 */
};

/*
 * A sketch operator Omega (ell x n) as device data.  Built by the caller
 * (the facade builds it from the same numpy RNG calls the reference makes,
 * sketching.py:100-107, :144-147, so signs, indices and G are bit-exact).
 */
typedef struct sqb_sketch {
  int32_t kind;               /* sqb_sketch_kind */
  int32_t reserved;
  int64_t ell;                /* rows of Omega */
  int64_t n;                  /* columns of Omega (input length) */
  /* SRHT */
  int64_t n_pad;              /* 1 << bit_length(n-1) (sketching.py:141) */
  double scale;               /* float(sqrt(n_pad/ell)) (sketching.py:147), fp64 */
  const uint32_t* sign_bits;  /* device, n_pad bits, bit e set <=> signs[e] == -1 */
  const int64_t* indices;     /* device, ell sampled rows, ORDERED (sketching.py:146) */
  /* DENSE */
  const double* G;            /* device, ell x n ROW-major (G[i*ldg + r]) */
  int64_t ldg;
} sqb_sketch;

typedef struct sqb_ctx sqb_ctx;

/* Linear operator for the Krylov driver (krylov.py:28-35 accepts a callable,
 * a scipy sparse matrix or a dense array). */
enum sqb_operator_kind { SQB_OP_CSR = 0, SQB_OP_DENSE = 1, SQB_OP_CALLBACK = 2 };
/* Callback operator: the library writes x (n values of the low dtype) into
 * the caller's device buffer `xbuf`, calls cb(user, stream), and reads the
 * float64 product A x from the caller's device buffer `ybuf`.  The callback
 * must enqueue its work on `stream` and return 0. */
typedef int (*sqb_matvec_cb)(void* user, void* stream);
typedef struct sqb_operator {
  int32_t kind;             /* sqb_operator_kind */
  int32_t reserved;
  int64_t n;                /* A is n x n */
  const int64_t* indptr;    /* CSR, device: n+1 */
  const int32_t* indices;   /* CSR, device: nnz */
  const double* data;       /* CSR, device: nnz */
  const double* A;          /* DENSE, device, row-major */
  int64_t lda;
  sqb_matvec_cb cb;         /* CALLBACK */
  void* user;
  void* xbuf;               /* CALLBACK: n values of the low dtype (device) */
  double* ybuf;             /* CALLBACK: n doubles (device) */
} sqb_operator;

/* ---- context ------------------------------------------------------------ */
int sqb_version(void);
int sqb_ctx_create(int device, void* stream, sqb_ctx** out);
int sqb_ctx_destroy(sqb_ctx* ctx);
int sqb_ctx_set_stream(sqb_ctx* ctx, void* stream);
/* message of the last host-side error of this context ("" if none) */
const char* sqb_ctx_last_error(sqb_ctx* ctx);
/* synchronise the stream, return the device status word and reset it */
int sqb_ctx_status(sqb_ctx* ctx, int* code, int* col, double* val);
/* Round a double to `dtype` the way the reference's numpy path does
 * (`dtype.type(x)`; bf16 through fp32 as ml_dtypes does).  Host helper. */
double sqb_round_scalar(int dtype, double x);
/* Kernel launches issued by this context since creation (instrumentation). */
int64_t sqb_ctx_launches(sqb_ctx* ctx);
/* Time every launch of the dominant kernel (rhqr_col_kernel) with CUDA events
 * on the context stream; read back the summed device time and algorithmic
 * bytes (used by bench.py for the roofline).  enable=0 turns it off. */
int sqb_ctx_profile(sqb_ctx* ctx, int enable);
int sqb_ctx_profile_read(sqb_ctx* ctx, double* total_ms, double* total_bytes, int64_t* launches);
/* Instrumentation: the step kernel of `column` writes per-phase clock64 stamps
 * (8 per cluster rank) to the device buffer dev_buf (NULL disables). */
int sqb_debug_step_stamps(sqb_ctx* ctx, long long* dev_buf, int column);
/* Instrumentation: stream trace.  While enabled an event is recorded after
 * every kernel launch of the library on the context stream; trace_read
 * synchronises and writes one line per kernel name, "name launches ms", the
 * in-stream time (launch gap + run) summed over its launches. */
int sqb_ctx_trace(sqb_ctx* ctx, int enable);
int sqb_ctx_trace_read(sqb_ctx* ctx, char* buf, int64_t size);
/* Instrumentation: every block b of the column pass of `column` writes
 * {SM id, globaltimer ns at entry, after the flag wait, after the bulk GEMV,
 * after griddepcontrol.wait, at exit} to dev_buf[8 b ..]; the step kernel of
 * the same column writes {entry, after its wait, exit} of cluster rank 0 to
 * dev_buf[8 nblocks ..] (nblocks = the pass's grid size).  NULL disables. */
int sqb_debug_col_stamps(sqb_ctx* ctx, long long* dev_buf, int column);

/* ---- sketches ------------------------------------------------------------
 * Y (ell x k, fp64, ldy) = Omega X, X (n x k, `dtype`, ldx), arithmetic in
 * `dtype` (replaces SketchOperator.apply, sketching.py:72-76; SRHT _apply
 * :149-155 + fwht :21-43 bit-exact; Gaussian _apply :109-125).           */
int sqb_sketch_apply(sqb_ctx* ctx, const sqb_sketch* sk, int dtype,
                     const void* X, int64_t ldx, int64_t k,
                     double* Y, int64_t ldy);

/* Psi X = [X[:m]; Omega X[m:]] (EmbeddedSketch.apply, sketching.py:255-260);
 * X is (m+n) x k, Y is (m+ell) x k. */
int sqb_embedded_apply(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, int dtype,
                       const void* X, int64_t ldx, int64_t k,
                       double* Y, int64_t ldy);

/* ---- factorizations ------------------------------------------------------
 * Left-looking RHQR (rhqr_left, rhqr.py:254-267; sweep :219-251).
 * W: N x m in `lo_dtype` (already rounded to it, rhqr.py:264); outputs U
 * (N x m, lo_dtype), S ((m+ell) x m), T (m x m), R (m x m), sigmas, rhos,
 * betas (m), all zero-initialised by the call.  High precision is fp64.
 * Breakdown -> device status SQB_ERR_BREAKDOWN with the 1-based column.   */
int sqb_rhqr_left(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                  const void* W, int64_t N, int64_t m, int64_t ldw,
                  void* U, int64_t ldu, double* S, int64_t lds,
                  double* T, int64_t ldt, double* R, int64_t ldr,
                  double* sigmas, double* rhos, double* betas);

/* The same factorization with HOST operands: the call shape of the
 * reference's rhqr_left (numpy W in, float64 numpy factors out,
 * rhqr.py:254-267).  W: N x m float64 host array, row-major (w_layout 0,
 * C-order, element (i, j) at W[i*ldw + j]) or column-major (w_layout 1,
 * W[i + j*ldw]); it is rounded to lo_dtype on the device (round_to,
 * rhqr.py:264; overflow -> device status SQB_ERR_RANGE, val = largest
 * offending |w|).  Outputs are float64 host arrays, column-major: U (N x m,
 * ldu), S ((m+ell) x m), T, R (m x m), sigmas/rhos/betas (m).  The PCIe
 * transfers overlap the factorization: a column-major W streams in column
 * groups as the sweep needs them, and U streams back in column groups as
 * they become final.  Host buffers should be page-locked (pageable ones are
 * staged synchronously by the driver, which removes the overlap).  Returns
 * after the outputs are written; device scratch belongs to the context.   */
int sqb_rhqr_left_host(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                       const double* W, int64_t N, int64_t m, int64_t ldw, int w_layout,
                       double* U, int64_t ldu, double* S, int64_t lds,
                       double* T, int64_t ldt, double* R, int64_t ldr,
                       double* sigmas, double* rhos, double* betas);

/* rec_rhqr with HOST operands (rhqr.py:368-395; replaces the whole
 * reference call with numpy W in and numpy factors out): W (float64,
 * row-major w_layout = 0 or column-major 1) is uploaded in row blocks aligned
 * to the split-K slabs of the Gaussian sketch GEMM, and each block's slabs
 * start on a side stream as soon as it is resident (the sketch runs under the
 * upload; Z is bitwise that of sqb_rec_rhqr).  Other sketches / precisions:
 * blocked upload, then the device path.  U (float64, column-major, ldu) comes
 * back after the reconstruction solve; S, T, R and the scalars as in
 * sqb_rec_rhqr.  Host buffers should be page-locked.  Returns after the
 * outputs are written.                                                     */
int sqb_rec_rhqr_host(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                      const double* W, int64_t N, int64_t m, int64_t ldw, int w_layout,
                      double* U, int64_t ldu, double* S, int64_t lds,
                      double* T, int64_t ldt, double* R, int64_t ldr,
                      double* sigmas, double* rhos, double* betas);

/* Release the context's grow-only device scratch (workspace and the
 * host-operand arena); it is re-allocated on the next call that needs it. */
int sqb_ctx_trim(sqb_ctx* ctx);

/* Blocked left-looking RHQR (rhqr_block, rhqr.py:334-365): panels of
 * block_size columns; every earlier panel is applied compactly to the panel
 * (one re-sketch per earlier panel), then the panel is swept with pivot
 * offset j0.  T receives the panel triangles on its diagonal blocks
 * (BlockRHQRFactors.panels[k].T) and zeros elsewhere; the stacked compact T
 * is sqb_t_factor(S).  Other outputs as sqb_rhqr_left.                    */
int sqb_rhqr_block(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                   const void* W, int64_t N, int64_t m, int64_t ldw, int64_t block_size,
                   void* U, int64_t ldu, double* S, int64_t lds,
                   double* T, int64_t ldt, double* R, int64_t ldr,
                   double* sigmas, double* rhos, double* betas);

/* Right-looking RHQR (rhqr_right, rhqr.py:270-301): per column, sketch the
 * trailing block, one reflector, rank-1 update of the trailing block; T from
 * sqb_t_factor(S) at the end.  Arguments as sqb_rhqr_left.                 */
int sqb_rhqr_right(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                   const void* W, int64_t N, int64_t m, int64_t ldw,
                   void* U, int64_t ldu, double* S, int64_t lds,
                   double* T, int64_t ldt, double* R, int64_t ldr,
                   double* sigmas, double* rhos, double* betas);

/* Trimmed left-looking RHQR (trim_rhqr_left, trim.py:272-325).  The sketch
 * sk acts on all N coordinates; the column-scaled wrapper (sketching.py:
 * 216-235) multiplies coordinates k < mscale by scales[k] first (mscale >= m:
 * the span the operator was normalised over — an operator wrapped for more
 * columns than W has is used unchanged, trim.py:59-60), and E (ell x m,
 * ld lde) holds its unit leading-column sketches (normalize_leading_columns,
 * trim.py:51-77, built by the caller).  Outputs U (N x m, lo dtype, 16-byte
 * aligned), S (ell x m), T, T~, R, L (m x m, fp64) and the scalars.
 * Breakdown -> SQB_ERR_BREAKDOWN, col = j | kind << 24 (0: sketched tail
 * annihilated, 1: sketched reflector cancelled, val = norm; 2: unit pivot
 * vanished, val = pivot).                                                 */
int sqb_trim_rhqr_left(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales,
                       int64_t mscale, const double* E, int64_t lde, int scaling, int lo_dtype,
                       const void* W, int64_t N, int64_t m, int64_t ldw,
                       void* U, int64_t ldu, double* S, int64_t lds,
                       double* T, int64_t ldt, double* Tt, int64_t ldtt,
                       double* R, int64_t ldr, double* L, int64_t ldl,
                       double* sigmas, double* rhos, double* betas);

/* Trimmed right-looking RHQR (trim_rhqr_right, trim.py:238-269): per column
 * the tail reflector, then the trailing block updated through the masked
 * sketch; T = t_factor_from_sketches(S), T~ = t_tilde_from_factors(S, E, U),
 * L = tril(S^t E, -1) after the sweep.  Arguments as sqb_trim_rhqr_left.  */
int sqb_trim_rhqr_right(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales,
                        int64_t mscale, const double* E, int64_t lde, int scaling, int lo_dtype,
                        const void* W, int64_t N, int64_t m, int64_t ldw,
                        void* U, int64_t ldu, double* S, int64_t lds,
                        double* T, int64_t ldt, double* Tt, int64_t ldtt,
                        double* R, int64_t ldr, double* L, int64_t ldl,
                        double* sigmas, double* rhos, double* betas);

/* The column-scaled operator alone (ColumnScaledSketch._apply,
 * sketching.py:230-235): Y = Omega (X with rows k < m times scales[k] in the
 * arithmetic dtype).  X: sk->n x k (dtype), Y: ell x k fp64.               */
int sqb_colscaled_apply(sqb_ctx* ctx, const sqb_sketch* sk, const double* scales, int64_t m,
                        int dtype, const void* X, int64_t ldx, int64_t k, double* Y, int64_t ldy);

/* Trimmed thin Q = [I;0] - U T triu(S^t E) in fp64 (trim_thin_q,
 * trim.py:211-225).  U: N x k (lo), T: k x k, S and E: ell x k.            */
int sqb_trim_thin_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t k,
                    const double* T, int64_t ldt, const double* S, int64_t lds,
                    const double* E, int64_t lde, int64_t ell, double* Q, int64_t ldq);

/* T of the compact form from S = Psi U alone (t_factor_from_sketches,
 * rhqr.py:122-132): T^{-1} = triu(S^t S, 1) + diag(S^t S)/2, inverted by back
 * substitution.  S: od x k fp64, T: k x k.  Singular -> SQB_ERR_SINGULAR.  */
int sqb_t_factor(sqb_ctx* ctx, const double* S, int64_t lds, int64_t od, int64_t k,
                 double* T, int64_t ldt);

/* Reconstructed RHQR (rec_rhqr, rhqr.py:368-395): one sketch Z = Psi W,
 * Householder QR of Z in fp64 (baselines.py:33-89), Mfac = triu(T^t S^t Z)
 * (zero diagonal -> SQB_ERR_BREAKDOWN with val = -1), U2 = W2 Mfac^{-1} by
 * forward substitution (right_tri_solve, linalg.py:119-129), U = [S[:m]; U2].
 * Same operands as sqb_rhqr_left. */
int sqb_rec_rhqr(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                 const void* W, int64_t N, int64_t m, int64_t ldw,
                 void* U, int64_t ldu, double* S, int64_t lds,
                 double* T, int64_t ldt, double* R, int64_t ldr,
                 double* sigmas, double* rhos, double* betas);

/* ---- multi-GPU (row partition) ------------------------------
 * Rank p of P owns Omega coordinates [p n_pad/P, (p+1) n_pad/P) (whole SRHT
 * tiles; needs n_pad/P >= the tile size) and rank 0 also the m identity rows.
 * W/U local storage: rank 0 [m identity rows; its Omega rows], others [their
 * Omega rows].  One all-gather of an (ell+m)-vector per column (NCCL); the
 * top log2(P) SRHT tree levels are completed in rank order, so every output
 * is bitwise identical to the single-GPU factorization. */
int sqb_nccl_unique_id(char* out, int size);
int sqb_ctx_init_comm(sqb_ctx* ctx, const char* id, int nranks, int rank);

/* In-kernel peer-memory exchange for the row-partitioned factorizations
 * (replaces the per-column ncclAllGather of sqb_rhqr_left_dist /
 * sqb_rec_rhqr_dist).  Each rank allocates a mailbox of
 * 2 x nranks slots of `count` doubles (count >= m (m + ell)) and returns its
 * CUDA IPC handle (64 bytes) in handle_out; the handles are exchanged by the
 * caller (e.g. torch.distributed.all_gather_object) and passed, rank-ordered,
 * to sqb_p2p_open, which maps every peer's mailbox (NVLink peer access).  From
 * then on a rank's partials are stored straight into the peers' mailboxes by
 * a kernel and published with system-scope release flags that the consuming
 * step kernel acquires: no collective launch on the per-column path.
 * sqb_p2p_virtual sets up the same exchange between `nranks` virtual ranks on
 * one device (sqb_*_virtual entries); sqb_p2p_close releases it.          */
int sqb_p2p_mailbox(sqb_ctx* ctx, int nranks, int64_t count, void* handle_out);
int sqb_p2p_open(sqb_ctx* ctx, int rank, const void* handles);
int sqb_p2p_virtual(sqb_ctx* ctx, int nranks, int64_t count);
int sqb_p2p_close(sqb_ctx* ctx);
/* A consumer that waits longer than `ms` (default 20 s; 0 restores it) for a
 * peer's flag records SQB_ERR_NCCL with col = -(peer + 1) in the device status
 * instead of spinning for ever (a rank that died must not hang the others'
 * streams).  An all-zero handle in sqb_p2p_open's table stands for such a
 * peer (tests). */
int sqb_p2p_set_timeout_ms(sqb_ctx* ctx, int64_t ms);

/* Halo ranges of the row-partitioned SpMV in the distributed RHQR-Arnoldi
 * (exchange only the referenced entries — one grid row with
 * each neighbour for the 5-point stencil — instead of all-gathering q):
 * table[(r P + p) 2 + {0, 1}] = [lo, hi) of rank p's segment that rank r's
 * CSR rows reference.  NULL clears it (all-gather of q).                  */
int sqb_ctx_set_halo(sqb_ctx* ctx, int nranks, const int64_t* table);
int sqb_rhqr_left_dist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                       const void* W, int64_t n_local, int64_t m, int64_t ldw,
                       void* U, int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt,
                       double* R, int64_t ldr, double* sigmas, double* rhos, double* betas,
                       void* Utop_scratch);
/* The same algorithm with P "virtual ranks" on one device (row blocks
 * W_parts[p], the all-gather as device copies): the single-GPU test of the
 * multi-GPU path.  Outputs are rank 0's; scratch >= (P-1)*((m+ell)m + 3m^2 + 3m)
 * doubles. */
int sqb_rhqr_left_virtual(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                          int nranks, const void* const* W_parts, const int64_t* ldw,
                          void* const* U_parts, const int64_t* ldu, int64_t m,
                          double* S, int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr,
                          double* sigmas, double* rhos, double* betas, double* scratch);

/* Row-partitioned recRHQR (rec_rhqr, rhqr.py:368-395) on the same partition:
 * rank-local SRHT subtrees of Psi W, ONE all-gather of the (ell+m) x m
 * partials, the rank-order combine (Z bitwise the single-GPU sketch), the
 * sketch-space QR and Mfac redundantly on every rank, then each rank solves
 * its own rows U2 = W2 Mfac^{-1} (rank 0 also U[:m] = S[:m]).  Arguments as
 * sqb_rhqr_left_dist (no Utop scratch); the _virtual form runs P ranks on
 * one device (scratch as sqb_rhqr_left_virtual). */
int sqb_rec_rhqr_dist(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                      const void* W, int64_t n_local, int64_t m, int64_t ldw,
                      void* U, int64_t ldu, double* S, int64_t lds, double* T, int64_t ldt,
                      double* R, int64_t ldr, double* sigmas, double* rhos, double* betas);
int sqb_rec_rhqr_virtual(sqb_ctx* ctx, const sqb_sketch* sk, int scaling, int lo_dtype,
                         int nranks, const void* const* W_parts, const int64_t* ldw,
                         void* const* U_parts, const int64_t* ldu, int64_t m,
                         double* S, int64_t lds, double* T, int64_t ldt, double* R, int64_t ldr,
                         double* sigmas, double* rhos, double* betas, double* scratch);

/* Left-looking Householder QR with compact T of a small fp64 A (p x m) in one
 * CTA (householder_qr, baselines.py:33-89; the sketch-space QR of recRHQR).
 * Outputs U (p x m), T, R (m x m), sigmas/rhos/betas; an exactly dependent
 * column -> SQB_ERR_BREAKDOWN. */
int sqb_householder_qr(sqb_ctx* ctx, int scaling, const double* A, int64_t lda, int64_t p, int64_t m,
                       double* U, int64_t ldu, double* T, int64_t ldt, double* R, int64_t ldr,
                       double* sigmas, double* rhos, double* betas);

/* R X = B for upper-triangular fp64 R (m x m), B/X (m x k) (upper_tri_solve,
 * linalg.py:102-116); zero/subnormal diagonal -> SQB_ERR_SINGULAR. */
int sqb_upper_tri_solve(sqb_ctx* ctx, const double* R, int64_t ldr, int64_t m, const double* B,
                        int64_t ldb, int64_t k, double* X, int64_t ldx);

/* (I - U T S^t Psi) X, or with transpose_t the reflectors in reverse
 * (apply_reflectors_compact, rhqr.py:100-119).  U: N x r (lo), S: (m+ell) x r,
 * T: r x r, X/Out: N x k (lo).  Out may alias X. */
int sqb_apply_reflectors(sqb_ctx* ctx, const sqb_sketch* sk, int64_t m, int lo_dtype,
                         const void* U, int64_t ldu, int64_t N, int64_t r,
                         const double* S, int64_t lds, const double* T, int64_t ldt,
                         int transpose_t, const void* X, int64_t ldx, int64_t k,
                         void* Out, int64_t ldo);

/* thin Q = [I;0] - U (T U1^t) in fp64 (thin_q, rhqr.py:171-178).  U: N x k. */
int sqb_thin_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N,
               int64_t k, const double* T, int64_t ldt, double* Q, int64_t ldq);

/* Gram matrix G = A^t A (k x k, fp64) of a fp64 N x k matrix (diagnostics
 * orthogonality_error/cond_number, linalg.py:151-160, :193-197). */
int sqb_gram(sqb_ctx* ctx, const double* A, int64_t lda, int64_t N, int64_t k,
             double* G, int64_t ldgm);

/* Psi Q = [I;0] - S (T U1^t) without touching n-dimensional data
 * (sketch_q, rhqr.py:181-188).  S: od x k, U: top k rows used. */
int sqb_sketch_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t k,
                 const double* T, int64_t ldt, const double* S, int64_t lds, int64_t od,
                 double* Q, int64_t ldq);

/* out[j] = ||(W - Q R)[:, j]||^2, out[kc + j] = ||W[:, j]||^2 (fp64; the
 * sums behind factorization_errors, linalg.py:169-190).  W: N x kc,
 * Q: N x k, R: k x kc. */
int sqb_residual_norms(sqb_ctx* ctx, const double* W, int64_t ldw, const double* Q, int64_t ldq,
                       const double* R, int64_t ldr, int64_t N, int64_t k, int64_t kc,
                       double* out);

/* One randomized Householder reflector from w (n, lo_dtype) and its sketch
 * y = Psi w (od, fp64) eliminating entries j+1.. (1-based j; rh_vector,
 * rhqr.py:51-97): writes u (n, lo_dtype), s = Psi u (od, fp64) and
 * scalars[0..4] = sigma, rho, beta, f, gamma.  Breakdown (rho == 0 or
 * non-finite beta) goes to the device status word. */
int sqb_rh_vector(sqb_ctx* ctx, int scaling, int lo_dtype, const void* w, int64_t n,
                  const double* y, int64_t od, int64_t j, void* u, double* s,
                  double* scalars);

/* RHQR-Arnoldi (rhqr_arnoldi, krylov.py:82-150): m steps of the Krylov basis
 * of (A, b - A x0) in compact reflector form.  b: n doubles; x0lo: n values
 * already rounded to lo_dtype; outputs U (n x (m+1), lo_dtype), S
 * ((m+1+ell) x (m+1)), T ((m+1)^2), H ((m+1) x m), optional Q (n x m fp64,
 * krylov.py:139; pass NULL when store_q is false), beta (device double).
 * Omega must take n-m-1 coordinates.  happy_tol: krylov.py:101-102.
 * Synchronises once at the end; *attained = -1 for a full run, else the
 * dimension at which the space closed. */
int sqb_rhqr_arnoldi(sqb_ctx* ctx, const sqb_sketch* sk, const sqb_operator* A, int m,
                     int scaling, int lo_dtype, double happy_tol, const double* b,
                     const void* x0lo, void* U, int64_t ldu, double* S, int64_t lds,
                     double* T, int64_t ldt, double* H, int64_t ldh, double* Q, int64_t ldq,
                     double* beta, int* attained);

/* min_y ||beta e1 - H y|| by Givens rotations (hessenberg_lstsq,
 * krylov.py:153-190): H is p x k (p = k+1 normally), outputs y (k), the
 * residual history (k+1) and the final residual; work >= p*k + p doubles. */
int sqb_hessenberg_lstsq(sqb_ctx* ctx, const double* H, int64_t ldh, int64_t p, int64_t k,
                         double beta, double* y, double* hist, double* resid, double* work);

/* Basis columns q_1..q_c from the compact form: Q = [I;0] - U (T S[:c, :]^t)
 * (arnoldi_q, krylov.py:64-79).  U: N x r (lo_dtype), S: od x r, T: r x r. */
int sqb_arnoldi_q(sqb_ctx* ctx, int lo_dtype, const void* U, int64_t ldu, int64_t N, int64_t r,
                  const double* T, int64_t ldt, const double* S, int64_t lds, int64_t c,
                  double* Q, int64_t ldq);

/* y = lo(b - A x) (bsub != NULL) or lo(A x): CSR SpMV, row sums in CSR order
 * with separate mul/add roundings (scipy's csr_matvec). */
int sqb_csr_spmv(sqb_ctx* ctx, int dtype, int64_t n, const int64_t* indptr,
                 const int32_t* indices, const double* data, const void* x,
                 const double* bsub, void* y);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHQR_B200_H */
