"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `sketchqr` from /root/reference/pkg/src unmodified (a bf16 tag is
injected at runtime for the mixed-precision fixture, exactly as SURVEY A.6 —
the reference source is not edited) and writes small `.npz` files next to
this script.  The fixtures pin the oracle (`oracle/sketchqr_oracle.py`) and
are the GPU parity tests' known answers.  Nothing on the GPU box reads
/root/reference.
"""

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import sketchqr  # noqa: E402
from sketchqr import precision as P  # noqa: E402
from sketchqr.baselines import householder_qr  # noqa: E402
from sketchqr.experiments import gen_cmatrix  # noqa: E402
from sketchqr.krylov import hessenberg_lstsq, rhqr_arnoldi, rhqr_gmres  # noqa: E402
from sketchqr.linalg import cond_number, factorization_errors, orthogonality_error  # noqa: E402
from sketchqr.rhqr import (apply_reflectors_compact, rec_rhqr, rh_vector,  # noqa: E402
                           rhqr_block, rhqr_left, rhqr_right, sketch_q, t_factor_from_sketches,
                           thin_q)
from sketchqr.sketching import (EmbeddedSketch, GaussianSketch,  # noqa: E402
                                IdentitySketch, SRHTSketch)


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    print("wrote", name, {k: np.shape(v) for k, v in arrs.items()})


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def srht_cases():
    # (ell, n, seed, k) — includes the padding case n=12 (test_sketching.py:92)
    # and the config-1 Omega shape (n = 2^14 - 32)
    cases = [(8, 12, 3, 3), (5, 6, 21, 1), (64, 1000, 5, 4), (128, 16352, 7, 2),
             (256, 65536 - 128, 11, 2), (400, 8191, 13, 1)]
    for ell, n, seed, k in cases:
        op = SRHTSketch(ell, n, seed)
        rng = np.random.default_rng(seed + 1000)
        X = rng.standard_normal((n, k))
        out = dict(ell=ell, n=n, seed=seed, n_pad=op.n_pad, scale=op.scale,
                   signbits=np.packbits(op.signs < 0, bitorder="little"),
                   indices=op.indices, X=X, Y64=op.apply(X),
                   Y32=op.apply(P.round_to(X, "single"), dtype=np.float32))
        if n <= 4096:  # fp16 overflows for large n
            out["Y16"] = op.apply(P.round_to(X, "half"), dtype=np.float16)
        save(f"srht_{ell}_{n}_{seed}", **out)


def gauss_cases():
    op = GaussianSketch(8, 50, 2)
    rng = np.random.default_rng(77)
    X = rng.standard_normal((50, 3))
    G = op._cache[np.dtype(np.float64)]
    save("gauss_8_50_2", G=G, X=X, Y=op.apply(X))
    op = GaussianSketch(24, 5000, 9)  # 24*5000 <= 2^23: cached
    save("gauss_24_5000_9_sha", sha=np.frombuffer(
        bytes.fromhex(sha(op._cache[np.dtype(np.float64)])), dtype=np.uint8))


def rh_vector_cases():
    psi = EmbeddedSketch(2, IdentitySketch(2))
    w = np.array([3.0, 0.0, 4.0, 0.0])
    a = rh_vector(w, psi.apply(w), 1)
    b = rh_vector(w, psi.apply(w), 1, scaling="unit")
    save("rh_vector_345", w=w, u_sqrt2=a.u, s_sqrt2=a.s, beta_sqrt2=a.beta,
         rho=a.rho, sigma=a.sigma, u_unit=b.u, s_unit=b.s, beta_unit=b.beta)


def factor_dump(F):
    return dict(U=F.U, S=F.S, T=F.T, R=F.R, sigmas=F.sigmas, rhos=F.rhos,
                betas=F.betas)


def diag_dump(W, F):
    Q = thin_q(F)
    fro, mx, _ = factorization_errors(W, Q, F.R)
    return dict(cond_q=cond_number(Q), orth=orthogonality_error(F.psi.apply(Q)),
                orth_sq=orthogonality_error(sketch_q(F)), fro=fro, maxcol=mx)


def rhqr_cases():
    # reduced config 1 / config 2 shapes plus unit scaling and a ragged n
    rng = np.random.default_rng(1)
    W = rng.standard_normal((2048, 16))
    F = rhqr_left(W, SRHTSketch(64, 2048 - 16, 5))
    save("rhqr_left_2048x16_srht64", W=W, seed=5, ell=64, **factor_dump(F), **diag_dump(W, F))
    F = rhqr_left(W, SRHTSketch(64, 2048 - 16, 5), scaling="unit")
    save("rhqr_left_2048x16_srht64_unit", W=W, seed=5, ell=64, **factor_dump(F))
    rng = np.random.default_rng(2)
    W = rng.standard_normal((1000, 12))
    F = rhqr_left(W, GaussianSketch(40, 1000 - 12, 8))
    save("rhqr_left_1000x12_gauss40", W=W, seed=8, ell=40, **factor_dump(F))
    # config-1 full size (2^14 x 32, SRHT 128): keep the small factors and U checksums
    rng = np.random.default_rng(2024)
    W = rng.standard_normal((1 << 14, 32))
    F = rhqr_left(W, SRHTSketch(128, (1 << 14) - 32, 17))
    d = factor_dump(F)
    U = d.pop("U")
    save("rhqr_left_cfg1", W_seed=2024, seed=17, ell=128, U_colnorm=np.linalg.norm(U, axis=0),
         U_head=U[:64], U_tail=U[-64:], **d, **diag_dump(W, F))
    # ill-conditioned config-2 shape at reduced n
    rng = np.random.default_rng(3)
    n, m = 1 << 14, 32
    A = np.linalg.qr(rng.standard_normal((n, m)))[0]
    B = np.linalg.qr(rng.standard_normal((m, m)))[0]
    W = A @ np.diag(np.logspace(0, -15, m)) @ B
    F = rhqr_left(W, SRHTSketch(64, n - m, 23))
    d = factor_dump(F)
    U = d.pop("U")
    # W is regenerated by tests/golden/inputs.py (same numpy recipe); its sha pins it
    save("rhqr_left_illcond_16384x32", W_sha=np.array(sha(W)), seed=23, ell=64,
         U_colnorm=np.linalg.norm(U, axis=0), U_head=U[:64], **d, **diag_dump(W, F))
    # breakdown on an exactly dependent column (test_rhqr.py:296-301)
    W = np.zeros((32, 2))
    W[0] = 1.0
    try:
        rhqr_left(W, SRHTSketch(12, 30, 34))
        msg = "none"
    except sketchqr.BreakdownError as e:
        msg = str(e)
    save("rhqr_breakdown", W=W, msg=np.array(msg))


def mixed_cases():
    rng = np.random.default_rng(4)
    W = rng.standard_normal((4096, 16))
    for tag in ("single", "half"):
        pol = P.PrecisionPolicy(high="double", low=tag)
        F = rhqr_left(W, SRHTSketch(64, 4096 - 16, 29), policy=pol)
        save(f"rhqr_left_4096x16_{tag}", W=W, seed=29, ell=64, **factor_dump(F))
    # bf16 injection — runtime only, reference source untouched
    import ml_dtypes
    if "bf16" not in P.PRECISIONS:
        P.PRECISIONS = P.PRECISIONS + ("bf16",)
        P.DTYPES["bf16"] = ml_dtypes.bfloat16
        P.UNIT_ROUNDOFF["bf16"] = 2.0 ** -8
    Ws = W * np.logspace(0, -8, 16)[None, :]
    pol = P.PrecisionPolicy(high="double", low="bf16")
    F = rhqr_left(Ws, SRHTSketch(64, 4096 - 16, 31), policy=pol)
    save("rhqr_left_4096x16_bf16", W=Ws, seed=31, ell=64, **factor_dump(F))
    op = SRHTSketch(64, 4096 - 16, 31)
    Xb = P.round_to(rng.standard_normal((4096 - 16, 2)), "bf16")
    save("srht_bf16_64_4080_31", X=Xb, Y=op.apply(Xb, dtype=ml_dtypes.bfloat16))


def rec_cases():
    W = gen_cmatrix(4096, 16)
    F = rec_rhqr(W, GaussianSketch(64, 4096 - 16, 41))
    save("rec_rhqr_cmatrix_4096x16", W=W, seed=41, ell=64, **factor_dump(F), **diag_dump(W, F))
    Z = np.random.default_rng(5).standard_normal((80, 16))
    Q, R, _, aux = householder_qr(Z)
    save("householder_80x16", Z=Z, Q=Q, R=R, U=aux["U"], T=aux["T"])


def krylov_cases():
    rng = np.random.default_rng(6)
    n, m = 400, 20
    A = rng.standard_normal((n, n)) / np.sqrt(n) + 2.0 * np.eye(n)
    A[rng.random((n, n)) < 0.9] = 0.0
    A += 2.0 * np.eye(n)
    b = rng.standard_normal(n)
    om = SRHTSketch(4 * (m + 1), n - m - 1, 43)
    bun = rhqr_arnoldi(A, b, None, m, om)
    x, hist = rhqr_gmres(A, b, None, m, om)
    save("arnoldi_400_m20", A=A, b=b, seed=43, ell=4 * (m + 1), U=bun.U, S=bun.S, T=bun.T,
         H=bun.H, beta=bun.beta, Q=bun.Q_cols, x=x, hist=hist)
    H = np.triu(np.random.default_rng(7).standard_normal((11, 10)), -1)
    y, res, h = hessenberg_lstsq(H, 1.7, history=True)
    save("hessenberg_11x10", H=H, beta=1.7, y=y, res=res, hist=h)


def apply_compact_cases():
    rng = np.random.default_rng(8)
    n, m = 600, 8
    W = rng.standard_normal((n, m))
    F = rhqr_left(W, SRHTSketch(32, n - m, 47))
    X = rng.standard_normal((n, 3))
    save("apply_compact_600x8", W=W, seed=47, ell=32, X=X,
         Y=apply_reflectors_compact(F.U, F.S, F.T, X, F.psi),
         Yt=apply_reflectors_compact(F.U, F.S, F.T, X, F.psi, transpose_t=True),
         Q=thin_q(F), SQ=sketch_q(F))


def block_cases():
    # rhqr_block: one panel, degenerate, ragged final panel (test_rhqr.py:225-235)
    rng = np.random.default_rng(11)
    n, m = 1500, 20
    W = rng.standard_normal((n, m))
    out = dict(W=W, seed=53, ell=48)
    for bs in (20, 1, 6, 8):
        B = rhqr_block(W, SRHTSketch(48, n - m, 53), block_size=bs)
        Fs = B.stacked()
        out[f"R_{bs}"] = B.R
        out[f"U_{bs}"] = Fs.U
        out[f"S_{bs}"] = Fs.S
        out[f"Tst_{bs}"] = Fs.T
        out[f"Tblk_{bs}"] = np.concatenate([p.T.ravel() for p in B.panels])
        out[f"scal_{bs}"] = np.stack([B.sigmas, B.rhos, B.betas])
    save("rhqr_block_1500x20_srht48", **out)
    S = rng.standard_normal((30, 8))
    save("t_factor_30x8", S=S, T=t_factor_from_sketches(S))
    # rhqr_right (rhqr.py:270-301), fp64 and unit scaling
    W = rng.standard_normal((900, 12))
    F = rhqr_right(W, SRHTSketch(36, 900 - 12, 59))
    Fu = rhqr_right(W, SRHTSketch(36, 900 - 12, 59), scaling="unit")
    save("rhqr_right_900x12_srht36", W=W, seed=59, ell=36, **factor_dump(F),
         U_unit=Fu.U, R_unit=Fu.R, T_unit=Fu.T)


def experiment_cases():
    """The stability-sweep harness (experiments.py:125-339) on small inputs:
    metric rows and the deterministic CSV bytes, per algorithm."""
    import io
    import tempfile

    import scipy.sparse
    from sketchqr.experiments import (ExperimentConfig, run_factor_experiment, run_gmres_experiment,
                                      write_csv)

    def pack(rows):
        return (np.array([r[0] for r in rows], dtype=np.int64),
                np.array([list(r[1:-1]) for r in rows], dtype=np.float64),
                np.array([r[-1] for r in rows]))

    def csv_bytes(rows, cfg):
        with tempfile.NamedTemporaryFile("r", suffix=".csv") as fh:
            write_csv(fh.name, rows, config=cfg, extra="golden")
            return np.frombuffer(open(fh.name, "rb").read(), dtype=np.uint8)

    out = {}
    W = gen_cmatrix(2048, 48)
    cases = {
        "left": ExperimentConfig(algo="rhqr-left", seed=3, every=8, deterministic=True),
        "right": ExperimentConfig(algo="rhqr-right", seed=3, every=8, deterministic=True),
        "block": ExperimentConfig(algo="rhqr-block", seed=3, every=8, block_size=16, deterministic=True),
        "rec": ExperimentConfig(algo="rec-rhqr", seed=3, every=16, deterministic=True),
        "leftgauss": ExperimentConfig(algo="rhqr-left", sketch="gauss", ell=120, seed=5, every=12,
                                      deterministic=True),
        "mixed": ExperimentConfig(algo="rhqr-left", ell=96, seed=2, precision="mixed", every=8,
                                  deterministic=True),
    }
    for name, cfg in cases.items():
        rows = run_factor_experiment(W, cfg)
        j, vals, st = pack(rows)
        out[f"{name}_j"], out[f"{name}_vals"], out[f"{name}_status"] = j, vals, st
        out[f"{name}_csv"] = csv_bytes(rows, cfg)
    # breakdown: an all-zero column 4 (rhqr.py:73-79 -> 'breakdown@4', NaN rows after)
    Wb = np.random.default_rng(77).standard_normal((512, 10))
    Wb[:, 3] = 0.0
    cfg = ExperimentConfig(algo="rhqr-left", seed=1, every=2, deterministic=True)
    j, vals, st = pack(run_factor_experiment(Wb, cfg))
    out.update(bd_W=Wb, bd_j=j, bd_vals=vals, bd_status=st)
    save("experiments_cmatrix_2048x48", W_sha=np.array(sha(W)), **out)

    # GMRES sweep (experiments.py:247-299) on a 24^2 convection-diffusion grid
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2405_10923_b200.workloads import convection_diffusion_csr
    ip, ix, dv = convection_diffusion_csr(24)
    A = scipy.sparse.csr_matrix((dv, ix, ip), shape=(576, 576))
    b = np.random.default_rng(81).standard_normal(576)
    g = {}
    for name, cfg in {"srht": ExperimentConfig(algo="rhqr", seed=4, deterministic=True),
                      "gauss": ExperimentConfig(algo="rhqr", sketch="gauss", ell=100, seed=6,
                                                deterministic=True)}.items():
        rows = run_gmres_experiment(A, b, 24, cfg)
        j, vals, st = pack(rows)
        g[f"{name}_j"], g[f"{name}_vals"], g[f"{name}_status"] = j, vals, st
        g[f"{name}_csv"] = csv_bytes(rows, cfg)
    rows = run_gmres_experiment(np.eye(32), b[:32], 5, ExperimentConfig(algo="rhqr", sketch="gauss", seed=1))
    j, vals, st = pack(rows)
    g.update(eye_j=j, eye_vals=vals, eye_status=st)
    save("experiments_gmres_cd24", indptr=ip, indices=ix, data=dv, b=b, **g)


def trim_cases():
    """Trimmed RHQR (trim.py:51-325): ell < m, left and right drivers, both
    scalings, a single-precision policy, and the exact-dependence breakdown."""
    from sketchqr.trim import (normalize_leading_columns, trim_rhqr_left, trim_rhqr_right,
                               trim_thin_q)
    rng = np.random.default_rng(71)
    N, m, ell, seed = 2048, 16, 12, 73
    W = rng.standard_normal((N, m)) * np.logspace(0, -6, m)
    om = SRHTSketch(ell, N, seed)
    wrapped = normalize_leading_columns(om, m)

    def dump(F, pre=""):
        return {pre + k: getattr(F, k) for k in ("U", "S", "T", "T_tilde", "R", "L", "E",
                                                  "sigmas", "rhos", "betas")}
    F = trim_rhqr_left(W, om)
    Fu = trim_rhqr_left(W, om, scaling="unit")
    Fr = trim_rhqr_right(W, om)
    Fs = trim_rhqr_left(W, om, policy=P.policy_from_tag("single"))
    save("trim_2048x16_srht12", W=W, seed=seed, ell=ell, scales=wrapped.scales[:m],
         Q=trim_thin_q(F), **dump(F), **dump(Fu, "unit_"), **dump(Fr, "right_"), **dump(Fs, "single_"))
    Wd = np.zeros((64, 2))
    Wd[0] = 1.0  # test_trim.py:215-220: the second tail is exactly zero after the update
    try:
        trim_rhqr_left(Wd, SRHTSketch(12, 64, 37))
        msg = ""
    except Exception as e:  # BreakdownError
        msg = str(e)
    save("trim_breakdown", W=Wd, seed=37, ell=12, msg=np.array(msg))
    # the stability-sweep harness on the trimmed drivers (experiments.py:161-164, 196-199)
    from sketchqr.experiments import ExperimentConfig, run_factor_experiment
    Wx = rng.standard_normal((2048, 24)) * np.logspace(0, -4, 24)
    out = {}
    for name, algo in (("trimleft", "trim-left"), ("trimright", "trim-right")):
        rows = run_factor_experiment(Wx, ExperimentConfig(algo=algo, ell=20, seed=3, every=6,
                                                          deterministic=True))
        out[f"{name}_j"] = np.array([r[0] for r in rows], dtype=np.int64)
        out[f"{name}_vals"] = np.array([list(r[1:-1]) for r in rows], dtype=np.float64)
        out[f"{name}_status"] = np.array([r[-1] for r in rows])
    save("experiments_trim", W=Wx, **out)


# ---------------------------------------------------------------------------
# BASELINE configs at their own shapes (round 2).  Inputs are regenerated on
# the GPU box by paper_2405_10923_b200.workloads (the same numpy recipes, same
# seeds as bench.py) and pinned here by sha256; only small outputs are stored.
# Each section takes tens of seconds to minutes of CPU; run them in parallel:
#   for s in cfg2 cfg3 cfg4 cfg5 cfg5r; do python make_golden.py $s & done
# ---------------------------------------------------------------------------
W_SEED, SK_SEED = 7, 8          # bench.py CFG
ROW_SAMPLE_SEED = 99


def _row_sample(N, k=256):
    return np.sort(np.random.default_rng(ROW_SAMPLE_SEED).choice(N, size=k, replace=False))


def _workloads():
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from paper_2405_10923_b200 import workloads
    return workloads


def _factor_summary(W, F, rows):
    """Small outputs of a full-size factorization: the sketch-space factors,
    scalars, U checksums and sampled rows, sketch_q (Psi Q), sampled rows of Q
    and the reference diagnostics (linalg.py:151-197)."""
    Q = thin_q(F)
    fro, mx, _ = factorization_errors(W, Q, F.R)
    PQ = F.psi.apply(Q)
    return dict(R=F.R, S=F.S, T=F.T, sigmas=F.sigmas, rhos=F.rhos, betas=F.betas,
                U_colnorm=np.linalg.norm(F.U, axis=0), U_head=F.U[:F.U.shape[1] + 64], rows=rows,
                U_rows=F.U[rows], Q_rows=Q[rows], SQ=sketch_q(F), PsiQ=PQ,
                cond_q=cond_number(Q), orth=orthogonality_error(PQ),
                orth_sq=orthogonality_error(sketch_q(F)), fro=fro, maxcol=mx)


def cfg2_case():
    """Config 2 at full size: rhqr_left of the 2^20 x 128 ill-conditioned W
    (sigma = logspace(0,-15)), SRHT ell = 256 (rhqr.py:254-267), plus the
    reference cond_number of W itself (the drop-in check for linalg.py:151)."""
    wl = _workloads()
    N, m, ell = 1 << 20, 128, 256
    W = wl.illcond_w(N, m, W_SEED)
    F = rhqr_left(W, SRHTSketch(ell, N - m, SK_SEED))
    rows = _row_sample(N)
    out = _factor_summary(W, F, rows)
    # W comes out of LAPACK QRs, whose last bits depend on the host CPU's
    # BLAS kernels: sampled rows + column norms pin it to rounding level
    out.update(W_rows=W[rows], W_colnorm=np.linalg.norm(W, axis=0))
    save("cfg2_rhqr_left_full", W_sha=np.array(sha(W)), N=N, m=m, ell=ell, w_seed=W_SEED,
         sk_seed=SK_SEED, cond_w=cond_number(W), **out)


def cfg2_spread_case():
    """How much of config 2's output is defined at all: the REFERENCE re-run
    on W perturbed by one unit roundoff per entry (W * (1 + u r), r uniform
    in [-1, 1], two seeds).  The spread of cond(Q), R and Psi Q over these
    runs is the parity bar's floor for any implementation."""
    wl = _workloads()
    N, m, ell = 1 << 20, 128, 256
    W = wl.illcond_w(N, m, W_SEED)
    out = {}
    for i, ps in enumerate((101, 102)):
        r = np.random.default_rng(ps).uniform(-1.0, 1.0, W.shape)
        Wp = W * (1.0 + 2.0 ** -53 * r)
        F = rhqr_left(Wp, SRHTSketch(ell, N - m, SK_SEED))
        Q = thin_q(F)
        out[f"cond_q_{i}"] = cond_number(Q)
        out[f"R_{i}"] = F.R
        out[f"SQ_{i}"] = sketch_q(F)
        out[f"sigmas_{i}"] = F.sigmas
    save("cfg2_perturbation_spread", **out)


def cfg3_case():
    """Config 3 at full size: rec_rhqr of gen_cmatrix(2^22, 64) with the
    Gaussian ell = 256 sketch regenerated per apply (rhqr.py:368-395,
    sketching.py:100-125)."""
    N, m, ell = 1 << 22, 64, 256
    W = gen_cmatrix(N, m)
    F = rec_rhqr(W, GaussianSketch(ell, N - m, SK_SEED))
    out = _factor_summary(W, F, _row_sample(N))
    save("cfg3_rec_rhqr_full", W_sha=np.array(sha(W)), N=N, m=m, ell=ell, sk_seed=SK_SEED, **out)


def cfg3_spread_case():
    """Config 3's own sensitivity: the REFERENCE rec_rhqr re-run on W
    perturbed by one unit roundoff per entry (two seeds), as for config 2."""
    N, m, ell = 1 << 22, 64, 256
    W = gen_cmatrix(N, m)
    rows = _row_sample(N)
    out = {}
    for i, ps in enumerate((101, 102)):
        r = np.random.default_rng(ps).uniform(-1.0, 1.0, W.shape)
        Wp = W * (1.0 + 2.0 ** -53 * r)
        del r
        F = rec_rhqr(Wp, GaussianSketch(ell, N - m, SK_SEED))
        out[f"R_{i}"], out[f"S_{i}"], out[f"T_{i}"] = F.R, F.S, F.T
        out[f"SQ_{i}"] = sketch_q(F)
        out[f"U_rows_{i}"] = F.U[rows]
        out[f"cond_q_{i}"] = cond_number(thin_q(F))
    save("cfg3_perturbation_spread", **out)


class _SplitKGaussian:
    """The reference's own Gaussian operator (identical G rows, from
    GaussianSketch._rows) applied with another summation order along n: the
    product is formed as the sum of `parts` K-slabs, each a BLAS dgemm.
    Passing it to the unmodified rec_rhqr measures how much of config 3's
    output is defined by the sketch GEMM's rounding (its apply() is the only
    thing that differs)."""

    kind = "gauss"

    def __init__(self, ell, n, seed, parts):
        self.ell, self.n, self.seed, self.parts = ell, n, seed, parts
        self._g = GaussianSketch(ell, n, seed)

    @property
    def shape(self):
        return (self.ell, self.n)

    def apply(self, X, dtype=np.float64):
        X = np.asarray(X, dtype=np.float64)
        one = X.ndim == 1
        X2 = X.reshape(-1, 1) if one else X
        step = max(1, (1 << 23) // self.n)
        Y = np.zeros((self.ell, X2.shape[1]))
        cuts = np.linspace(0, self.n, self.parts + 1).astype(np.int64)
        for i0 in range(0, self.ell, step):
            i1 = min(i0 + step, self.ell)
            G = self._g._rows(i0, i1)
            acc = np.zeros((i1 - i0, X2.shape[1]))
            for a, b in zip(cuts[:-1], cuts[1:]):
                acc += G[:, a:b] @ X2[a:b]
            Y[i0:i1] = acc
        return Y[:, 0] if one else Y


def cfg3_sum_order_spread_case():
    """Config 3 with the sketch GEMM summed in 2 and in 16 K-slabs (same G,
    same reference rec_rhqr): the reference's own sensitivity to the GEMM's
    summation order, the bar for any other valid order (the DMMA split-K)."""
    N, m, ell = 1 << 22, 64, 256
    W = gen_cmatrix(N, m)
    rows = _row_sample(N)
    out = {}
    for i, parts in enumerate((2, 16)):
        F = rec_rhqr(W, _SplitKGaussian(ell, N - m, SK_SEED, parts))
        out[f"parts_{i}"] = parts
        out[f"R_{i}"], out[f"S_{i}"], out[f"T_{i}"] = F.R, F.S, F.T
        out[f"SQ_{i}"] = sketch_q(F)
        out[f"U_rows_{i}"] = F.U[rows]
    save("cfg3_sum_order_spread", **out)


def cfg4_case():
    """Config 4 shape at reduced rows: bf16 storage / fp64 sketch space
    (bf16 tag injected at runtime), 2^18 x 256 with column scales
    logspace(0,-8), SRHT ell = 512 (precision.py:104-109)."""
    import ml_dtypes
    if "bf16" not in P.PRECISIONS:
        P.PRECISIONS = P.PRECISIONS + ("bf16",)
        P.DTYPES["bf16"] = ml_dtypes.bfloat16
        P.UNIT_ROUNDOFF["bf16"] = 2.0 ** -8
    wl = _workloads()
    N, m, ell = 1 << 18, 256, 512
    W = wl.scaled_gaussian_w(N, m, W_SEED)
    pol = P.PrecisionPolicy(high="double", low="bf16")
    F = rhqr_left(W, SRHTSketch(ell, N - m, SK_SEED), policy=pol)
    Wb = P.round_to(W, "bf16")  # the storage-rounded W the factors describe
    out = _factor_summary(Wb, F, _row_sample(N))
    # size: the leading 64 columns of Psi Q are what the parity bar reads
    out["SQ"], out["PsiQ"] = out["SQ"][:, :64].copy(), out["PsiQ"][:, :64].copy()
    out.pop("U_head")
    save("cfg4_rhqr_left_bf16_2p18", W_sha=np.array(sha(W)), N=N, m=m, ell=ell, w_seed=W_SEED,
         sk_seed=SK_SEED, **out)


def _cfg5_problem():
    import scipy.sparse
    wl = _workloads()
    k = 2048
    ip, ix, dv = wl.convection_diffusion_csr(k)
    N = k * k
    A = scipy.sparse.csr_matrix((dv, ix, ip), shape=(N, N))
    b = np.random.default_rng(11).standard_normal(N)
    return A, b, N, sha(ip) + sha(ix) + sha(dv)


def cfg5_case():
    """Config 5 at full size: one RHQR-GMRES(200) cycle on the 2048^2
    convection-diffusion CSR, SRHT ell = 400 over N - 201 coordinates
    (krylov.py:82-222).  The Arnoldi bundle is captured by wrapping
    krylov.rhqr_arnoldi at runtime (the reference source is not edited)."""
    from sketchqr import krylov as K
    A, b, N, csr_sha = _cfg5_problem()
    m, ell = 200, 400
    cap = {}
    orig = K.rhqr_arnoldi

    def spy(*a, **kw):
        cap["b"] = orig(*a, **kw)
        return cap["b"]
    K.rhqr_arnoldi = spy
    try:
        x, hist = K.rhqr_gmres(A, b, None, m, SRHTSketch(ell, N - m - 1, SK_SEED))
    finally:
        K.rhqr_arnoldi = orig
    bun = cap["b"]
    rows = _row_sample(N)
    save("cfg5_gmres200_full", csr_sha=np.array(csr_sha), b_sha=np.array(sha(b)), N=N, m=m, ell=ell,
         sk_seed=SK_SEED, hist=hist, H=bun.H, beta=bun.beta, S=bun.S, T=bun.T,
         U_colnorm=np.linalg.norm(bun.U, axis=0), U_head=bun.U[:m + 65], rows=rows, U_rows=bun.U[rows],
         x_rows=x[rows], x_norm=np.linalg.norm(x), x_head=x[:256], x_tail=x[-256:],
         true_resid=np.linalg.norm(b - A @ x) / np.linalg.norm(b))


def cfg5_restart_case():
    """Config 5 problem, the restarted driver's semantics at full size: two
    GMRES(10) cycles x1 = gmres(A, b, 0), x2 = gmres(A, b, x1) with the same
    Omega (SRHT 400 over N - 11 coordinates) — what rhqr_gmres_restarted runs."""
    A, b, N, csr_sha = _cfg5_problem()
    m, ell = 10, 400
    om = SRHTSketch(ell, N - m - 1, SK_SEED)
    x1, h1 = rhqr_gmres(A, b, None, m, om)
    x2, h2 = rhqr_gmres(A, b, x1, m, om)
    rows = _row_sample(N)
    save("cfg5_gmres10_restart", csr_sha=np.array(csr_sha), N=N, m=m, ell=ell, sk_seed=SK_SEED,
         hist1=h1, hist2=h2, rows=rows, x1_rows=x1[rows], x2_rows=x2[rows],
         x1_norm=np.linalg.norm(x1), x2_norm=np.linalg.norm(x2),
         true_resid2=np.linalg.norm(b - A @ x2) / np.linalg.norm(b))


SECTIONS = dict(srht=srht_cases, gauss=gauss_cases, rh_vector=rh_vector_cases, rhqr=rhqr_cases,
                mixed=mixed_cases, rec=rec_cases, krylov=krylov_cases, apply_compact=apply_compact_cases,
                block=block_cases, experiments=experiment_cases, trim=trim_cases)
# the config-scale sections run only when named (minutes of CPU each)
BIG_SECTIONS = dict(cfg2=cfg2_case, cfg2spread=cfg2_spread_case, cfg3spread=cfg3_spread_case, cfg3sum=cfg3_sum_order_spread_case, cfg3=cfg3_case, cfg4=cfg4_case, cfg5=cfg5_case,
                    cfg5r=cfg5_restart_case)

if __name__ == "__main__":
    # no arguments: every section; otherwise only the named ones
    for name in (sys.argv[1:] or list(SECTIONS)):
        {**SECTIONS, **BIG_SECTIONS}[name]()
