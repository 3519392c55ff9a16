"""Differential fuzzer: the unmodified reference (baseline/_ref, CPU) against this
package (B200) on random shapes biased to the edges of the kernels' geometry
(N - m around powers of two and tile multiples, m = 1, ell = m, ell = n_pad,
ragged tails), both scalings, every sketch kind and storage format.

    python scripts/fuzz_diff.py [--seconds 240] [--seed 0]

Prints one line per mismatch (exception kind/message or relative error above
the bar) and a summary; exit code 1 if any case disagreed.  Needs baseline/_ref
(build() installs it) and a GPU.
"""
import argparse
import os
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import sketchqr as R  # noqa: E402
from sketchqr import trim as Rtrim  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import trim as Ptrim  # noqa: E402

BAR = 1e-10

# bf16 storage (config 4's format): the reference has no such tag; it is injected at runtime exactly as
# tests/golden/make_golden.py does, the reference's source untouched
import ml_dtypes  # noqa: E402
from sketchqr import precision as _RP  # noqa: E402

if "bf16" not in _RP.PRECISIONS:
    _RP.PRECISIONS = _RP.PRECISIONS + ("bf16",)
    _RP.DTYPES["bf16"] = ml_dtypes.bfloat16
    _RP.UNIT_ROUNDOFF["bf16"] = 2.0 ** -8


def policies(tag):
    if tag == "bf16":
        return R.PrecisionPolicy(high="double", low="bf16"), P.PrecisionPolicy("double", "bf16")
    return R.policy_from_tag(tag), P.policy_from_tag(tag)


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return np.inf
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d > 0 else float(np.linalg.norm(a - b))


class OutOfScope(Exception):
    pass


def outcome(fn):
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return ("ok", fn())
    except NotImplementedError as e:
        if "outside the B200 hot path" in str(e):
            raise OutOfScope(str(e)) from None
        return (type(e).__name__, str(e))
    except Exception as e:  # noqa: BLE001
        return (type(e).__name__, str(e))


def pick_n(rng):
    k = int(rng.integers(1, 17))
    base = 1 << k
    choice = rng.integers(0, 6)
    if choice == 0:
        return max(1, base - 1)
    if choice == 1:
        return base
    if choice == 2:
        return base + 1
    if choice == 3:
        return int(rng.integers(1, 300))
    if choice == 4:
        return 4096 * int(rng.integers(1, 6)) + int(rng.integers(-2, 3))
    return int(rng.integers(1, 70000))


def sketches(kind, ell, n, seed):
    if kind == "srht":
        return R.SRHTSketch(ell, n, seed), P.SRHTSketch(ell, n, seed)
    if kind == "gauss":
        return R.GaussianSketch(ell, n, seed), P.GaussianSketch(ell, n, seed)
    return R.IdentitySketch(n), P.IdentitySketch(n)


def compare_factors(tag, Fr, Fp, names, bar):
    bad = []
    for k in names:
        e = rel(getattr(Fp, k), getattr(Fr, k))
        if not e <= bar:
            bad.append(f"{k} {e:.2e}")
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--big", action="store_true",
                    help="N - m in [2^16, 2^21] (ragged, around powers of two), few columns: the multi-tile, "
                         "TMA and padded-tile paths; left / rec / srht / right only")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    n_cases = n_bad = 0
    per = {}
    while time.time() < t_end:
        op = str(rng.choice(["left", "left", "rec", "right", "block", "srht", "gauss", "gmres", "trim", "compact", "lsq",
                             "arnoldi", "diag", "experiment"]))
        m = int(rng.choice([1, 2, 3, 5, 8, 16, 33, 64, 100]))
        n = pick_n(rng)
        kind = str(rng.choice(["srht", "srht", "gauss", "identity"]))
        if op in ("gauss",):
            kind = "gauss"
        if op == "srht":
            kind = "srht"
        if args.big:
            op = str(rng.choice(["left", "left", "rec", "srht", "right", "gmres_big"]))
            m = int(rng.choice([1, 2, 5, 8, 16]))
            k = int(rng.integers(16, 21))
            n = int(rng.choice([(1 << k) - 1, 1 << k, (1 << k) + 1, (1 << k) + 4097, int(rng.integers(1 << 16, 1 << 21)),
                                4096 * int(rng.integers(17, 300)) - 1]))
            kind = str(rng.choice(["srht", "srht", "srht", "gauss"]))
            if op == "srht":
                kind = "srht"
            if op == "gmres_big":
                kind = "srht"
        n_pad = 1 << max(0, (n - 1).bit_length())
        ell = int(rng.choice([m, m + 1, 2 * m, 4 * m, min(n_pad, 8 * m)]))
        if args.big:
            ell = int(rng.choice([max(m, 8), 4 * m, 64, 200, 256, 400, 512, 600]))
        if kind == "gauss" and ell * n > 3e7:
            n = max(1, int(3e7 // ell))
        if kind == "identity":
            n = min(n, 600)
            ell = n
        scaling = str(rng.choice(["sqrt2", "unit"]))
        tag = str(rng.choice(["double", "double", "double", "single", "mixed", "bf16"]))
        seed = int(rng.integers(0, 1 << 30))
        N = n + m
        desc = f"{op} N={N} m={m} n={n} ell={ell} {kind} {scaling} {tag} seed={seed}"
        n_cases += 1
        per[op] = per.get(op, 0) + 1
        wr = np.random.default_rng(seed)
        bar = BAR if tag == "double" else None
        try:
            if op in ("srht", "gauss"):
                k = int(rng.choice([1, 2, 7]))
                orr = outcome(lambda: sketches(kind, ell, n, seed))
                if orr[0] != "ok":
                    op2 = outcome(lambda: (P.SRHTSketch if kind == "srht" else P.GaussianSketch)(ell, n, seed))
                    if op2[0] != orr[0]:
                        n_bad += 1
                        print("MISMATCH ctor", desc, orr[0], "vs", op2[0])
                    continue
                omr, omp = orr[1]
                X = wr.standard_normal((n, k)) if k > 1 else wr.standard_normal(n)
                dt = {"double": np.float64, "single": np.float32, "mixed": np.float16, "bf16": ml_dtypes.bfloat16}[tag]
                a, b = outcome(lambda: omr.apply(X, dtype=dt)), outcome(lambda: omp.apply(X, dtype=dt))
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    if kind == "srht":
                        good = np.array_equal(np.asarray(a[1]), np.asarray(b[1]), equal_nan=True)
                    else:
                        good = rel(b[1], a[1]) <= (1e-12 if tag == "double" else 5e-3)
                    if not good:
                        n_bad += 1
                        print("MISMATCH values", desc, rel(b[1], a[1]))
                continue
            if op == "diag":
                # the stability diagnostics on matrices of every conditioning (linalg.py:151-197)
                k = min(m, 40)
                Nd = min(N, 20000)
                if Nd < k:
                    continue
                M = wr.standard_normal((Nd, k)) * np.logspace(0, -float(rng.choice([0, 3, 8, 14])), k)[None, :]
                Q, Rq = np.linalg.qr(M)
                ca, cb = R.cond_number(M), P.cond_number(M)
                oa, ob = R.orthogonality_error(Q), P.orthogonality_error(Q)
                fa, fb = R.factorization_errors(M, Q, Rq), P.factorization_errors(M, Q, Rq)
                bad = []
                if not abs(cb - ca) <= 2e-2 * ca * max(1.0, ca * 2.2e-16 * 100):
                    bad.append(f"cond {ca:.6e} vs {cb:.6e}")
                if not abs(ob - oa) <= 1e-14 + 0.5 * oa:
                    bad.append(f"orth {oa:.3e} vs {ob:.3e}")
                if not (abs(fb.fro_rel_err - fa.fro_rel_err) <= 1e-15 + 0.5 * fa.fro_rel_err
                        and abs(fb.max_col_rel_err - fa.max_col_rel_err) <= 1e-15 + 0.5 * fa.max_col_rel_err
                        and tuple(fb.flagged_columns) == tuple(fa.flagged_columns)):
                    bad.append(f"errors {fa} vs {fb}")
                if bad:
                    n_bad += 1
                    print("MISMATCH diag", desc, bad)
                continue
            if op == "experiment":
                Ne, me = min(N, 6000), min(max(m, 4), 24)
                if Ne < 3 * me + 8:
                    continue
                We = R.gen_cmatrix(Ne, me) if rng.random() < 0.5 else wr.standard_normal((Ne, me))
                algo = str(rng.choice(["rhqr-left", "rhqr-right", "rhqr-block", "rec-rhqr", "trim-left", "hqr"]))
                kw = dict(algo=algo, sketch="srht" if kind == "identity" else kind, ell=0, seed=seed % 1000,
                          precision=str(rng.choice(["double", "single"])), every=int(rng.choice([3, 8])),
                          scaling=scaling, block_size=int(rng.choice([2, 5])))
                a = outcome(lambda: R.run_factor_experiment(We, R.ExperimentConfig(**kw)))
                b = outcome(lambda: P.run_factor_experiment(We, P.ExperimentConfig(**kw)))
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH experiment", desc, kw, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    ra, rb = a[1], b[1]
                    okrows = len(ra) == len(rb)
                    for x, y in zip(ra, rb):
                        okrows = okrows and x.j == y.j and x.status == y.status
                        if x.status == "ok" and np.isfinite(x.cond_q) and x.cond_q < 1e3 and kw["precision"] == "double":
                            okrows = okrows and abs(y.cond_q - x.cond_q) <= 1e-2 * x.cond_q
                            okrows = okrows and abs(y.cond_sq - x.cond_sq) <= 1e-2 * x.cond_sq
                            okrows = okrows and y.fro_rel_err <= max(1e-13, 10 * x.fro_rel_err)
                            okrows = okrows and y.orth_err <= max(1e-12, 10 * x.orth_err)
                    if not okrows:
                        n_bad += 1
                        print("MISMATCH experiment rows", desc, kw, [(x.j, x.status, x.cond_q) for x in ra],
                              [(y.j, y.status, y.cond_q) for y in rb])
                continue
            W = wr.standard_normal((N, m))
            if rng.random() < 0.1 and m > 1:
                W[:, m - 1] = 0.0  # breakdown at the last column
            lay = int(rng.integers(0, 4))  # host layouts a caller may pass: C, Fortran, strided views
            if lay == 1:
                W = np.asfortranarray(W)
            elif lay == 2:
                big = np.zeros((N, 2 * m))
                big[:, ::2] = W
                W = big[:, ::2]
            elif lay == 3:
                big = np.zeros((N + 3, m + 2))
                big[2:N + 2, 1:m + 1] = W
                W = big[2:N + 2, 1:m + 1]
            desc += f" lay={lay}"
            pol_r, pol_p = policies(tag)
            sk = outcome(lambda: sketches(kind, ell, n, seed))
            if sk[0] != "ok":
                sp = outcome(lambda: (P.SRHTSketch if kind == "srht" else P.GaussianSketch)(ell, n, seed))
                if sp[0] != sk[0]:
                    n_bad += 1
                    print("MISMATCH ctor", desc, sk, "vs", sp[0])
                continue
            omr, omp = sk[1]
            if op == "left":
                a = outcome(lambda: R.rhqr_left(W, omr, scaling=scaling, policy=pol_r))
                b = outcome(lambda: P.rhqr_left(W, omp, scaling=scaling, policy=pol_p))
                names = ("R", "S", "T", "U", "sigmas", "rhos", "betas")
            elif op == "right":
                a = outcome(lambda: R.rhqr_right(W, omr, scaling=scaling, policy=pol_r))
                b = outcome(lambda: P.rhqr_right(W, omp, scaling=scaling, policy=pol_p))
                names = ("R", "S", "T", "U")
            elif op == "rec":
                a = outcome(lambda: R.rec_rhqr(W, omr, scaling=scaling, policy=pol_r))
                b = outcome(lambda: P.rec_rhqr(W, omp, scaling=scaling, policy=pol_p))
                names = ("R", "S", "T", "U")
            elif op == "block":
                bs = int(rng.choice([1, 2, 3, 8]))
                a = outcome(lambda: R.rhqr_block(W, omr, block_size=bs, scaling=scaling, policy=pol_r).stacked())
                b = outcome(lambda: P.rhqr_block(W, omp, block_size=bs, scaling=scaling, policy=pol_p).stacked())
                names = ("R", "S", "T", "U")
            elif op == "compact":
                Fr = outcome(lambda: R.rhqr_left(W, omr, scaling=scaling))
                Fp = outcome(lambda: P.rhqr_left(W, omp, scaling=scaling))
                if Fr[0] != "ok" or Fp[0] != "ok":
                    if Fr[0] != Fp[0]:
                        n_bad += 1
                        print("MISMATCH", desc, Fr[0], "vs", Fp[0])
                    continue
                X = wr.standard_normal((N, 3))
                tt = bool(rng.integers(0, 2))
                ar = R.rhqr.apply_reflectors_compact(Fr[1].U, Fr[1].S, Fr[1].T, X, Fr[1].psi, transpose_t=tt)
                bp = P.apply_reflectors_compact(Fp[1].U, Fp[1].S, Fp[1].T, X, Fp[1].psi, transpose_t=tt)
                e = max(rel(bp, ar), rel(P.thin_q(Fp[1]), R.thin_q(Fr[1])), rel(P.sketch_q(Fp[1]), R.sketch_q(Fr[1])))
                if not e <= 1e-9:
                    n_bad += 1
                    print("MISMATCH compact/thin_q", desc, f"{e:.2e}")
                continue
            elif op == "lsq":
                Fr = outcome(lambda: R.rhqr_left(W, omr, scaling=scaling))
                Fp = outcome(lambda: P.rhqr_left(W, omp, scaling=scaling))
                if Fr[0] != "ok" or Fp[0] != "ok":
                    if Fr[0] != Fp[0]:
                        n_bad += 1
                        print("MISMATCH", desc, Fr[0], "vs", Fp[0])
                    continue
                bb = wr.standard_normal(N)
                e = rel(P.lsq_via_implicit_q(Fp[1], bb), R.lsq_via_implicit_q(Fr[1], bb))
                if not e <= 1e-8:
                    n_bad += 1
                    print("MISMATCH lsq", desc, f"{e:.2e}")
                continue
            elif op == "trim":
                if kind == "identity":
                    omr, omp = R.IdentitySketch(N), P.IdentitySketch(N)
                else:
                    ellt = max(2, ell // 2, m // 3)  # far below m / 3 the reference itself moves by O(1) under a 1-ulp change of W
                    omr, omp = sketches(kind, ellt, N, seed)
                left = bool(rng.integers(0, 2))
                fr = Rtrim.trim_rhqr_left if left else Rtrim.trim_rhqr_right
                fp = Ptrim.trim_rhqr_left if left else Ptrim.trim_rhqr_right
                a = outcome(lambda: fr(W, omr, scaling=scaling, policy=pol_r))
                b = outcome(lambda: fp(W, omp, scaling=scaling, policy=pol_p))
                names = ("R", "U", "S", "T", "T_tilde", "L")
                if bar:
                    bar = 1e-8
            elif op == "gmres_big":
                import scipy.sparse as sp
                Ng = N
                mg = int(rng.choice([3, 8, 20]))
                A = sp.diags([np.full(Ng - 1, -1.0), np.linspace(2.0, 3.0, Ng), np.full(Ng - 1, -0.5)], [-1, 0, 1],
                             format="csr")
                bb = wr.standard_normal(Ng)
                ng = Ng - mg - 1
                npg = 1 << max(0, (ng - 1).bit_length())
                ellg = min(max(ell, 2 * (mg + 1)), npg)
                sg = sketches("srht", ellg, ng, seed)
                a = outcome(lambda: R.rhqr_gmres(A, bb, None, mg, sg[0], scaling=scaling))
                b = outcome(lambda: P.rhqr_gmres(A, bb, None, mg, sg[1], scaling=scaling))
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    e = max(rel(b[1][0], a[1][0]), rel(b[1][1], a[1][1]))
                    if not e <= 1e-9:
                        n_bad += 1
                        print("MISMATCH gmres_big", desc, f"mg={mg} {e:.2e}")
                continue
            elif op == "arnoldi":
                import scipy.sparse as sp
                Ng = min(N, 5000)
                mg = min(m, 30, Ng - 2)
                if mg < 1:
                    continue
                which = int(rng.integers(0, 3))
                if which == 0:
                    A = np.diag(np.linspace(1.0, 4.0, Ng)) + 0.05 * wr.standard_normal((Ng, Ng)) / np.sqrt(Ng)
                    Ar, Ap = A, A
                elif which == 1:
                    A = sp.random(Ng, Ng, density=min(1.0, 6.0 / Ng), random_state=seed % 9973, format="csr") + sp.eye(Ng, format="csr") * 3.0
                    Ar, Ap = A, A
                else:
                    d = np.linspace(1.0, 2.0, Ng)
                    Ar = Ap = (lambda v, d=d: d * v)  # a callable operator (krylov.py:28-35)
                bb = wr.standard_normal(Ng)
                x0 = wr.standard_normal(Ng) if rng.random() < 0.3 else None
                ng = Ng - mg - 1
                npg = 1 << max(0, (ng - 1).bit_length())
                ellg = min(max(ell, mg + 1), npg)
                sg = outcome(lambda: sketches("srht" if kind == "identity" else kind, ellg, ng, seed))
                if sg[0] != "ok":
                    continue
                sq = bool(rng.integers(0, 2))
                a = outcome(lambda: R.rhqr_arnoldi(Ar, bb, x0, mg, sg[1][0], scaling=scaling, store_q=sq))
                b = outcome(lambda: P.rhqr_arnoldi(Ap, bb, x0, mg, sg[1][1], scaling=scaling, store_q=sq))
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    Ba, Bb = a[1], b[1]
                    e = max(rel(Bb.H, Ba.H), rel(Bb.S, Ba.S), rel(Bb.T, Ba.T), rel(Bb.U, Ba.U), abs(Bb.beta - Ba.beta) / abs(Ba.beta))
                    if sq:
                        e = max(e, rel(Bb.Q_cols, Ba.Q_cols))
                    if Ba.breakdown != Bb.breakdown or not e <= 1e-9:
                        n_bad += 1
                        print("MISMATCH arnoldi", desc, f"mg={mg} op={which} {e:.2e} breakdown {Ba.breakdown} vs {Bb.breakdown}")
                continue
            elif op == "gmres":
                Ng = min(N, 3000)
                mg = min(m, 24, Ng - 2)
                if mg < 1:
                    continue
                A = np.diag(np.linspace(1.0, 4.0, Ng)) + 0.05 * wr.standard_normal((Ng, Ng)) / np.sqrt(Ng)
                bb = wr.standard_normal(Ng)
                ng = Ng - mg - 1
                npg = 1 << max(0, (ng - 1).bit_length())
                ellg = min(max(ell, mg + 1), npg)
                sg = outcome(lambda: sketches("srht" if kind == "identity" else kind, ellg, ng, seed))
                if sg[0] != "ok":
                    continue
                a = outcome(lambda: R.rhqr_gmres(A, bb, None, mg, sg[1][0], scaling=scaling))
                b = outcome(lambda: P.rhqr_gmres(A, bb, None, mg, sg[1][1], scaling=scaling))
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    e = max(rel(b[1][0], a[1][0]), rel(b[1][1], a[1][1]))
                    if not e <= 1e-8:
                        n_bad += 1
                        print("MISMATCH gmres", desc, f"mg={mg} {e:.2e}")
                continue
            if a[0] != b[0]:
                n_bad += 1
                print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
            elif a[0] != "ok":
                if a[1] != b[1]:
                    print("note: messages differ", desc, "|", a[1], "|", b[1])
            elif bar:
                bad = compare_factors(tag, a[1], b[1], names, bar)
                if bad:
                    n_bad += 1
                    print("MISMATCH values", desc, bad)
            else:
                # low-precision storage: R within a few storage roundoffs times sqrt(N)
                u = {"single": 2.0 ** -24, "mixed": 2.0 ** -11, "bf16": 2.0 ** -8}[tag]
                e = rel(b[1].R, a[1].R)
                if not np.isfinite(np.asarray(a[1].R)).all():
                    continue  # the reference overflowed its half-precision transform
                if not e <= (400 if op == "trim" else 40) * u * np.sqrt(m):  # trim: ell < m sketches amplify
                    n_bad += 1
                    print("MISMATCH lowprec R", desc, f"{e:.2e} (u={u:.1e})")
        except OutOfScope:
            n_cases -= 1
            per[op] -= 1
        except Exception as exc:  # noqa: BLE001
            n_bad += 1
            print("HARNESS ERROR", desc, type(exc).__name__, exc)
    print(f"fuzz_diff: {n_cases} cases, {n_bad} disagreements; per op {per}")
    return 1 if n_bad else 0


if __name__ == "__main__":
    sys.exit(main())
