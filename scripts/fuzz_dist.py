"""Row-partition fuzzer: the multi-GPU algorithm on P virtual ranks of ONE B200
(the same kernels, partition and rank-order combine a P-GPU run uses; the
exchange is a device copy or the peer-memory mailboxes) against the single-GPU
factorization on random shapes — ragged last ranks, ranks that own only
padding, n_pad / P down to one SRHT tile, every storage format.  The sketches,
hence S, T, R, H and (for the sweeps) U, must be BITWISE the single-GPU ones.

    python scripts/fuzz_dist.py [--seconds 240] [--seed 0]

The bitwise twin of the partitioned sweep is the launch chain, so the
single-GPU side runs with SQB_PERSIST=0.
"""
import argparse
import os
import sys
import time
import warnings

import numpy as np

os.environ["SQB_PERSIST"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import dist as D  # noqa: E402


def rel(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / d) if d > 0 else float(np.linalg.norm(a - b))


def outcome(fn):
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return ("ok", fn())
    except Exception as e:  # noqa: BLE001
        return (type(e).__name__, str(e))


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args(argv)
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    n_cases = n_bad = n_skip = 0
    per = {}
    kinds = {}
    while time.time() < t_end:
        op = str(rng.choice(["left", "left", "rec", "arnoldi"]))
        nranks = int(rng.choice([1, 2, 4, 8]))
        tag = str(rng.choice(["double", "double", "single", "half", "bf16"]))
        tile = 1 << D.TILE_LOG[tag]
        m = int(rng.choice([1, 2, 5, 8, 16, 24, 33, 64]))
        # n_pad from nranks tiles up to 2^19; n anywhere in (n_pad/2, n_pad], biased to the partition edges
        kmin = (nranks * tile).bit_length() - 1
        n_pad = 1 << int(rng.integers(kmin, 20))
        span = n_pad // nranks
        choice = int(rng.integers(0, 6))
        if choice == 0:
            n = n_pad
        elif choice == 1:
            n = n_pad // 2 + 1
        elif choice == 2:
            n = int(rng.integers(1, nranks + 1)) * span - int(rng.integers(0, 3))  # the last ranks own only padding
        elif choice == 3:
            n = int(rng.integers(1, nranks + 1)) * span - span + 1 + int(rng.integers(0, 2))  # a rank with 1-2 rows
        elif choice == 4:
            n = n_pad // 2 + tile * int(rng.integers(0, max(1, n_pad // (2 * tile)))) + int(rng.integers(-1, 2))
        else:
            n = int(rng.integers(n_pad // 2 + 1, n_pad + 1))
        n = int(min(max(n, n_pad // 2 + 1), n_pad))
        ell = int(rng.choice([max(m, 2), 2 * m + 1, 4 * m, 128, 256]))
        ell = min(max(ell, m), n_pad, 512)
        if ell < m:
            continue
        scaling = str(rng.choice(["sqrt2", "unit"]))
        exchange = str(rng.choice(["copy", "p2p"]))
        seed = int(rng.integers(0, 1 << 30))
        pol = P.PrecisionPolicy("double", tag)
        wr = np.random.default_rng(seed)
        desc = f"{op} P={nranks} n={n} n_pad={n_pad} m={m} ell={ell} {tag} {scaling} {exchange} seed={seed}"
        n_cases += 1
        per[op] = per.get(op, 0) + 1
        if args.verbose:
            print("case", desc, flush=True)
        try:
            if op in ("left", "rec"):
                N = n + m
                if op == "rec" and m < 2:
                    m = 2
                    N = n + m
                    ell = max(ell, m)
                W = wr.standard_normal((N, m)) if op == "left" else P.gen_cmatrix(N, m) + 1e-3 * wr.standard_normal((N, m))
                if rng.random() < 0.08 and m > 1:
                    W[:, m - 1] = 0.0
                om = P.SRHTSketch(ell, n, seed % 9973)
                f1 = P.rhqr_left if op == "left" else P.rec_rhqr
                fv = D.rhqr_left_virtual if op == "left" else D.rec_rhqr_virtual
                a = outcome(lambda: f1(W, om, scaling=scaling, policy=pol))
                b = outcome(lambda: fv(W, om, nranks, scaling=scaling, policy=pol, exchange=exchange))
                kinds[(a[0], b[0])] = kinds.get((a[0], b[0]), 0) + 1
                if a[0] != "ok" and args.verbose:
                    print("  outcome", a[0], a[1][:200])
                if a[0] != b[0] or (a[0] != "ok" and a[1] != b[1]):
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    bad = [k for k in ("R", "S", "T", "sigmas", "rhos", "betas")
                           if not np.array_equal(getattr(b[1], k), getattr(a[1], k), equal_nan=True)]
                    if op == "left":
                        if not np.array_equal(b[1].U, a[1].U, equal_nan=True):
                            bad.append("U")
                    elif not rel(b[1].U, a[1].U) <= 1e-13:
                        bad.append(f"U {rel(b[1].U, a[1].U):.2e}")
                    if bad:
                        n_bad += 1
                        print("MISMATCH bits", desc, bad)
            else:
                import scipy.sparse as sp
                if tag in ("half", "bf16"):
                    n_cases -= 1
                    per[op] -= 1
                    continue
                mg = int(min(m, 20))
                Ng = n + mg + 1
                band = int(rng.choice([1, 3, 700]))
                A = sp.diags([np.full(Ng - band, -1.0), np.linspace(2.0, 3.0, Ng), np.full(Ng - band, -0.5)],
                             [-band, 0, band], format="csr")
                if rng.random() < 0.3:
                    nz = 2 * Ng  # scattered entries: the halo of a rank then reaches into every peer
                    A = (A + sp.coo_matrix((0.01 * wr.standard_normal(nz), (wr.integers(0, Ng, nz), wr.integers(0, Ng, nz))),
                                           shape=(Ng, Ng)).tocsr()).tocsr()
                    A.sum_duplicates()
                    A.sort_indices()
                bb = wr.standard_normal(Ng)
                om = P.SRHTSketch(min(max(ell, mg + 1), n_pad), n, seed % 9973)
                halo = bool(rng.integers(0, 2))
                a = outcome(lambda: P.rhqr_arnoldi(A, bb, None, mg, om, scaling=scaling, policy=pol))
                b = outcome(lambda: D.rhqr_arnoldi_virtual(A, bb, None, mg, om, nranks, scaling=scaling, policy=pol, halo=halo))
                kinds[(a[0], b[0])] = kinds.get((a[0], b[0]), 0) + 1
                if a[0] != "ok" and args.verbose:
                    print("  outcome", a[0], a[1][:200])
                if a[0] != b[0]:
                    n_bad += 1
                    print("MISMATCH", desc, a[0], a[1] if a[0] != "ok" else "", "vs", b[0], b[1] if b[0] != "ok" else "")
                elif a[0] == "ok":
                    bad = [k for k in ("H", "S", "T", "U") if not np.array_equal(getattr(b[1], k), getattr(a[1], k))]
                    if b[1].beta != a[1].beta or b[1].breakdown != a[1].breakdown:
                        bad.append("beta/breakdown")
                    if bad:
                        n_bad += 1
                        print("MISMATCH bits", desc, f"halo={halo} band={band}", bad)
        except Exception as exc:  # noqa: BLE001
            n_bad += 1
            print("HARNESS ERROR", desc, type(exc).__name__, exc)
    print(f"fuzz_dist: {n_cases} cases, {n_bad} disagreements; per op {per}; outcomes (single GPU, partitioned) {kinds}")
    return 1 if n_bad else 0


if __name__ == "__main__":
    sys.exit(main())
