"""Measure the GPU path against the reference goldens at the BASELINE config
shapes (tests/golden/cfg*.npz, written by tests/golden/make_golden.py running
the reference).  Prints one JSON object of relative discrepancies per config;
tests/test_gpu_configs.py asserts the bars.  Usage: python scripts/probe_config_parity.py [cfg2 cfg3 cfg4 cfg5 cfg5r]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden  # noqa: E402
import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb else 1.0))


def colrel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b, axis=0) / np.maximum(np.linalg.norm(b, axis=0), 1e-300)


def factor_report(F, g, W, lead):
    Q = P.thin_q(F)
    fro, mx, _ = P.factorization_errors(W, Q, F.R)
    SQ = P.sketch_q(F)
    PQ = F.psi.apply(Q)
    rows = g["rows"]
    out = dict(R=rel(F.R, g["R"]), S_lead=rel(F.S[:, :lead], g["S"][:, :lead]), S=rel(F.S, g["S"]),
               T_lead=rel(F.T[:lead, :lead], g["T"][:lead, :lead]), T=rel(F.T, g["T"]),
               SQ_lead=rel(SQ[:, :lead], g["SQ"][:, :lead]), SQ=rel(SQ[:, :g["SQ"].shape[1]], g["SQ"]),
               PsiQ_lead=rel(PQ[:, :lead], g["PsiQ"][:, :lead]) if "PsiQ" in g else None,
               U_rows_lead=rel(F.U[rows][:, :lead], g["U_rows"][:, :lead]),
               U_rows=rel(F.U[rows], g["U_rows"]),
               Q_rows_lead=rel(Q[rows][:, :lead], g["Q_rows"][:, :lead]),
               U_colnorm=rel(np.linalg.norm(F.U, axis=0), g["U_colnorm"]),
               rhos=rel(F.rhos, g["rhos"]), sigmas_equal=int((F.sigmas == g["sigmas"]).sum()),
               cond_q=P.cond_number(Q), cond_q_ref=float(g["cond_q"]),
               orth=P.orthogonality_error(PQ), orth_ref=float(g["orth"]),
               orth_sq=P.orthogonality_error(SQ), orth_sq_ref=float(g["orth_sq"]),
               fro=fro, fro_ref=float(g["fro"]), maxcol=mx, maxcol_ref=float(g["maxcol"]))
    out["cond_q_rel"] = abs(out["cond_q"] - out["cond_q_ref"]) / out["cond_q_ref"]
    c = colrel(SQ[:, :g["SQ"].shape[1]], g["SQ"])
    out["SQ_first_col_above_1e-10"] = int(np.argmax(c > 1e-10)) if (c > 1e-10).any() else None
    return out


def cfg2():
    g = golden("cfg2_rhqr_left_full")
    N, m = int(g["N"]), int(g["m"])
    W = workloads.illcond_w(N, m, int(g["w_seed"]))
    # QR-generated: equal to the reference's W up to rounding (host BLAS kernels)
    w_rows = rel(W[g["rows"]], g["W_rows"])
    assert w_rows < 1e-14, w_rows
    t = time.time()
    F = P.rhqr_left(W, P.SRHTSketch(int(g["ell"]), N - m, int(g["sk_seed"])))
    out = factor_report(F, g, W, 43)
    cw = P.cond_number(W)
    out.update(W_rows=w_rows, W_sha_equal=workloads.sha256(W) == str(g["W_sha"]), cond_w=cw, cond_w_ref=float(g["cond_w"]), cond_w_rel=abs(cw - float(g["cond_w"])) / float(g["cond_w"]),
               secs=time.time() - t)
    return out


def cfg3():
    g = golden("cfg3_rec_rhqr_full")
    N, m = int(g["N"]), int(g["m"])
    W = workloads.gen_cmatrix(N, m)
    assert workloads.sha256(W) == str(g["W_sha"])
    t = time.time()
    F = P.rec_rhqr(W, P.GaussianSketch(int(g["ell"]), N - m, int(g["sk_seed"])))
    out = factor_report(F, g, W, m)
    out["secs"] = time.time() - t
    return out


def cfg4():
    g = golden("cfg4_rhqr_left_bf16_2p18")
    N, m = int(g["N"]), int(g["m"])
    W = workloads.scaled_gaussian_w(N, m, int(g["w_seed"]))
    assert workloads.sha256(W) == str(g["W_sha"])
    F = P.rhqr_left(W, P.SRHTSketch(int(g["ell"]), N - m, int(g["sk_seed"])), policy=P.PrecisionPolicy("double", "bf16"))
    Wb = P.round_to(W, "bf16")
    out = factor_report(F, g, Wb, 64)
    out["colrel_R_diag"] = np.abs(np.diag(F.R) - np.diag(g["R"])).max() / np.abs(np.diag(g["R"])).max()
    return out


def _cfg5_problem(g):
    import scipy.sparse
    ip, ix, dv = workloads.convection_diffusion_csr(2048)
    N = 2048 * 2048
    assert workloads.sha256(ip) + workloads.sha256(ix) + workloads.sha256(dv) == str(g["csr_sha"])
    A = scipy.sparse.csr_matrix((dv, ix, ip), shape=(N, N))
    b = np.random.default_rng(11).standard_normal(N)
    return A, b, N


def cfg5():
    g = golden("cfg5_gmres200_full")
    A, b, N = _cfg5_problem(g)
    m, ell = int(g["m"]), int(g["ell"])
    om = P.SRHTSketch(ell, N - m - 1, int(g["sk_seed"]))
    t = time.time()
    bun = P.rhqr_arnoldi(A, b, None, m, om, store_q=False)
    x, hist = P.rhqr_gmres(A, b, None, m, om)
    rows = g["rows"]
    return dict(H=rel(bun.H, g["H"]), beta=abs(bun.beta - float(g["beta"])) / abs(float(g["beta"])),
                S=rel(bun.S, g["S"]), T=rel(bun.T, g["T"]), U_rows=rel(bun.U[rows], g["U_rows"]),
                U_colnorm=rel(np.linalg.norm(bun.U, axis=0), g["U_colnorm"]),
                hist=rel(hist, g["hist"]), hist_last_rel=abs(hist[-1] - g["hist"][-1]) / g["hist"][-1],
                x_rows=rel(x[rows], g["x_rows"]), x_norm=abs(np.linalg.norm(x) - float(g["x_norm"])) / float(g["x_norm"]),
                x_head=rel(x[:256], g["x_head"]),
                true_resid=float(np.linalg.norm(b - A @ x) / np.linalg.norm(b)), true_resid_ref=float(g["true_resid"]),
                secs=time.time() - t)


def cfg5r():
    g = golden("cfg5_gmres10_restart")
    A, b, N = _cfg5_problem(g)
    m, ell = int(g["m"]), int(g["ell"])
    om = P.SRHTSketch(ell, N - m - 1, int(g["sk_seed"]))
    x1, h1 = P.rhqr_gmres(A, b, None, m, om)
    x2, h2 = P.rhqr_gmres(A, b, x1, m, om)
    xr, hr = P.rhqr_gmres_restarted(A, b, None, m, om, tol=0.0, max_cycles=2)
    rows = g["rows"]
    return dict(hist1=rel(h1, g["hist1"]), hist2=rel(h2, g["hist2"]), x1=rel(x1[rows], g["x1_rows"]),
                x2=rel(x2[rows], g["x2_rows"]), restarted_x=rel(xr[rows], g["x2_rows"]),
                restarted_hist=rel(np.concatenate(hr), np.concatenate([g["hist1"], g["hist2"]])),
                true_resid2=float(np.linalg.norm(b - A @ x2) / np.linalg.norm(b)),
                true_resid2_ref=float(g["true_resid2"]))


if __name__ == "__main__":
    res = {}
    for name in (sys.argv[1:] or ["cfg2", "cfg3", "cfg4", "cfg5", "cfg5r"]):
        try:
            res[name] = globals()[name]()
        except Exception as e:  # keep going: this is a measurement script
            res[name] = {"error": repr(e)[:500]}
        print(name, json.dumps(res[name]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "config_parity.json"), "w") as f:
        json.dump(res, f, indent=1)
