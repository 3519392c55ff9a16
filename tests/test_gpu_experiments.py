"""The device stability-sweep harness against the reference harness's own
rows on the same inputs (tests/golden/experiments_*.npz, written by running
the unmodified reference).  Widths and status strings must match exactly;
cond(Q) and cond(Psi Q) to 1e-9 relative in double; the error metrics are
rounding noise (~1e-15) in both implementations, so they must stay within
a small factor of the reference's (with an absolute floor)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


CASES = {
    "left": dict(algo="rhqr-left", seed=3, every=8),
    "right": dict(algo="rhqr-right", seed=3, every=8),
    "block": dict(algo="rhqr-block", seed=3, every=8, block_size=16),
    "rec": dict(algo="rec-rhqr", seed=3, every=16),
    "leftgauss": dict(algo="rhqr-left", sketch="gauss", ell=120, seed=5, every=12),
    "mixed": dict(algo="rhqr-left", ell=96, seed=2, precision="mixed", every=8),
}


def check_rows(rows, g, name, cond_tol, noise_factor, floor):
    assert [r.j for r in rows] == g[f"{name}_j"].tolist()
    assert [r.status for r in rows] == g[f"{name}_status"].tolist()
    for r, want in zip(rows, g[f"{name}_vals"]):
        got = np.array(r[1:-1], dtype=float)
        if np.isnan(want).all():
            assert np.isnan(got).all()
            continue
        assert got[:2] == pytest.approx(want[:2], rel=cond_tol)
        assert np.all(got[2:] <= noise_factor * want[2:] + floor), (got, want)


@pytest.mark.parametrize("name", list(CASES))
def test_factor_sweep_matches_reference(P, name):
    g = golden("experiments_cmatrix_2048x48")
    rows = P.run_factor_experiment(P.gen_cmatrix(2048, 48), P.ExperimentConfig(**CASES[name]))
    if name == "mixed":  # fp16 storage: every metric is rounding noise of the low format
        check_rows(rows, g, name, cond_tol=0.2, noise_factor=3.0, floor=0.0)
    else:
        check_rows(rows, g, name, cond_tol=1e-9, noise_factor=10.0, floor=1e-14)


def test_factor_sweep_breakdown_rows(P):
    g = golden("experiments_cmatrix_2048x48")
    rows = P.run_factor_experiment(g["bd_W"], P.ExperimentConfig(algo="rhqr-left", seed=1, every=2))
    check_rows(rows, g, "bd", cond_tol=1e-9, noise_factor=10.0, floor=1e-14)


def test_factor_sweep_device_input_and_csv(P, tmp_path):
    import torch
    W = torch.from_numpy(P.gen_cmatrix(4096, 40)).cuda()
    cfg = P.ExperimentConfig(algo="rhqr-left", ell=160, seed=9, every=10, deterministic=True)
    rows = P.run_factor_experiment(W, cfg)
    assert [r.j for r in rows] == [10, 20, 30, 40]
    assert all(r.status == "ok" and r.orth_err < 1e-13 and r.fro_rel_err < 1e-14 for r in rows)
    p = tmp_path / "s.csv"
    P.write_csv(str(p), rows, config=cfg)
    assert p.read_text().splitlines()[1] == "j,cond_q,cond_sq,fro_rel_err,max_col_rel_err,orth_err,status"


@pytest.mark.parametrize("name,cfg", [("srht", dict(algo="rhqr", seed=4)),
                                      ("gauss", dict(algo="rhqr", sketch="gauss", ell=100, seed=6))])
def test_gmres_sweep_matches_reference(P, name, cfg):
    import scipy.sparse
    g = golden("experiments_gmres_cd24")
    A = scipy.sparse.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(576, 576))
    rows = P.run_gmres_experiment(A, g["b"], 24, P.ExperimentConfig(**cfg))
    assert [r.j for r in rows] == g[f"{name}_j"].tolist()
    assert [r.status for r in rows] == g[f"{name}_status"].tolist()
    want = g[f"{name}_vals"]
    got = np.array([r[1:-1] for r in rows], dtype=float)
    assert got[:, 0] == pytest.approx(want[:, 0], rel=1e-9)   # sketched residual
    assert got[:, 1] == pytest.approx(want[:, 1], rel=1e-7)   # true residual
    assert np.all(got[:, 2] <= 10 * want[:, 2] + 1e-16)       # relation error (noise)
    assert got[:, 3] == pytest.approx(want[:, 3], rel=1e-9)   # cond of the basis


def test_gmres_identity_closes_immediately(P):
    g = golden("experiments_gmres_cd24")
    rows = P.run_gmres_experiment(np.eye(32), g["b"][:32], 5,
                                  P.ExperimentConfig(algo="rhqr", sketch="gauss", seed=1))
    assert len(rows) == 1 and rows[0].status == str(g["eye_status"][0]) == "closed@1"
    assert rows[0].true_resid <= 1e-12 * np.linalg.norm(g["b"][:32])


@pytest.mark.parametrize("name,algo", [("trimleft", "trim-left"), ("trimright", "trim-right")])
def test_trim_factor_sweep_matches_reference(P, name, algo):
    """The trimmed drivers in the harness (experiments.py:161-164, 196-199):
    ell = 20 < m = 24, so orth_err is O(1) by design and compared as a value."""
    g = golden("experiments_trim")
    rows = P.run_factor_experiment(g["W"], P.ExperimentConfig(algo=algo, ell=20, seed=3, every=6))
    assert [r.j for r in rows] == g[f"{name}_j"].tolist()
    assert [r.status for r in rows] == g[f"{name}_status"].tolist()
    for r, want in zip(rows, g[f"{name}_vals"]):
        got = np.array(r[1:-1], dtype=float)
        assert got[[0, 1, 4]] == pytest.approx(want[[0, 1, 4]], rel=1e-8)
        assert np.all(got[2:4] <= 10.0 * want[2:4] + 1e-14), (got, want)
