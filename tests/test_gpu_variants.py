"""GPU parity of the factorization variants next to the hot path (SURVEY
§8(f) rank 1 and 4): rhqr_block (rhqr.py:334-365), rhqr_right (:270-301) and
t_factor_from_sketches (:122-132), against the reference's golden vectors,
the CPU oracle and the reference's own cross-variant tests
(test_rhqr.py:207-235, test_acceptance.py:100-120).  fp64 bar: 1e-12
relative (the reference's own test tolerance for these variants)."""

import numpy as np
import pytest

from conftest import golden
from oracle import sketchqr_oracle as O
from paper_2405_10923_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)


# ------------------------------------------------------------ t_factor
def test_t_factor_known_answers(P):
    S = np.zeros((6, 2))
    S[0, 0] = S[1, 1] = np.sqrt(2.0)
    assert np.allclose(P.t_factor_from_sketches(S), np.eye(2), atol=1e-14)
    assert np.allclose(P.t_factor_from_sketches(np.array([[2.0], [1.0]])), [[0.4]], atol=1e-15)
    g = golden("t_factor_30x8")
    assert rel(P.t_factor_from_sketches(g["S"]), g["T"]) < 1e-13


def test_t_factor_round_trip(P):
    S = np.random.default_rng(3).standard_normal((30, 8))
    T = P.t_factor_from_sketches(S)
    G = S.T @ S
    Ti = np.linalg.inv(T)
    assert np.linalg.norm(G - (Ti + Ti.T)) <= 1e-12 * np.linalg.norm(G)


def test_t_factor_singular(P):
    with pytest.raises(P.SingularFactorError):
        P.t_factor_from_sketches(np.zeros((5, 2)))


# ------------------------------------------------------------ rhqr_block
@pytest.mark.parametrize("bs", [20, 1, 6, 8])
def test_rhqr_block_matches_reference(P, bs):
    g = golden("rhqr_block_1500x20_srht48")
    W = g["W"]
    om = P.SRHTSketch(int(g["ell"]), W.shape[0] - W.shape[1], int(g["seed"]))
    B = P.rhqr_block(W, om, block_size=bs)
    assert len(B.panels) == -(-20 // bs)
    assert [p.offset for p in B.panels] == list(range(0, 20, bs))
    assert rel(B.R, g[f"R_{bs}"]) < 1e-12
    tb = np.concatenate([np.asarray(p.T).ravel() for p in B.panels])
    assert rel(tb, g[f"Tblk_{bs}"]) < 1e-12
    assert np.allclose(np.stack([B.sigmas, B.rhos, B.betas]), g[f"scal_{bs}"], rtol=1e-12, atol=1e-14)
    F = B.stacked()
    assert rel(F.U, g[f"U_{bs}"]) < 1e-12
    assert rel(F.S, g[f"S_{bs}"]) < 1e-12
    assert rel(F.T, g[f"Tst_{bs}"]) < 1e-11


def test_rhqr_block_matches_unblocked(P):
    # test_rhqr.py:225-235 with the device Gaussian sketch
    rng = np.random.default_rng(5)
    n, m = 60, 8
    W = rng.standard_normal((n, m))
    om = P.GaussianSketch(24, n - m, 22)
    ref = P.rhqr_left(W, om)
    for bs in (m, 1, 3):
        B = P.rhqr_block(W, om, block_size=bs)
        assert np.allclose(B.R, ref.R, atol=1e-12 * np.linalg.norm(ref.R))
        F = B.stacked()
        assert np.allclose(F.U, ref.U, atol=1e-12 * np.linalg.norm(ref.U))
        fro, _, _ = P.factorization_errors(W, P.thin_q(F), F.R)
        assert fro <= 1e-13


def test_rhqr_block_identity_is_householder(P):
    # test_acceptance.py:100-120 (criterion 1) for the blocked variant
    rng = np.random.default_rng(101)
    for _ in range(3):
        W = rng.standard_normal((64, 8))
        _, R_ref, aux = O.householder_qr(W)
        F = P.rhqr_block(W, P.IdentitySketch(56), block_size=3).stacked()
        assert rel(F.R, R_ref) <= 1e-13
        assert rel(F.U, aux["U"]) <= 1e-13


@pytest.mark.parametrize("N,m,bs,ell", [(1 << 16, 64, 16, 128), (50_003, 40, 32, 96), (1 << 18, 96, 32, 192)])
def test_rhqr_block_against_oracle(P, N, m, bs, ell):
    W = np.random.default_rng(N + m).standard_normal((N, m)) * np.logspace(0, -6, m)
    om_d = P.SRHTSketch(ell, N - m, 77)
    om_o = O.SRHT(ell, N - m, 77)
    B = P.rhqr_block(W, om_d, block_size=bs)
    Bo = O.rhqr_block(W, om_o, block_size=bs)
    assert rel(B.R, Bo.R) < 1e-10
    F, Fo = B.stacked(), Bo.stacked()
    assert rel(F.U, Fo.U) < 1e-9
    assert rel(F.S, Fo.S) < 1e-9
    fro, _, _ = P.factorization_errors(W, P.thin_q(F), F.R)
    assert fro < 1e-13


# bar: 4 unit roundoffs of the storage format (measured on the B200,
# scripts/probe_lowprec_bars.py: single 0.7-0.9 u, half bitwise, bf16 0.1-1.0 u)
@pytest.mark.parametrize("tag,tol", [("single", 4 * 2.0 ** -24), ("half", 4 * 2.0 ** -11), ("bf16", 4 * 2.0 ** -8)])
def test_rhqr_block_low_precision(P, tag, tol):
    # same bars as the rhqr_left mixed-precision parity (low-format GEMV
    # accumulation order differs from numpy's)
    rng = np.random.default_rng(9)
    N, m = 8192, 16
    W = rng.standard_normal((N, m))
    B = P.rhqr_block(W, P.SRHTSketch(64, N - m, 12), block_size=6, policy=P.PrecisionPolicy("double", tag))
    Bo = O.rhqr_block(W, O.SRHT(64, N - m, 12), block_size=6, policy=O.Policy("double", tag))
    assert rel(B.R, Bo.R) < tol
    U = B.stacked().U
    assert np.array_equal(P.round_to(U, tag), U)


@pytest.mark.parametrize("tag,tol", [("single", 4 * 2.0 ** -24), ("bf16", 4 * 2.0 ** -8)])
def test_rhqr_right_low_precision(P, tag, tol):
    rng = np.random.default_rng(10)
    N, m = 8192, 12
    W = rng.standard_normal((N, m))
    F = P.rhqr_right(W, P.SRHTSketch(48, N - m, 13), policy=P.PrecisionPolicy("double", tag))
    Fo = O.rhqr_right(W, O.SRHT(48, N - m, 13), policy=O.Policy("double", tag))
    assert rel(F.R, Fo.R) < tol


def test_rhqr_block_breakdown_and_args(P):
    W = np.zeros((40, 4))
    W[0] = 1.0
    with pytest.raises(P.BreakdownError, match="column 2"):
        P.rhqr_block(W, P.SRHTSketch(8, 36, 3), block_size=1)
    with pytest.raises(ValueError, match="block_size must be positive"):
        P.rhqr_block(np.ones((40, 4)), P.SRHTSketch(8, 36, 3), block_size=0)


# ------------------------------------------------------------ rhqr_right
def test_rhqr_right_matches_reference(P):
    g = golden("rhqr_right_900x12_srht36")
    W = g["W"]
    om = P.SRHTSketch(int(g["ell"]), W.shape[0] - W.shape[1], int(g["seed"]))
    F = P.rhqr_right(W, om)
    for k in ("U", "S", "R"):
        assert rel(getattr(F, k), g[k]) < 1e-12, k
    assert rel(F.T, g["T"]) < 1e-11
    assert np.allclose(np.stack([F.sigmas, F.rhos, F.betas]),
                       np.stack([g["sigmas"], g["rhos"], g["betas"]]), rtol=1e-12, atol=1e-14)
    Fu = P.rhqr_right(W, om, scaling="unit")
    assert rel(Fu.U, g["U_unit"]) < 1e-12 and rel(Fu.R, g["R_unit"]) < 1e-12


def test_rhqr_right_agrees_with_left(P):
    rng = np.random.default_rng(21)
    N, m = 20_000, 24
    W = rng.standard_normal((N, m))
    om = P.SRHTSketch(64, N - m, 4)
    Fr, Fl = P.rhqr_right(W, om), P.rhqr_left(W, om)
    assert rel(Fr.R, Fl.R) < 1e-12
    assert rel(Fr.U, Fl.U) < 1e-11
    assert rel(Fr.T, Fl.T) < 1e-10
    Fo = O.rhqr_right(W, O.SRHT(64, N - m, 4))
    assert rel(Fr.R, Fo.R) < 1e-12


def test_rhqr_right_identity_is_householder(P):
    rng = np.random.default_rng(102)
    W = rng.standard_normal((64, 8))
    _, R_ref, aux = O.householder_qr(W)
    F = P.rhqr_right(W, P.IdentitySketch(56))
    assert rel(F.R, R_ref) <= 1e-13
    assert rel(F.U, aux["U"]) <= 1e-13


@pytest.mark.parametrize("tag", ["bf16", "half"])
@pytest.mark.parametrize("N,m,ell", [(1 << 15, 12, 48), ((1 << 16) + 8 * 1000 + 3, 9, 40), (3 * 8192 + 77, 5, 20)])
def test_packed16_tile_fwht_is_bitwise(P, monkeypatch, tag, N, m, ell):
    """The column pass's packed 16-bit in-tile FWHT (srht.cuh p16_*, full
    2^13 tiles) must give bitwise the factors of the fp32-staged path, which
    is the reference's correctly rounded op sequence."""
    rng = np.random.default_rng(N)
    W = rng.standard_normal((N, m)) * np.logspace(0, -2, m)[None, :]
    om = P.SRHTSketch(ell, N - m, 5)
    pol = P.PrecisionPolicy("double", tag)
    F1 = P.rhqr_left(W, om, policy=pol)
    monkeypatch.setenv("SQB_NO_P16", "1")
    F2 = P.rhqr_left(W, om, policy=pol)
    for k in ("U", "S", "T", "R"):
        assert np.array_equal(getattr(F1, k), getattr(F2, k)), k


# ------------------------------------------------------------ cross-pass overlap, partial tile
@pytest.mark.parametrize("tag,N,m,ell", [
    ("double", (1 << 19) + 4096 + 24, 24, 64),    # partial last tile of whole 16-byte runs, many tiles
    ("double", (1 << 19) + 1003, 24, 64),         # ragged partial tile (generic loop)
    ("bf16", (1 << 20) + 2048 + 32, 32, 96),      # 16-bit storage, 3-CTA/SM ring variant
    ("single", (1 << 19) + 8 + 16, 16, 48),
])
def test_column_pass_overlap_and_partial_tile_are_bitwise(P, monkeypatch, tag, N, m, ell):
    """The device-resident sweep with the cross-pass overlap (per-block flags,
    step kernel triggering its dependents early: SQB_EARLY=2 forces it, 0 is
    the plain PDL order) and with the pipelined partial last tile (SQB_NO_PART=1
    restores the generic loop) must give bitwise the same factors: same
    operations in the same order, only scheduled differently
    (rhqr.py:236-250)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(N)
    W = torch.randn(m, N, generator=g, device="cuda", dtype=torch.float64).t() * torch.logspace(
        0, -3, m, dtype=torch.float64, device="cuda")
    om = P.SRHTSketch(ell, N - m, 5)
    pol = P.PrecisionPolicy("double", tag)
    out = {}
    for early, nopart in (("2", "0"), ("0", "0"), ("2", "1"), ("0", "1")):
        monkeypatch.setenv("SQB_EARLY", early)
        monkeypatch.setenv("SQB_NO_PART", nopart)
        for rep in range(2):  # the overlap is a race if it is wrong: run it twice
            F = P.rhqr_left(W, om, policy=pol)
            cur = {k: getattr(F, k).clone() for k in ("U", "S", "T", "R")}
            if not out:
                out = cur
            for k in out:
                assert torch.equal(out[k], cur[k]), (k, early, nopart, rep)
    assert float(torch.linalg.norm(out["R"])) > 0


# ------------------------------------------------------------ tall Householder QR (baseline, cond_number)
@pytest.mark.parametrize("p,m,scaling", [(40000, 24, "sqrt2"), ((1 << 17) + 77, 33, "unit"), (30001, 5, "sqrt2")])
def test_tall_householder_qr_matches_the_oracle(P, p, m, scaling):
    """householder_qr beyond one CTA's shared memory (csrc/hqr_tall.cu: two
    transposed GEMVs and one GEMV over the finished reflectors per column)
    against the oracle's restatement of baselines.py:33-89."""
    rng = np.random.default_rng(p)
    A = rng.standard_normal((p, m)) * np.logspace(0, -6, m)[None, :]
    got = P.householder_qr(A, scaling=scaling)
    Q, R, aux = O.householder_qr(A, scaling=scaling)
    assert rel(got.R, R) < 1e-12
    assert rel(got.aux["U"], aux["U"]) < 1e-12 and rel(got.aux["T"], aux["T"]) < 1e-12
    assert rel(got.Q, Q) < 1e-12
    assert np.linalg.norm(got.Q.T @ got.Q - np.eye(m)) < 1e-13
    assert np.linalg.norm(got.Q @ got.R - A) <= 1e-14 * np.linalg.norm(A)


def test_tall_householder_qr_breakdown_and_singular_cond(P):
    p, m = 50000, 4
    A = np.random.default_rng(1).standard_normal((p, m))
    A[:, 2] = 2.0 * A[:, 0] - A[:, 1]  # rank deficient, but not exactly in floating point
    assert P.cond_number(A) > 1e14
    Z = np.zeros((p, 3))
    Z[:, 0] = 1.0
    with pytest.raises(P.BreakdownError, match="column 2"):
        P.householder_qr(Z)
    assert P.cond_number(Z) == np.inf


def test_cond_number_of_a_tall_illconditioned_matrix_uses_the_library_qr(P):
    """linalg.py:151-160 on a tall matrix with cond 1e11: the Gram probe
    cannot resolve it, the value comes from the library's tall Householder QR
    and a k x k SVD — within 1e-3 of numpy's SVD of the same matrix."""
    p, m = 1 << 17, 32
    W = workloads.illcond_w(p, m, 3, smin_exp=-11.0)
    ref = np.linalg.cond(W)
    assert 1e10 < ref < 1e12
    # sigma_min is defined to ~u cond = 1e-5 relative: two backward-stable routes agree to that
    assert P.cond_number(W) == pytest.approx(ref, rel=1e-3)
