"""The C ABI as the drop-in boundary, from the reference's side: the
UNMODIFIED reference package (baseline/_ref, installed by build()) is patched
in place with integration/sketchqr_b200_binding.py — ctypes against
libsketchqr_b200.so, none of this package's Python — and must return what it
returned on the CPU: SRHT sketches bitwise, factors to 1e-12, the same
exceptions.  Skipped when baseline/_ref is absent."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
LIB = os.path.join(ROOT, "paper_2405_10923_b200", "libsketchqr_b200.so")


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b))


@pytest.fixture()
def patched():
    if not os.path.isdir(os.path.join(REF, "sketchqr")):
        pytest.skip("baseline/_ref not installed")
    import torch
    assert torch.cuda.is_available()
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    try:
        import sketchqr
        import sketchqr_b200_binding as b200
        yield sketchqr, b200
        b200.uninstall(sketchqr)
    finally:
        sys.path.remove(REF)
        sys.path.remove(os.path.join(ROOT, "integration"))


def test_reference_package_dispatches_its_hot_path_through_the_c_abi(patched):
    R, b200 = patched
    rng = np.random.default_rng(12)
    N, m, ell = 3000, 10, 40
    W = rng.standard_normal((N, m))
    X = rng.standard_normal((N - m, 3))
    cpu = {}
    for kind, mk in (("srht", lambda: R.SRHTSketch(ell, N - m, 5)), ("gauss", lambda: R.GaussianSketch(ell, N - m, 5))):
        om = mk()
        cpu[kind] = (om.apply(X), om.apply(X[:, 0], dtype=np.float32), R.rhqr_left(W, om),
                     R.rhqr_left(np.asfortranarray(W), om, scaling="unit"), R.rec_rhqr(W, om))
    Wz = W.copy()
    Wz[:, 6] = 0.0
    b200.install(R, LIB)
    assert R.rhqr_left.__module__ == "sketchqr_b200_binding"      # the package-level name is patched too
    for kind, mk in (("srht", lambda: R.SRHTSketch(ell, N - m, 5)), ("gauss", lambda: R.GaussianSketch(ell, N - m, 5))):
        om = mk()
        y, y32, F, Fu, Fr = cpu[kind]
        if kind == "srht":                                         # K1 through sqb_sketch_apply: bitwise
            assert np.array_equal(om.apply(X), y)
            assert np.array_equal(om.apply(X[:, 0], dtype=np.float32), y32)
        G = R.rhqr_left(W, om)
        Gu = R.rhqr_left(np.asfortranarray(W), om, scaling="unit")
        Gr = R.rec_rhqr(W, om)
        for a, b in ((G, F), (Gu, Fu), (Gr, Fr)):
            assert isinstance(a, type(b))
            for k in ("R", "S", "T", "U", "sigmas", "rhos", "betas"):
                assert rel(getattr(a, k), getattr(b, k)) < 1e-12, (kind, k)
        # the reference's own helpers keep working on the returned factors
        assert R.orthogonality_error(G.psi.apply(R.thin_q(G))) < 1e-13
        assert rel(G.prefix(4).R, F.prefix(4).R) < 1e-12
        with pytest.raises(R.BreakdownError, match="sketched tail annihilated at column 7"):
            R.rhqr_left(Wz, om)
        with pytest.raises(R.BreakdownError, match="column 7 exactly dependent"):
            R.rec_rhqr(Wz, om)
    with pytest.raises(ValueError):
        R.rhqr_left(W, R.SRHTSketch(ell, N - m - 1, 5))            # the reference's own shape check
    with pytest.raises(ValueError):
        R.rhqr_left(W, R.SRHTSketch(ell, N - m, 5), scaling="bogus")
    # a policy the library does not cover falls through to the reference's code
    Fs = R.rhqr_left(W, R.SRHTSketch(ell, N - m, 5), policy=R.policy_from_tag("single"))
    assert np.isfinite(Fs.R).all()
    b200.uninstall(R)
    assert R.rhqr_left.__module__ == "sketchqr.rhqr"


def test_reference_gmres_runs_its_arnoldi_through_the_c_abi(patched):
    import scipy.sparse as sp
    R, b200 = patched
    rng = np.random.default_rng(3)
    n, m = 4000, 18
    A = sp.diags([np.full(n - 1, -1.0), np.linspace(2.0, 3.0, n), np.full(n - 1, -0.5)], [-1, 0, 1], format="csr")
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    d = np.linspace(1.0, 2.0, n)
    ops = (A, A.toarray(), lambda v: d * v)
    om = R.SRHTSketch(4 * (m + 1), n - m - 1, 9)
    cpu = [(R.rhqr_arnoldi(op, b, x0, m, om), R.rhqr_gmres(op, b, None, m, om)) for op in ops]
    b200.install(R, LIB)
    assert R.krylov.rhqr_arnoldi.__module__ == "sketchqr_b200_binding"
    for op, (Bc, (xc, hc)) in zip(ops, cpu):
        Bg = R.rhqr_arnoldi(op, b, x0, m, om)
        assert Bg.breakdown == Bc.breakdown and abs(Bg.beta - Bc.beta) <= 1e-13 * abs(Bc.beta)
        for k in ("H", "S", "T", "U", "Q_cols"):
            assert rel(getattr(Bg, k), getattr(Bc, k)) < 1e-10, k
        xg, hg = R.rhqr_gmres(op, b, None, m, om)          # the reference's own driver around the patched Arnoldi
        assert rel(xg, xc) < 1e-10 and rel(hg, hc) < 1e-10
    with pytest.raises(ZeroDivisionError):                  # a failing user matvec surfaces as itself
        R.rhqr_arnoldi(lambda v: v / 0 if False else (_ for _ in ()).throw(ZeroDivisionError()), b, None, m, om)
    b200.uninstall(R)
