"""The persistent single-kernel sweep (csrc/rhqr_persist.cu) for small fp64
problems is bitwise the launch-chain path (rhqr_col_kernel + rhqr_step_kernel),
which is itself pinned to the reference (test_gpu_parity.py): same tiles, same
association order of every reduction (SQB_PERSIST=1, measured at parity with
the chain).  The default for small problems is the fast-step kernel
(SQB_PERSIST unset or 2: one block reduction on the critical path, config 1
0.43 -> 0.24 ms), held to the chain and the oracle at 1e-12."""

import os

import numpy as np
import pytest

from oracle import sketchqr_oracle as O
from paper_2405_10923_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


def both(fn, mode="1"):
    """(launch chain, persistent kernel in `mode`)"""
    out = []
    for env in ("0", mode):
        os.environ["SQB_PERSIST"] = env
        try:
            out.append(fn())
        finally:
            os.environ.pop("SQB_PERSIST")
    return out


def launched_persist(P, fn):
    ctx = P._lib.context()
    ctx.profile(True)
    fn()
    _, _, n = ctx.profile_read()
    ctx.profile(False)
    return n


@pytest.mark.parametrize("N,m,ell,seed,scaling", [
    (1 << 14, 32, 128, 17, "sqrt2"),     # BASELINE config 1
    (1 << 14, 32, 128, 17, "unit"),
    (5000, 9, 40, 3, "sqrt2"),           # ragged last tile
    (1 << 16, 24, 96, 5, "sqrt2"),       # n_pad = 2^16: 128 tile CTAs
    (3000, 2, 8, 7, "sqrt2"),
])
def test_persistent_sweep_is_bitwise_the_launch_chain(P, N, m, ell, seed, scaling):
    W = workloads.gaussian_w(N, m, seed)
    om = P.SRHTSketch(ell, N - m, seed + 1)
    chain, pers = both(lambda: P.rhqr_left(W, om, scaling=scaling))
    for k in ("U", "S", "T", "R", "sigmas", "rhos", "betas"):
        assert np.array_equal(getattr(chain, k), getattr(pers, k)), k


@pytest.mark.parametrize("N,m,ell,seed,scaling", [
    (1 << 14, 32, 128, 17, "sqrt2"),     # BASELINE config 1 (register tree, 32 tiles)
    (1 << 14, 32, 128, 17, "unit"),
    (5000, 9, 40, 3, "sqrt2"),           # ragged last tile, staged leaves
    (1 << 16, 24, 96, 5, "unit"),        # 128 tile CTAs
    (3000, 2, 8, 7, "sqrt2"),
])
def test_fast_step_persistent_sweep_matches_the_chain_and_the_oracle(P, N, m, ell, seed, scaling):
    """SQB_PERSIST=2: the single-reduction step (csrc/rhqr_persist.cu
    ps_step_fast) is the launch chain's mathematics in another association:
    every factor within 1e-12 of the chain and of the CPU oracle
    (rhqr.py:219-251)."""
    W = workloads.gaussian_w(N, m, seed)
    om = P.SRHTSketch(ell, N - m, seed + 1)
    chain, fast = both(lambda: P.rhqr_left(W, om, scaling=scaling), mode="2")
    Fo = O.rhqr_left(W, O.SRHT(ell, N - m, seed + 1), scaling=scaling)
    for k in ("U", "S", "T", "R", "sigmas", "rhos", "betas"):
        a, b, o = getattr(chain, k), getattr(fast, k), getattr(Fo, k)
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(a), k
        assert np.linalg.norm(o - b) <= 1e-12 * np.linalg.norm(o), k


def test_fast_step_breakdown(P, monkeypatch):
    monkeypatch.setenv("SQB_PERSIST", "2")
    N = 2048
    W = np.zeros((N, 4))
    W[0] = 1.0
    with pytest.raises(P.BreakdownError, match="column 2"):
        P.rhqr_left(W, P.SRHTSketch(16, N - 4, 3))
    W2 = np.random.default_rng(0).standard_normal((N, 4))
    assert np.all(np.isfinite(P.rhqr_left(W2, P.SRHTSketch(16, N - 4, 3)).R))


def test_config1_runs_the_persistent_kernel_and_matches_the_oracle(P):
    import torch
    N, m, ell, seed = 1 << 14, 32, 128, 17
    W = workloads.gaussian_w(N, m, 2024)
    om = P.SRHTSketch(ell, N - m, seed)
    Wd = torch.from_numpy(W).cuda()
    os.environ["SQB_PERSIST"] = "1"
    try:
        assert launched_persist(P, lambda: P.rhqr_left(Wd, om)) == 1  # one persistent launch
        F = P.rhqr_left(W, om)
    finally:
        os.environ.pop("SQB_PERSIST")
    Fo = O.rhqr_left(W, O.SRHT(ell, N - m, seed))
    for k in ("U", "S", "T", "R"):
        a, b = getattr(F, k), getattr(Fo, k)
        assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-12, k


def test_persistent_breakdown_and_recovery(P, monkeypatch):
    # an exactly dependent column stops the persistent grid at column 2 (all CTAs)
    monkeypatch.setenv("SQB_PERSIST", "1")
    N = 2048
    W = np.zeros((N, 4))
    W[0] = 1.0  # every column the same, in the identity block only (test_rhqr.py:296-301)
    with pytest.raises(P.BreakdownError, match="column 2"):
        P.rhqr_left(W, P.SRHTSketch(16, N - 4, 3))
    W2 = np.random.default_rng(0).standard_normal((N, 4))
    F = P.rhqr_left(W2, P.SRHTSketch(16, N - 4, 3))
    assert np.all(np.isfinite(F.R))
