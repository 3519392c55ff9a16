"""Host-operand entry point sqb_rhqr_left_host (csrc/host_pipe.cu): numpy W
in, float64 factors out, PCIe transfers overlapped with the sweep.  It must
return exactly what the device-resident path returns (same kernels, same
rounding of W), for both host layouts and every storage format, and map an
overflowing W to PrecisionRangeError like round_to (precision.py:45-50)."""

import numpy as np
import pytest

from oracle import sketchqr_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


def device_factors(P, W, om, pol):
    import torch
    from paper_2405_10923_b200.devarray import to_device, to_numpy
    from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device
    Wd = to_device(torch.from_numpy(np.asarray(O.round_to(W, pol.low))).cuda(), pol.low, align_row=W.shape[1])
    out = rhqr_left_device(Wd, _embed(om, *W.shape), "sqrt2", pol)
    return [to_numpy(x) for x in out]


@pytest.mark.parametrize("tag", ["double", "single", "half", "bf16"])
@pytest.mark.parametrize("order", ["C", "F"])
@pytest.mark.parametrize("N,m,ell", [(3000, 13, 40), (1 << 16, 20, 64), (4096 + 17, 1, 8)])
def test_host_path_equals_device_path(P, tag, order, N, m, ell):
    rng = np.random.default_rng(N + m)
    W = np.asarray(rng.standard_normal((N, m)) * np.logspace(0, -3, m)[None, :], order=order)
    om = P.SRHTSketch(ell, N - m, 11)
    pol = P.PrecisionPolicy("double", tag)
    F = P.rhqr_left(W, om, policy=pol)
    ref = device_factors(P, W, om, pol)
    for name, a, b in zip(("U", "S", "T", "R", "sigmas", "rhos", "betas"),
                          (F.U, F.S, F.T, F.R, F.sigmas, F.rhos, F.betas), ref):
        assert a.shape == b.shape, name
        assert np.array_equal(a, b), name


def test_host_path_matches_oracle(P):
    rng = np.random.default_rng(5)
    N, m, ell = 1 << 15, 24, 96
    W = rng.standard_normal((N, m))
    om = P.SRHTSketch(ell, N - m, 3)
    F = P.rhqr_left(W, om)
    Fo = O.rhqr_left(W, O.SRHT(ell, N - m, 3))
    for k in ("U", "S", "T", "R"):
        a, b = getattr(F, k), getattr(Fo, k)
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b), k


def test_host_path_pinned_tensor_input(P):
    import torch
    rng = np.random.default_rng(9)
    N, m, ell = 1 << 14, 16, 64
    W = rng.standard_normal((N, m))
    om = P.SRHTSketch(ell, N - m, 2)
    F1 = P.rhqr_left(W, om)
    F2 = P.rhqr_left(torch.from_numpy(W).pin_memory(), om)
    F3 = P.rhqr_left(np.asfortranarray(W), om)
    for k in ("U", "S", "T", "R"):
        assert np.array_equal(getattr(F1, k), getattr(F2, k)), k
        assert np.array_equal(getattr(F1, k), getattr(F3, k)), k


@pytest.mark.parametrize("tag", ["half", "bf16"])
def test_host_path_overflow_raises(P, tag):
    W = np.random.default_rng(1).standard_normal((2048, 4))
    W[100, 2] = 1e39 if tag == "bf16" else 7e4
    W[7, 1] = 3e39 if tag == "bf16" else 9e4
    with pytest.raises(P.PrecisionRangeError, match="overflows"):
        P.rhqr_left(W, P.SRHTSketch(16, 2044, 1), policy=P.PrecisionPolicy("double", tag))
    # the context is usable afterwards
    F = P.rhqr_left(W[:, :1], P.SRHTSketch(16, 2047, 1))
    assert np.isfinite(F.R).all()


def test_host_path_breakdown(P):
    from conftest import golden
    g = golden("rhqr_breakdown")
    for W in (g["W"], np.asfortranarray(g["W"])):
        with pytest.raises(P.BreakdownError, match="column 2"):
            P.rhqr_left(W, P.SRHTSketch(12, 30, 34))
