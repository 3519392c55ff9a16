"""rec_rhqr with host operands (sqb_rec_rhqr_host: the Gaussian sketch GEMM
streamed under the blocked upload) is bitwise the device-resident path, for
both host layouts, and the non-streamed sketches/precisions still match."""

import numpy as np
import pytest

from paper_2405_10923_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    import paper_2405_10923_b200 as P
    return P


def _dev(P, W, om, policy=None):
    import torch
    F = P.rec_rhqr(torch.from_numpy(np.asfortranarray(W)).cuda(), om, policy=policy)
    out = {}
    for k in ("U", "S", "T", "R", "sigmas", "rhos", "betas"):
        v = getattr(F, k)
        out[k] = v.to(torch.float64).cpu().numpy() if hasattr(v, "cpu") else v
    return out


@pytest.mark.parametrize("order", ["C", "F"])
def test_streamed_gaussian_rec_rhqr_is_bitwise_the_device_path(P, order):
    N, m, ell = 1 << 18, 64, 256  # ~150 split-K slabs, several upload blocks
    W = workloads.gen_cmatrix(N, m)
    om = P.GaussianSketch(ell, N - m, 12)
    ref = _dev(P, W, om)
    Wh = np.ascontiguousarray(W) if order == "C" else np.asfortranarray(W)
    F = P.rec_rhqr(Wh, om)
    assert isinstance(F.U, np.ndarray) and F.U.shape == (N, m)
    for k, v in ref.items():
        assert np.array_equal(np.asarray(getattr(F, k)), v), k


@pytest.mark.parametrize("kind,tag", [("srht", "double"), ("gauss", "single"), ("srht", "bf16")])
def test_host_rec_rhqr_other_sketches_and_precisions(P, kind, tag):
    N, m = 40000, 24
    W = workloads.gen_cmatrix(N, m)
    om = (P.SRHTSketch if kind == "srht" else P.GaussianSketch)(4 * m, N - m, 5)
    pol = P.PrecisionPolicy("double", tag)
    ref = _dev(P, W, om, pol)
    F = P.rec_rhqr(W, om, policy=pol)
    for k, v in ref.items():
        assert np.array_equal(np.asarray(getattr(F, k)), v), (kind, tag, k)


def test_host_rec_rhqr_rejects_a_mismatched_sketch(P):
    W = np.random.default_rng(0).standard_normal((500, 8))
    with pytest.raises(ValueError):
        P.rec_rhqr(W, P.GaussianSketch(32, 400, 1))
