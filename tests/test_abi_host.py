"""CPU tests of the boundary: the C-ABI library loads and exports every symbol
include/sketchqr_b200.h declares; host-side helpers match numpy."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "sketchqr_b200.h")
LIB = os.path.join(ROOT, "paper_2405_10923_b200", "libsketchqr_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|const char\*|int64_t)\s+(sqb_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2405_10923_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_hot_path():
    names = declared()
    for must in ("sqb_ctx_create", "sqb_sketch_apply", "sqb_embedded_apply", "sqb_rhqr_left",
                 "sqb_apply_reflectors", "sqb_thin_q", "sqb_sketch_q", "sqb_rh_vector"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_python_binding_covers_header():
    from paper_2405_10923_b200 import _lib
    assert set(declared()) <= set(_lib.exported_symbols())


def test_version(lib):
    assert lib.sqb_version() == 1


@pytest.mark.parametrize("tag", ["single", "half", "bf16"])
def test_round_scalar_matches_numpy(lib, tag):
    from oracle.sketchqr_oracle import TAG_DTYPE
    f = lib.sqb_round_scalar
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_int, ctypes.c_double]
    code = {"single": 1, "half": 2, "bf16": 3}[tag]
    rng = np.random.default_rng(0)
    vals = np.concatenate([rng.standard_normal(2000) * 10.0 ** rng.integers(-9, 6, 2000),
                           [1 + 2 ** -8 + 2 ** -30, 1 + 2 ** -11 + 2 ** -40, 65519.0, 65520.0,
                            6e-8, 2.0 ** -25, np.sqrt(2 ** 20 / 256), (2 ** 21) ** -0.5, 0.0]])
    for v in vals:
        want = float(np.array([v]).astype(TAG_DTYPE[tag]).astype(np.float64)[0])
        got = f(code, float(v))
        assert got == want or (np.isinf(want) and np.isinf(got)), (tag, v, got, want)


def test_ctx_create_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    lib.sqb_ctx_create.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    assert lib.sqb_ctx_create(0, None, ctypes.byref(h)) == 4  # SQB_ERR_CUDA


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2405_10923_b200 as P
    om = P.SRHTSketch(8, 12, 3)
    with pytest.raises(RuntimeError, match="CUDA"):
        om.apply(np.ones(12))


def test_srht_host_state_matches_oracle():
    """Operator state (signs, indices, scale) is generated host-side with the
    reference's numpy calls (sketching.py:144-147)."""
    import paper_2405_10923_b200 as P
    from conftest import golden
    for name in ("srht_8_12_3", "srht_128_16352_7", "srht_400_8191_13"):
        g = golden(name)
        op = P.SRHTSketch(int(g["ell"]), int(g["n"]), int(g["seed"]))
        assert op.n_pad == int(g["n_pad"]) and op.scale == float(g["scale"])
        assert np.array_equal(op.indices, g["indices"])
        bits = op.sign_bits().view(np.uint8)[: g["signbits"].shape[0]]
        assert np.array_equal(bits, g["signbits"])


def test_gaussian_host_rows_bitwise():
    import paper_2405_10923_b200 as P
    from conftest import golden
    g = golden("gauss_8_50_2")
    assert np.array_equal(P.GaussianSketch(8, 50, 2).matrix(), g["G"])
    h = golden("gauss_24_5000_9_sha")
    from paper_2405_10923_b200.workloads import sha256
    assert bytes(h["sha"]).hex() == sha256(P.GaussianSketch(24, 5000, 9, threads=5).matrix())


def test_embed_validation_messages():
    import paper_2405_10923_b200 as P
    from paper_2405_10923_b200.rhqr import _embed
    with pytest.raises(ValueError, match="expected n-m=18"):
        _embed(P.SRHTSketch(8, 12, 3), 20, 2)
    with pytest.raises(ValueError, match="below column count"):
        _embed(P.SRHTSketch(2, 16, 3), 20, 4)
    with pytest.raises(ValueError):
        P.SRHTSketch(20, 12, 3)
