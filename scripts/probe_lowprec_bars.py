"""Measured low-precision parity errors (in units of the storage format's
unit roundoff u) behind the bars of tests/test_gpu_parity.py::
test_rhqr_left_mixed_precision and tests/test_gpu_variants.py::*_low_precision."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2405_10923_b200 as P
from oracle import sketchqr_oracle as O
from conftest import golden

U = {"single": 2.0 ** -24, "half": 2.0 ** -11, "bf16": 2.0 ** -8}
rel = lambda a, b: np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)
for tag in ("single", "half", "bf16"):
    g = golden(f"rhqr_left_4096x16_{tag}")
    seed = 31 if tag == "bf16" else 29
    F = P.rhqr_left(g["W"], P.SRHTSketch(64, 4096 - 16, seed), policy=P.PrecisionPolicy("double", tag))
    print(f"rhqr_left {tag}: rel R {rel(F.R, g['R']):.3e} = {rel(F.R, g['R']) / U[tag]:.2f} u")
    rng = np.random.default_rng(9)
    N, m = 8192, 16
    W = rng.standard_normal((N, m))
    B = P.rhqr_block(W, P.SRHTSketch(64, N - m, 12), block_size=6, policy=P.PrecisionPolicy("double", tag))
    Bo = O.rhqr_block(W, O.SRHT(64, N - m, 12), block_size=6, policy=O.Policy("double", tag))
    print(f"rhqr_block {tag}: rel R {rel(B.R, Bo.R):.3e} = {rel(B.R, Bo.R) / U[tag]:.2f} u")
    if tag != "half":
        rng = np.random.default_rng(10)
        N, m = 8192, 12
        W = rng.standard_normal((N, m))
        F = P.rhqr_right(W, P.SRHTSketch(48, N - m, 13), policy=P.PrecisionPolicy("double", tag))
        Fo = O.rhqr_right(W, O.SRHT(48, N - m, 13), policy=O.Policy("double", tag))
        print(f"rhqr_right {tag}: rel R {rel(F.R, Fo.R):.3e} = {rel(F.R, Fo.R) / U[tag]:.2f} u")
