"""End-to-end time of the UNMODIFIED reference package's own call,
sketchqr.rhqr_left(W, omega), with its hot path dispatched to the library by
integration/sketchqr_b200_binding.py — what a user of the reference gets without
touching their code (ordinary pageable numpy W in, numpy factors out), against
the same call on the CPU at a bounded size.  Config 2's shape."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "integration"))
sys.path.insert(0, ROOT)
import sketchqr  # noqa: E402
import sketchqr_b200_binding as b200  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402  (input generator only)

N, m, ell = 1 << 20, 128, 256
W = workloads.illcond_w(N, m, 7)
om = sketchqr.SRHTSketch(ell, N - m, 8)
Ns = 1 << 17
t0 = time.perf_counter()
Fc = sketchqr.rhqr_left(W[:Ns], sketchqr.SRHTSketch(ell, Ns - m, 8))
t_cpu = time.perf_counter() - t0
b200.install(sketchqr, os.path.join(ROOT, "paper_2405_10923_b200", "libsketchqr_b200.so"))
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    F = sketchqr.rhqr_left(W, om)
    ts.append(time.perf_counter() - t0)
alg = 8.0 * N * (m * m + 5 * m) / 2
print(f"patched reference, sketchqr.rhqr_left(W 2^20 x 128 pageable C-order): {[round(t * 1e3, 1) for t in ts]} ms "
      f"-> best {min(ts) * 1e3:.1f} ms = {alg / min(ts) / 1e9:.0f} GB/s effective")
print(f"unpatched reference on 2^17 rows: {t_cpu:.2f} s = {8.0 * Ns * (m * m + 5 * m) / 2 / t_cpu / 1e9:.2f} GB/s "
      f"(x 8 rows => ~{8 * t_cpu:.0f} s at full size)")
print("R finite:", bool(np.isfinite(F.R).all()), " ||R|| =", float(np.linalg.norm(F.R)))
