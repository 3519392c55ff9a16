"""Is config 1 (2^14 x 32 fp64) bound by the host's launch rate?  Times 20
factorizations (a) as issued, (b) with the stream pre-blocked by a sleep
kernel so that every launch is queued before the GPU reaches it, and
(c) the host's own enqueue time per factorization."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

if os.environ.get("HB_WORK") == "trim":  # trim_rhqr_left 2^20 x 128 fp64, SRHT 96 (scripts/time_trim.py)
    N, m, ell = 1 << 20, 128, 96
    g = torch.Generator(device="cuda").manual_seed(7)
    Wt = (torch.randn(m, N, generator=g, device="cuda", dtype=torch.float64).t()
          * torch.logspace(0, -10, m, dtype=torch.float64, device="cuda"))
    Wt = Wt.contiguous().t().contiguous().t()
    om = P.SRHTSketch(ell, N, 8)
    run = lambda: P.trim_rhqr_left(Wt, om)  # noqa: E731
else:
    N, m, ell = 1 << 14, 32, 128
    W = np.random.default_rng(1).standard_normal((N, m))
    Wd = to_device(W, "double", align_row=m)
    psi = _embed(P.SRHTSketch(ell, N - m, 3), N, m)
    pol = P.PrecisionPolicy("double", "double")
    run = lambda: rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)  # noqa: E731
for _ in range(5):
    run()
torch.cuda.synchronize()
reps = 20 if os.environ.get("HB_WORK") != "trim" else 5
for mode in ("issued", "preblocked"):
    gpu, host = [], []
    for r in range(reps):  # one factorization per sample: the facades may sync at the end (status read)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        if mode == "preblocked":
            torch.cuda._sleep(100_000_000)  # ~50 ms at 2 GHz: longer than the host's enqueue
        e0.record()
        t0 = time.perf_counter()
        run()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        gpu.append(e0.elapsed_time(e1) * 1e3)
        host.append((t1 - t0) * 1e6)
    print(f"{mode:10s}: GPU {min(gpu):9.1f} us/factorization (median {sorted(gpu)[len(gpu) // 2]:9.1f}), "
          f"host call {min(host):9.1f} us", flush=True)
