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

N, m, ell = 1 << 14, 32, 128
W = np.random.default_rng(1).standard_normal((N, m))
Wd = to_device(W, "double", align_row=m)
psi = _embed(P.SRHTSketch(ell, N - m, 3), N, m)
pol = P.PrecisionPolicy("double", "double")
for _ in range(5):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
torch.cuda.synchronize()
reps = 20
for mode in ("issued", "preblocked"):
    if True:  # the library runs on torch's current stream (_lib.context)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        if mode == "preblocked":
            torch.cuda._sleep(200_000_000)  # ~0.1 s at 2 GHz
        e0.record()
        t0 = time.perf_counter()
        for _ in range(reps):
            rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
        t1 = time.perf_counter()
        e1.record()
    torch.cuda.synchronize()
    print(f"{mode:10s}: GPU {e0.elapsed_time(e1) / reps * 1e3:7.1f} us/factorization, host enqueue "
          f"{(t1 - t0) / reps * 1e6:7.1f} us/factorization", flush=True)
