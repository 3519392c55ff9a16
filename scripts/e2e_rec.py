"""Wall time of rec_rhqr through host operands (config 3), C- and F-order
pinned W, against plain pinned H2D / D2H copies of the same bytes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402

N, m, ell = 1 << 22, 64, 256
W = workloads.gen_cmatrix(N, m)
om = P.GaussianSketch(ell, N - m, 8)
om.desc()
Wc = torch.from_numpy(np.ascontiguousarray(W)).pin_memory()
Wf = torch.from_numpy(np.asfortranarray(W).T).pin_memory().T
print("pinned:", Wc.is_pinned(), Wf.is_pinned())
d = torch.empty(N * m, dtype=torch.float64, device="cuda")
h = torch.empty(N * m, dtype=torch.float64).pin_memory()
for name, fn in (("H2D 2 GiB", lambda: d.copy_(Wc.view(-1), non_blocking=True)),
                 ("D2H 2 GiB", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{name}: {dt*1e3:.1f} ms = {N*m*8/dt/1e9:.1f} GB/s")
for name, Wp in (("C", Wc), ("F", Wf)):
    for _ in range(2):
        P.rec_rhqr(Wp, om)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        F = P.rec_rhqr(Wp, om)
        ts.append(time.perf_counter() - t)
    print(f"rec_rhqr host {name}-order: {np.median(ts)*1e3:.1f} ms")
