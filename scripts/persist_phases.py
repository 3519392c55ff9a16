"""Per-phase timing of the persistent config-1 kernel (clock64 stamps of
tile CTA 0 and the top CTA; csrc/rhqr_persist.cu PS_STAMP):
phase A (column pass), barrier wait, phase B (redundant step)."""
import os
import sys

import numpy as np
import torch

os.environ.setdefault("SQB_PERSIST", "2")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import _lib, workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

N, m, ell = 1 << 14, 32, 128
W = workloads.gaussian_w(N, m, 7)
om = P.SRHTSketch(ell, N - m, 8)
Wd = to_device(W, "double", align_row=m)
psi = _embed(om, N, m)
pol = P.PrecisionPolicy("double", "double")
ctx = _lib.context()
buf = torch.zeros(m * 4 * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
_lib.lib().sqb_debug_step_stamps(ctx.h, buf.data_ptr(), -2)
rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
torch.cuda.synchronize()
_lib.lib().sqb_debug_step_stamps(ctx.h, None, -1)
t = buf.cpu().numpy().reshape(m, 4, 16).astype(np.float64) / 1.965  # clock64 cycles -> ns at 1965 MHz
if os.environ["SQB_PERSIST"] == "2":
    for who, name in ((0, "tile CTA 0"), (1, "top CTA")):
        z = t[0, who]
        last = t[m - 1, who, 3]
        print(f"{name}: prologue {(z[1]-z[0])/1e3:.2f} us, step 0 {(z[2]-z[1])/1e3:.2f} us, "
              f"column loop {(last - z[2])/1e3:.2f} us, epilogue {(z[3]-last)/1e3:.2f} us, kernel {(z[3]-z[0])/1e3:.2f} us")
whos = ((0, "tile CTA 0"), (1, "top CTA")) + (((2, "T CTA"), (3, "ID CTA")) if os.environ["SQB_PERSIST"] == "2" else ())
for who, name in whos:
    x = t[1:, who]
    A = x[:, 1] - x[:, 0]
    Wt = x[:, 2] - x[:, 1]
    B = x[:, 3] - x[:, 2]
    gap = x[1:, 0] - x[:-1, 3]
    print(f"{name}: phaseA {np.median(A)/1e3:.2f} us, barrier wait {np.median(Wt)/1e3:.2f} us, "
          f"phaseB {np.median(B)/1e3:.2f} us, loop gap {np.median(gap)/1e3:.2f} us; "
          f"column period {np.median(np.diff(x[:, 0]))/1e3:.2f} us")
    d = lambda i, j: np.median(x[:, j] - x[:, i]) / 1e3  # noqa: E731
    if os.environ["SQB_PERSIST"] == "2":
        print(f"   phase B (fast step): pre-loads {d(2, 5):.2f}, leaves + trees {d(5, 4):.2f}, "
              f"fused reduction {d(4, 7):.2f}, scalars {d(7, 8):.2f} us")
        continue
    print(f"   phase B: pre-loads {d(2, 5):.2f}, leaf staging {d(5, 6):.2f}, trees {d(6, 4):.2f}, "
          f"rho reduction {d(4, 7):.2f}, scalars {d(7, 8):.2f}, s rows {d(8, 9):.2f}, "
          f"partial vectors {d(9, 10):.2f}, v/coef {d(10, 3):.2f} us")
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
e.record()
torch.cuda.synchronize()
print(f"rhqr_left config 1: {s.elapsed_time(e) / 20 * 1e3:.1f} us per factorization")
