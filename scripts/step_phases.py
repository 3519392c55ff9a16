"""Per-phase clock64 stamps of the step kernel at a few columns (config 2)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads
from paper_2405_10923_b200.devarray import to_device
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device

N, m, ell = 1 << 20, 128, 256
W = workloads.illcond_w(N, m, 7)
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
Wd = to_device(W, "double", align_row=m)
ctx = _lib.context()
buf = torch.zeros(64, dtype=torch.int64, device="cuda")
rhqr_left_device(Wd, psi, "sqrt2", P.DOUBLE_POLICY)
names = ["entry", "pdl_wait", "phaseA(tree)", "rho sync", "scalars", "partials", "sync2", "phaseD"]
for col in (1, 32, 64, 120):
    _lib.lib().sqb_debug_step_stamps(ctx.h, buf.data_ptr(), col)
    buf.zero_()
    rhqr_left_device(Wd, psi, "sqrt2", P.DOUBLE_POLICY)
    torch.cuda.synchronize()
    b = buf.cpu().numpy().reshape(8, 8)
    for r in (0, 5):
        d = [(b[r, i] - b[r, i - 1]) / 1.9e3 for i in range(1, 8)]
        print(f"col {col} rank {r}: " + " ".join(f"{names[i+1]}={d[i]:.2f}us" for i in range(7) if b[r, i + 1]))
_lib.lib().sqb_debug_step_stamps(ctx.h, None, -1)
