"""Config 4 (bf16 2^24 x 256, SRHT 512) rhqr_left on device, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200.devarray import to_device
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device
N, m, ell = int(os.environ.get("PN", 1 << 24)), 256, 512
g = torch.Generator(device="cuda").manual_seed(7)
scales = torch.logspace(0, -8, m, dtype=torch.float64, device="cuda")
W = (torch.randn(m, N, generator=g, device="cuda").t().double() * scales).float().bfloat16()
Wd = to_device(W, "bf16", align_row=m)
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
pol = P.PrecisionPolicy("double", "bf16")
for r in range(int(os.environ.get("REPS", 1))):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=(r == 0))
torch.cuda.synchronize()
