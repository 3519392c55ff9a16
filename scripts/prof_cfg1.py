import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200.devarray import to_device
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device
N, m, ell = 1 << 14, 32, 128
W = np.random.default_rng(1).standard_normal((N, m))
Wd = to_device(W, "double", align_row=m)
psi = _embed(P.SRHTSketch(ell, N - m, 3), N, m)
pol = P.PrecisionPolicy("double", "double")
for _ in range(3):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
e1.record(); torch.cuda.synchronize()
print("cfg1 ms/step", e0.elapsed_time(e1) / 20)
