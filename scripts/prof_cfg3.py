import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import workloads
from paper_2405_10923_b200.devarray import to_device
N, m, ell = 1 << 22, 64, 256
W = workloads.gen_cmatrix(N, m)
Wd = to_device(W, "double", align_row=m)
om = P.GaussianSketch(ell, N - m, 8); om.desc()
for _ in range(int(os.environ.get("REPS", 2))):
    F = P.rec_rhqr(Wd, om)
torch.cuda.synchronize()
