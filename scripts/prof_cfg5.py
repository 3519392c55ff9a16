"""Config 5 (one RHQR-GMRES(200) cycle, 2048^2 CSR, SRHT 400) twice, for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import workloads

k = int(os.environ.get("GRID", 2048)); m = int(os.environ.get("M", 200)); ell = 400
indptr, indices, data = workloads.convection_diffusion_csr(k)
N = k * k
A = P.CSRMatrix(indptr, indices, data, N)
b = torch.from_numpy(np.random.default_rng(11).standard_normal(N)).cuda()
om = P.SRHTSketch(ell, N - m - 1, 12)
for _ in range(int(os.environ.get("REPS", 2))):
    x, h = P.rhqr_gmres(A, b, None, m, om)
torch.cuda.synchronize()
