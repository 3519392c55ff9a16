"""Config-3 sketch GEMM only (G 256 x (2^22-64) times W2), for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200.devarray import empty_colmajor
N, m, ell = 1 << 22, 64, 256
n = N - m
om = P.GaussianSketch(ell, n, 3)
X = empty_colmajor(n, m, "double")
X.copy_(torch.randn(n, m, device="cuda", dtype=torch.float64))
for _ in range(int(os.environ.get("REPS", 2))):
    Y = om.apply(X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); Y = om.apply(X); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"dense sketch {ms:.3f} ms -> {2*ell*n*m/ms/1e9:.1f} TFLOP/s")
