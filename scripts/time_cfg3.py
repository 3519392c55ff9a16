"""Time config 3 (rec_rhqr, gen_cmatrix 2^22 x 64, Gaussian ell=256) on device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import workloads

N, m, ell = 1 << 22, 64, 256
t0 = time.time(); W = workloads.gen_cmatrix(N, m); print("gen W", time.time() - t0)
om = P.GaussianSketch(ell, N - m, 3)
t0 = time.time(); om.matrix(); print("gen G (host, threads)", time.time() - t0)
Wd = torch.from_numpy(W).cuda()
F = P.rec_rhqr(Wd, om); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    F = P.rec_rhqr(Wd, om)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
flops = 2.0 * ell * (N - m) * m
print(f"rec_rhqr cfg3: {ms:.3f} ms/step (incl. layout copy of W), sketch GEMM {flops/1e9:.1f} GFLOP")
Z = om.apply(Wd[m:])
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    Z = om.apply(Wd[m:])
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"Gaussian sketch G@W2: {ms:.3f} ms -> {flops/ms/1e9:.1f} TFLOP/s fp64 (incl. W2 layout copy)")
