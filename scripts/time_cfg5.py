"""Time one RHQR-GMRES(200) cycle of config 5 (2048^2 convection-diffusion CSR, SRHT ell=400)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import workloads

k = int(os.environ.get("GRID", 2048)); m = int(os.environ.get("M", 200)); ell = 400
t0 = time.time()
indptr, indices, data = workloads.convection_diffusion_csr(k)
N = k * k
A = P.CSRMatrix(indptr, indices, data, N)
print(f"CSR {N} rows nnz {A.nnz} built in {time.time()-t0:.1f}s")
b = torch.from_numpy(np.random.default_rng(11).standard_normal(N)).cuda()
om = P.SRHTSketch(ell, N - m - 1, 12)
x, h = P.rhqr_gmres(A, b, None, m, om); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
reps = 3
e0.record()
for _ in range(reps):
    x, h = P.rhqr_gmres(A, b, None, m, om)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = sum(8 * N * (2 * j + 5) for j in range(1, m + 1)) + m * (12 * A.nnz + 12 * N)
print(f"GMRES({m}) cycle: {ms:.2f} ms, alg bytes {alg/1e12:.3f} TB -> {alg/ms/1e6:.0f} GB/s; "
      f"resid {float(h[0]):.3e} -> {float(h[-1]):.3e}")
tol = float(os.environ.get("TOL", 1e-8))
t0 = time.time(); xr, hs = P.rhqr_gmres_restarted(A, b, None, m, om, tol=tol, max_cycles=int(os.environ.get("CYC", 3)))
torch.cuda.synchronize()
dt = time.time() - t0
true = float(torch.linalg.norm(b - A.matvec(xr)) / torch.linalg.norm(b))
print(f"restarted GMRES({m}) to tol {tol:g}: {len(hs)} cycles in {dt:.1f} s ({dt / len(hs) * 1e3:.1f} ms/cycle), "
      f"true relative residual {true:.3e}, last sketched residual {float(hs[-1][-1]):.3e}")
