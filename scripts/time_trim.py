"""Trimmed RHQR (trim_rhqr_left) timing on a config-2-shaped W:
N = 2^20 x m = 128 fp64, SRHT ell = 96 < m (the trimmed variant's point),
inputs resident in HBM, CUDA events.  Algorithmic bytes per factorization:
8 N sum_c (c + 5) — the U[:, :c] GEMV read, W[:, c] read, U[:, c] write and
the three N-vector sketches the algorithm takes per column (trim.py:293-300,
103-114).  CPU: the numpy oracle on a 2^14-row sample."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2405_10923_b200 as P
from oracle import sketchqr_oracle as O

N, m, ell = int(os.environ.get("TN", 1 << 20)), 128, 96
g = torch.Generator(device="cuda").manual_seed(7)
W = (torch.randn(m, N, generator=g, device="cuda", dtype=torch.float64).t()
     * torch.logspace(0, -10, m, dtype=torch.float64, device="cuda"))
W = W.contiguous().t().contiguous().t()  # column-major view
om = P.SRHTSketch(ell, N, 8)
F = P.trim_rhqr_left(W, om)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
ts = []
for _ in range(3):
    e0.record()
    F = P.trim_rhqr_left(W, om)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
alg = 8.0 * N * sum(c + 5 for c in range(m))
Q = P.trim_thin_q(F)
res = float(torch.linalg.norm(Q @ F.R - W) / torch.linalg.norm(W))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
Ns = 1 << 14
Wh = np.random.default_rng(7).standard_normal((Ns, m)) * np.logspace(0, -10, m)
t = time.perf_counter()
O.trim_rhqr_left(Wh, O.SRHT(ell, Ns, 8))
cpu = time.perf_counter() - t
print(json.dumps({"workload": f"trim_rhqr_left {N}x{m} fp64, SRHT ell={ell}", "ms": round(ms, 3),
                  "all_ms": [round(x, 3) for x in ts], "alg_bytes": alg, "GB/s": round(alg / ms / 1e6, 1),
                  "frac_hbm": round(alg / ms / 1e6 / peak, 3), "launches_per_column": 11,
                  "residual_QR": res,
                  "cpu_oracle_sample": {"rows": Ns, "seconds": round(cpu, 3),
                                        "GB/s": round(8.0 * Ns * sum(c + 5 for c in range(m)) / cpu / 1e9, 3)}}))
