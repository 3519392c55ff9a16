"""One warm-up + one profiled config-2 rhqr_left (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

N = int(os.environ.get("PROF_N", 1 << 20))
m = int(os.environ.get("PROF_M", 128))
ell = int(os.environ.get("PROF_ELL", 256))
reps = int(os.environ.get("PROF_REPS", 2))
W = workloads.illcond_w(N, m, 7)
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
Wd = to_device(W, "double", align_row=m)
for r in range(reps):
    rhqr_left_device(Wd, psi, "sqrt2", P.DOUBLE_POLICY, check=(r == 0))
torch.cuda.synchronize()
print("launches per call", P._lib.context().launches() // reps)
