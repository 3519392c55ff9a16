"""A/B of the recRHQR reconstruction solve (SQB_TRSM_BASE=1: the round-1
blocked kernel) on config 3, interleaved in one process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402

N, m, ell = 1 << 22, 64, 256
Wd = to_device(workloads.gen_cmatrix(N, m), "double", align_row=m)
om = P.GaussianSketch(ell, N - m, 3)
res = {"pipe": [], "base": []}
outs = {}
for rep in range(4):
    for v in res:
        if v == "base":
            os.environ["SQB_TRSM_BASE"] = "1"
        else:
            os.environ.pop("SQB_TRSM_BASE", None)
        F = P.rec_rhqr(Wd, om)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F = P.rec_rhqr(Wd, om)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1))
        outs[v] = F.U
d = (outs["pipe"] - outs["base"]).norm() / outs["base"].norm()
print(f"rel diff U pipe vs base: {float(d):.3e}")
for v, xs in res.items():
    print(f"{v}: best {min(xs):.3f} ms all {[round(x, 3) for x in xs]}")
