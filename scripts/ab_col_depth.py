"""A/B of the column-pass bulk-loop variants (SQB_COL_VARIANT) on config 4
(bf16 2^24 x 256, SRHT 512), interleaved in one process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

N, m, ell = int(os.environ.get("PN", 1 << 24)), 256, 512
g = torch.Generator(device="cuda").manual_seed(7)
scales = torch.logspace(0, -8, m, dtype=torch.float64, device="cuda")
W = (torch.randn(m, N, generator=g, device="cuda").t().double() * scales).float().bfloat16()
Wd = to_device(W, "bf16", align_row=m)
del W
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
pol = P.PrecisionPolicy("double", "bf16")
alg = 2 * N * (m * m + 5 * m) / 2
variants = os.environ.get("VARIANTS", "base,ring").split(",")
res = {v: [] for v in variants}
ref = None
for rep in range(4):
    for v in variants:
        os.environ["SQB_COL_VARIANT"] = v
        rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1))
        R = out[3].clone()
        if ref is None:
            ref = R
        assert torch.equal(R, ref), f"variant {v} changed R"
for v in variants:
    best = min(res[v])
    print(f"variant {v}: best {best:.2f} ms ({alg / best / 1e6:.0f} GB/s), all {[round(x, 2) for x in res[v]]}")
