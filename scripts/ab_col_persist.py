"""(Historical: the SQB_COL_PERSIST switch and the tile loop were removed after this
A/B.)  A/B of the column-pass grid (SQB_COL_PERSIST=1: one wave of CTAs walking
the tiles in a static stride; 0: one CTA per tile), interleaved in one
process, bitwise check of R and U between the two."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

TD = {"double": torch.float64, "bf16": torch.bfloat16, "single": torch.float32}
cases = [("bf16", 24, 256, 512), ("single", 24, 256, 512), ("double", 24, 256, 512), ("double", 20, 128, 256),
         ("bf16", 23, 256, 512)]
sel = os.environ.get("CASES")
if sel:
    cases = [cases[int(i)] for i in sel.split(",")]
for tag, lN, m, ell in cases:
    N = 1 << lN
    g = torch.Generator(device="cuda").manual_seed(7)
    scales = torch.logspace(0, -8, m, dtype=torch.float64, device="cuda")
    W = (torch.randn(m, N, generator=g, device="cuda").t().double() * scales).to(TD[tag])
    Wd = to_device(W, tag, align_row=m)
    del W
    om = P.SRHTSketch(ell, N - m, 8)
    psi = _embed(om, N, m)
    pol = P.PrecisionPolicy("double", tag)
    alg = Wd.element_size() * N * (m * m + 5 * m) / 2
    res = {"1": [], "0": []}
    ref = None
    for rep in range(3):
        for v in ("1", "0"):
            os.environ["SQB_COL_PERSIST"] = v
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
            e1.record()
            torch.cuda.synchronize()
            res[v].append(e0.elapsed_time(e1))
            if rep == 0:
                cur = (out[3].clone(), out[0].float().sum().item(), out[0][-4096:].clone())
                if ref is None:
                    ref = cur
                else:
                    assert torch.equal(cur[0], ref[0]) and cur[1] == ref[1] and torch.equal(cur[2], ref[2]), \
                        f"{tag} 2^{lN}: persistent grid changed the factors"
            del out
    for v in ("1", "0"):
        best = min(res[v][1:])
        print(f"{tag:6s} N=2^{lN} m={m} ell={ell} persist={v}: best {best:8.2f} ms ({alg / best / 1e6:6.0f} GB/s)"
              f" all {[round(x, 2) for x in res[v]]}", flush=True)
    del Wd
    torch.cuda.empty_cache()
