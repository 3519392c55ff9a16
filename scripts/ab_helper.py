"""A/B of a column-pass switch (env var FLAG, default SQB_HELPER_FIRST) on
configs 2 and 4, interleaved in one process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402


def case(name, Wd, N, m, ell, tag, b):
    om = P.SRHTSketch(ell, N - m, 8)
    psi = _embed(om, N, m)
    pol = P.PrecisionPolicy("double", tag)
    alg = b * N * (m * m + 5 * m) / 2
    res = {"0": [], "1": []}
    for rep in range(4):
        for v in res:
            os.environ[os.environ.get("FLAG", "SQB_HELPER_FIRST")] = v
            rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
            e1.record()
            torch.cuda.synchronize()
            res[v].append(e0.elapsed_time(e1))
    for v, xs in res.items():
        print(f"{name} {os.environ.get('FLAG', 'SQB_HELPER_FIRST')}={v}: best {min(xs):.3f} ms ({alg / min(xs) / 1e6:.0f} GB/s) all {[round(x, 3) for x in xs]}")


N, m = 1 << 20, 128
Wd = to_device(workloads.illcond_w(N, m, 7), "double", align_row=m)
case("cfg2", Wd, N, m, 256, "double", 8)
del Wd
N, m = 1 << 24, 256
g = torch.Generator(device="cuda").manual_seed(7)
scales = torch.logspace(0, -8, m, dtype=torch.float64, device="cuda")
W = (torch.randn(m, N, generator=g, device="cuda").t().double() * scales).float().bfloat16()
Wd = to_device(W, "bf16", align_row=m)
del W
case("cfg4", Wd, N, m, 512, "bf16", 2)
