"""Effective rhqr_left rate vs N, m and storage format (is the bf16 loss a
multi-wave / large-N effect or a 2-byte-format effect?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

TD = {"double": torch.float64, "bf16": torch.bfloat16, "single": torch.float32}
for tag, lN, m, ell in [("double", 20, 128, 256), ("double", 22, 128, 256), ("double", 24, 128, 256),
                        ("double", 22, 256, 512), ("double", 24, 256, 512),
                        ("bf16", 22, 256, 512), ("bf16", 24, 256, 512), ("bf16", 25, 128, 256),
                        ("bf16", 24, 128, 256), ("single", 24, 256, 512)]:
    N = 1 << lN
    g = torch.Generator(device="cuda").manual_seed(7)
    W = torch.randn(m, N, generator=g, device="cuda").t()
    Wd = to_device(W.to(TD[tag]), tag, align_row=m)
    del W
    om = P.SRHTSketch(ell, N - m, 8)
    psi = _embed(om, N, m)
    pol = P.PrecisionPolicy("double", tag)
    b = Wd.element_size()
    alg = b * N * (m * m + 5 * m) / 2
    ts = []
    for r in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rhqr_left_device(Wd, psi, "sqrt2", pol, check=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[1:])
    print(f"{tag:6s} N=2^{lN} m={m} ell={ell}: {t:8.2f} ms  {alg / t / 1e6:6.0f} GB/s  tiles={N // (4096 if b == 8 else 8192)}",
          flush=True)
    del Wd
    torch.cuda.empty_cache()
