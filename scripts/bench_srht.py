"""K1 alone: Y = Omega X for X (n x k) resident in HBM (SRHT apply, bit-exact)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib
from paper_2405_10923_b200.devarray import CODES, empty_colmajor, ld_of

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for (n, ell, k, tag) in [((1 << 20) - 128, 256, 128, "double"), ((1 << 22) - 201, 400, 16, "double"),
                         ((1 << 24) - 256, 512, 16, "bf16"), ((1 << 20) - 128, 256, 1, "double")]:
    om = P.SRHTSketch(ell, n, 8)
    X = empty_colmajor(n, k, tag)
    X.copy_(torch.randn(n, k, device="cuda", dtype=torch.float64).to(X.dtype))
    Y = empty_colmajor(ell, k, "double")
    ctx = _lib.context()
    d = om.desc()
    f = lambda: ctx.check(_lib.lib().sqb_sketch_apply(ctx.h, d, CODES[tag], X.data_ptr(), ld_of(X), k,
                                                      Y.data_ptr(), ld_of(Y)), "apply")
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 20
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    b = X.element_size() * n * k + 8 * ell * k
    print(f"SRHT apply n={n} ell={ell} k={k} {tag}: {ms*1e3:.1f} us, {b/ms/1e6:.0f} GB/s = {b/ms/1e6/peak:.2f} of measured HBM")
