"""Time rhqr_block vs rhqr_left on the config-2 input (2^20 x 128 fp64,
SRHT ell=256) for several panel widths; diagnostics of each factorization."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_block_device, rhqr_left_device  # noqa: E402

N, m, ell = int(os.environ.get("TB_N", 1 << 20)), int(os.environ.get("TB_M", 128)), 256
W = workloads.illcond_w(N, m, 7)
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
Wd = to_device(W, "double", align_row=m)
alg = 8.0 * N * (m * m + 5 * m) / 2


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timeit(lambda: rhqr_left_device(Wd, psi, "sqrt2", P.DOUBLE_POLICY, check=False))
print(f"rhqr_left           {ms:8.3f} ms  ({alg / ms / 1e6:7.0f} GB/s of rhqr_left algorithmic bytes)")
for bs in [int(x) for x in os.environ.get("TB_BS", "16,32,64").split(",")]:
    ms = timeit(lambda: rhqr_block_device(Wd, psi, bs, "sqrt2", P.DOUBLE_POLICY, check=False))
    B = P.rhqr_block(Wd, om, block_size=bs)
    F = B.stacked()
    Q = P.thin_q(F)
    fro = P.factorization_errors(Wd, Q, F.R).fro_rel_err
    orth = P.orthogonality_error(P.sketch_q(F))
    print(f"rhqr_block bs={bs:3d}  {ms:8.3f} ms  ({alg / ms / 1e6:7.0f} GB/s-equivalent)  "
          f"|W-QR|/|W| {fro:.2e}  orth {orth:.2e}")
