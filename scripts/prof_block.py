"""One rhqr_block call on the config-2 input (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_block_device  # noqa: E402

N, m, ell = 1 << 20, 128, 256
bs = int(os.environ.get("PB_BS", 32))
W = workloads.illcond_w(N, m, 7)
om = P.SRHTSketch(ell, N - m, 8)
psi = _embed(om, N, m)
Wd = to_device(W, "double", align_row=m)
torch.cuda.synchronize()
rhqr_block_device(Wd, psi, bs, "sqrt2", P.DOUBLE_POLICY, check=True)
torch.cuda.synchronize()
