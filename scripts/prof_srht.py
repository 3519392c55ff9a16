"""One SRHT apply (K1 standalone) for ncu: fp64/fp32 2^20 x 128 (PROF_TAG=double|single) or bf16 2^24 x 16."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib
from paper_2405_10923_b200.devarray import CODES, empty_colmajor, ld_of
tag = os.environ.get("PROF_TAG", "double")
n, ell, k = ((1 << 20) - 128, 256, 128) if tag in ("double", "single") else ((1 << 24) - 256, 512, 16)
om = P.SRHTSketch(ell, n, 8)
X = empty_colmajor(n, k, tag)
X.copy_(torch.randn(n, k, device="cuda", dtype=torch.float32).to(X.dtype))
Y = empty_colmajor(ell, k, "double")
ctx = _lib.context()
d = om.desc()
for _ in range(int(os.environ.get("REPS", 2))):
    ctx.check(_lib.lib().sqb_sketch_apply(ctx.h, d, CODES[tag], X.data_ptr(), ld_of(X), k, Y.data_ptr(), ld_of(Y)), "apply")
torch.cuda.synchronize()
