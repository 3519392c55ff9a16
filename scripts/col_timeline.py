"""Block timeline of one column pass inside the running pipeline (config 4 by
default): SM id and globaltimer stamps of every block (sqb_debug_col_stamps).
Prints how long the SM slots sit empty and where the blocks wait."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads
from paper_2405_10923_b200.devarray import to_device
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device

cfg = os.environ.get("CFG", "4")
if cfg == "4":
    N, m, ell, tag = int(os.environ.get("PN", 1 << 24)), 256, 512, "bf16"
    g = torch.Generator(device="cuda").manual_seed(7)
    scales = torch.logspace(0, -8, m, dtype=torch.float64, device="cuda")
    W = (torch.randn(m, N, generator=g, device="cuda").t().double() * scales).float().bfloat16()
    pol = P.PrecisionPolicy("double", "bf16")
    tile = 8192
else:
    N, m, ell, tag = 1 << 20, 128, 256, "double"
    W = workloads.illcond_w(N, m, 7)
    pol = P.DOUBLE_POLICY
    tile = 4096
Wd = to_device(W, tag, align_row=m)
psi = _embed(P.SRHTSketch(ell, N - m, 8), N, m)
ctx = _lib.context()
nb = (N - m + tile - 1) // tile + 2
buf = torch.zeros(8 * nb + 8, dtype=torch.int64, device="cuda")
rhqr_left_device(Wd, psi, "sqrt2", pol)
for col in [int(x) for x in os.environ.get("COLS", "16,64,128,200").split(",")]:
    outs = []
    for cc in (col, col + 1):
        _lib.lib().sqb_debug_col_stamps(ctx.h, buf.data_ptr(), cc)
        buf.zero_()
        rhqr_left_device(Wd, psi, "sqrt2", pol)
        torch.cuda.synchronize()
        outs.append(buf.cpu().numpy().copy())
    _lib.lib().sqb_debug_col_stamps(ctx.h, None, -1)
    b = outs[0][: 8 * nb].reshape(nb, 8)
    st = outs[0][8 * nb: 8 * nb + 3]
    t0 = b[:, 1].min()
    sm, ent, fl, bulk, wt, ex = (b[:, i] for i in range(6))
    tiles = b[2:]
    print(f"col {col}: pass span {(ex.max() - t0) / 1e3:.1f} us; entry spread of blocks "
          f"{(ent.max() - t0) / 1e3:.1f} us; step {col}: entry {(st[0] - t0) / 1e3:.1f} wait-done {(st[1] - t0) / 1e3:.1f} "
          f"exit {(st[2] - t0) / 1e3:.1f} us")
    d = tiles
    print(f"   tile blocks: flag wait {np.mean(d[:,2]-d[:,1])/1e3:.2f} us, bulk {np.mean(d[:,3]-d[:,2])/1e3:.1f} us, "
          f"pdl wait {np.mean(d[:,4]-d[:,3])/1e3:.1f} us (max {np.max(d[:,4]-d[:,3])/1e3:.1f}), tail {np.mean(d[:,5]-d[:,4])/1e3:.1f} us; "
          f"helper {(b[0,5]-b[0,4])/1e3:.1f} us after its wait (entry {(b[0,1]-t0)/1e3:.1f})")
    # busy slot-time / (slots * span)
    busy = np.sum(tiles[:, 5] - tiles[:, 1])
    last = int(np.argmax(ex))
    print(f"   last block to exit: {last} of {nb} (entry {(ent[last]-t0)/1e3:.1f}, exit {(ex[last]-t0)/1e3:.1f} us); helper wait-done {(b[0,4]-t0)/1e3:.1f}")
    slots = 148 * (3 if cfg == "4" else 2)
    print(f"   slot occupancy {busy / (slots * (ex.max() - t0)):.3f}; quantiles of block exit (us): "
          + " ".join(f"{np.quantile(ex - t0, q) / 1e3:.0f}" for q in (0.1, 0.5, 0.9, 0.99, 1.0))
          + "; entry: " + " ".join(f"{np.quantile(ent - t0, q) / 1e3:.0f}" for q in (0.1, 0.5, 0.9, 0.99, 1.0)))
    # next pass relative
    b2 = outs[1][: 8 * nb].reshape(nb, 8)
    print(f"   (second run) pass {col+1} first entry .. last exit: {(b2[:,5].max() - b2[:,1].min()) / 1e3:.1f} us")
