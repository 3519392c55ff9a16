"""In-stream kernel times (sqb_ctx_trace) of the Krylov extras and the
row-partitioned (virtual-rank) paths at config shapes: arnoldi_q, the dense
and callable operators, the row-partitioned rhqr_left with 8 virtual ranks
(copy and peer-memory exchange) and the row-partitioned Arnoldi."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads, dist as D
from paper_2405_10923_b200.devarray import to_device

ctx = _lib.context()


def trace(name, fn, reps=1):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    _lib.lib().sqb_ctx_trace(ctx.h, 1)
    fn()
    buf = ctypes.create_string_buffer(1 << 16)
    _lib.lib().sqb_ctx_trace_read(ctx.h, buf, len(buf))
    _lib.lib().sqb_ctx_trace(ctx.h, 0)
    rows = [l.split() for l in buf.value.decode().splitlines()]
    tot = sum(float(r[-1]) for r in rows)
    print(f"== {name}: {wall:.3f} ms wall; library kernels in-stream {tot:.3f} ms")
    for r in sorted(rows, key=lambda r: -float(r[-1]))[:7]:
        nm, n, t = " ".join(r[:-2]), int(r[-2]), float(r[-1])
        print(f"     {nm:30s} {n:5d} {t:9.3f} ms {t / max(tot, 1e-9) * 100:5.1f}%  {t / n * 1e3:8.2f} us/launch")


# Krylov, 1024^2 grid, m = 50
k, m, ell = 1024, 50, 128
indptr, indices, data = workloads.convection_diffusion_csr(k)
n = k * k
A = P.CSRMatrix(indptr, indices, data, n)
b = torch.from_numpy(np.random.default_rng(11).standard_normal(n)).cuda()
om = P.SRHTSketch(ell, n - m - 1, 12)
trace("rhqr_arnoldi (CSR, store_q)", lambda: P.rhqr_arnoldi(A, b, None, m, om, store_q=True))
bun = P.rhqr_arnoldi(A, b, None, m, om, store_q=False)
trace("arnoldi_q", lambda: P.arnoldi_q(bun))
trace("rhqr_gmres", lambda: P.rhqr_gmres(A, b, None, m, om))
bh = b.cpu().numpy()
import scipy.sparse as sp
As = sp.csr_matrix((data, indices, indptr), shape=(n, n))
trace("rhqr_gmres_virtual P=8", lambda: D.rhqr_gmres_virtual(As, bh, None, m, om, 8))
del bun
torch.cuda.empty_cache()
# row-partitioned rhqr_left, config-2 shape, 8 virtual ranks
N, mm, el = 1 << 20, 128, 256
W = workloads.illcond_w(N, mm, 7)
Wd = to_device(W, "double", align_row=mm)
om2 = P.SRHTSketch(el, N - mm, 8)
trace("rhqr_left 1 GPU", lambda: P.rhqr_left(Wd, om2))
trace("rhqr_left_virtual P=8 (copy exchange)", lambda: D.rhqr_left_virtual(W, om2, 8))
trace("rhqr_left_virtual P=8 (p2p exchange)", lambda: D.rhqr_left_virtual(W, om2, 8, exchange="p2p"))
