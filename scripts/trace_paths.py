"""In-stream kernel times (sqb_ctx_trace) of the factorization variants next
to the hot path, on the config-2 input (2^20 x 128 fp64, SRHT 256):
rhqr_block, rhqr_right, trim_rhqr_left, thin_q, sketch_q, rec_rhqr (2^22 x 64)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads
from paper_2405_10923_b200.devarray import to_device

ctx = _lib.context()


def trace(name, fn, alg_bytes=None):
    fn(); fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    _lib.lib().sqb_ctx_trace(ctx.h, 1)
    fn()
    buf = ctypes.create_string_buffer(1 << 16)
    _lib.lib().sqb_ctx_trace_read(ctx.h, buf, len(buf))
    _lib.lib().sqb_ctx_trace(ctx.h, 0)
    rows = [l.split() for l in buf.value.decode().splitlines()]
    tot = sum(float(r[-1]) for r in rows)
    extra = f", {alg_bytes / ms / 1e6:.0f} GB/s of its algorithmic bytes" if alg_bytes else ""
    print(f"== {name}: {ms:.3f} ms untraced{extra}; traced {tot:.3f} ms")
    for r in sorted(rows, key=lambda r: -float(r[-1]))[:8]:
        nm, n, t = " ".join(r[:-2]), int(r[-2]), float(r[-1])
        print(f"     {nm:30s} {n:5d} {t:9.3f} ms {t / tot * 100:5.1f}%  {t / n * 1e3:8.2f} us/launch")


N, m, ell = 1 << 20, 128, 256
W = workloads.illcond_w(N, m, 7)
Wd = to_device(W, "double", align_row=m)
om = P.SRHTSketch(ell, N - m, 8)
alg = 8.0 * N * (m * m + 5 * m) / 2
trace("rhqr_left", lambda: P.rhqr_left(Wd, om), alg)
trace("rhqr_block bs=32", lambda: P.rhqr_block(Wd, om, block_size=32), alg)
F = P.rhqr_left(Wd, om)
trace("thin_q", lambda: P.thin_q(F), 8.0 * N * m * 2)
trace("sketch_q", lambda: P.sketch_q(F))
Qd = P.thin_q(F)
trace("cond_number(Q)", lambda: P.cond_number(Qd))
trace("cond_number(W)", lambda: P.cond_number(Wd))
trace("factorization_errors", lambda: P.factorization_errors(Wd, Qd, F.R))
trace("orthogonality_error(sketch_q)", lambda: P.orthogonality_error(P.sketch_q(F)))
del Qd
Ns = 1 << 18
Ws = to_device(workloads.illcond_w(Ns, 64, 7), "double", align_row=64)
oms = P.SRHTSketch(128, Ns - 64, 8)
trace("rhqr_right 2^18 x 64", lambda: P.rhqr_right(Ws, oms), 8.0 * Ns * 64 * 64 * 1.5)
g = torch.Generator(device="cuda").manual_seed(7)
Wt = (torch.randn(m, N, generator=g, device="cuda", dtype=torch.float64).t()
      * torch.logspace(0, -10, m, dtype=torch.float64, device="cuda"))
Wt = Wt.contiguous().t().contiguous().t()
omt = P.SRHTSketch(96, N, 8)
trace("trim_rhqr_left", lambda: P.trim_rhqr_left(Wt, omt), 8.0 * N * sum(c + 5 for c in range(m)))
del Wd, Wt, F
torch.cuda.empty_cache()
N3, m3 = 1 << 22, 64
W3 = to_device(workloads.gen_cmatrix(N3, m3), "double", align_row=m3)
om3 = P.GaussianSketch(256, N3 - m3, 8)
trace("rec_rhqr 2^22 x 64 gaussian", lambda: P.rec_rhqr(W3, om3), 8.0 * N3 * m3 * 3 + 8.0 * 256 * N3)
