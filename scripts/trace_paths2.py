"""In-stream kernel times (sqb_ctx_trace) of the remaining §8 entry points at
config-2-like shapes: apply_reflectors_compact (1 and 16 columns),
lsq_via_implicit_q, householder_qr, upper_tri_solve, t_factor, sketch apply
variants, the stability harness."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads, experiments as E
from paper_2405_10923_b200.devarray import to_device

ctx = _lib.context()


def trace(name, fn):
    fn(); fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    _lib.lib().sqb_ctx_trace(ctx.h, 1)
    fn()
    buf = ctypes.create_string_buffer(1 << 16)
    _lib.lib().sqb_ctx_trace_read(ctx.h, buf, len(buf))
    _lib.lib().sqb_ctx_trace(ctx.h, 0)
    rows = [l.split() for l in buf.value.decode().splitlines()]
    tot = sum(float(r[-1]) for r in rows)
    print(f"== {name}: {wall:.3f} ms wall (host + device); library kernels in-stream {tot:.3f} ms")
    for r in sorted(rows, key=lambda r: -float(r[-1]))[:6]:
        nm, n, t = " ".join(r[:-2]), int(r[-2]), float(r[-1])
        print(f"     {nm:30s} {n:5d} {t:9.3f} ms {t / max(tot, 1e-9) * 100:5.1f}%  {t / n * 1e3:8.2f} us/launch")


N, m, ell = 1 << 20, 128, 256
W = workloads.illcond_w(N, m, 7)
Wd = to_device(W, "double", align_row=m)
om = P.SRHTSketch(ell, N - m, 8)
F = P.rhqr_left(Wd, om)
g = torch.Generator(device="cuda").manual_seed(1)
x1 = torch.randn(N, generator=g, device="cuda", dtype=torch.float64)
X16 = torch.randn(16, N, generator=g, device="cuda", dtype=torch.float64).t()
trace("apply_reflectors_compact 1 col", lambda: P.apply_reflectors_compact(F.U, F.S, F.T, x1, F.psi))
trace("apply_reflectors_compact 16 cols", lambda: P.apply_reflectors_compact(F.U, F.S, F.T, X16, F.psi))
trace("apply_reflectors_compact 16 cols, T^t", lambda: P.apply_reflectors_compact(F.U, F.S, F.T, X16, F.psi, transpose_t=True))
trace("lsq_via_implicit_q", lambda: P.lsq_via_implicit_q(F, x1))
trace("psi.apply 16 cols (embedded)", lambda: F.psi.apply(X16))
Ah = torch.randn(64, 4096, generator=g, device="cuda", dtype=torch.float64).t()
trace("householder_qr 4096 x 64", lambda: P.householder_qr(Ah))
Rr = torch.triu(torch.randn(128, 128, generator=g, device="cuda", dtype=torch.float64)) + 10 * torch.eye(128, device="cuda", dtype=torch.float64)
B = torch.randn(128, 16, generator=g, device="cuda", dtype=torch.float64)
trace("upper_tri_solve 128 x 16", lambda: P.upper_tri_solve(Rr, B))
trace("t_factor_from_sketches", lambda: P.t_factor_from_sketches(F.S))
Wh = workloads.gen_cmatrix(1 << 18, 64)
for algo in ("rhqr-left", "rec-rhqr", "hqr"):
    cfg = E.ExperimentConfig(algo=algo, ell=256, every=16, seed=8)
    trace(f"run_factor_experiment {algo} 2^18 x 64 (every 16)", lambda: E.run_factor_experiment(Wh, cfg))
