"""In-stream time of every kernel of one RHQR-GMRES(200) cycle (config 5),
from events recorded after each launch (sqb_ctx_trace): launch gap + run, as
issued.  Compare with the cold, serialised ncu launch list."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads

k = int(os.environ.get("GRID", 2048)); m = int(os.environ.get("M", 200)); ell = 400
indptr, indices, data = workloads.convection_diffusion_csr(k)
N = k * k
A = P.CSRMatrix(indptr, indices, data, N)
b = torch.from_numpy(np.random.default_rng(11).standard_normal(N)).cuda()
om = P.SRHTSketch(ell, N - m - 1, 12)
ctx = _lib.context()
for _ in range(2):
    x, h = P.rhqr_gmres(A, b, None, m, om)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); x, h = P.rhqr_gmres(A, b, None, m, om); e1.record(); torch.cuda.synchronize()
print(f"untraced cycle: {e0.elapsed_time(e1):.2f} ms")
_lib.lib().sqb_ctx_trace(ctx.h, 1)
x, h = P.rhqr_gmres(A, b, None, m, om)
buf = ctypes.create_string_buffer(1 << 16)
_lib.lib().sqb_ctx_trace_read(ctx.h, buf, len(buf))
_lib.lib().sqb_ctx_trace(ctx.h, 0)
rows = [l.split() for l in buf.value.decode().splitlines()]
tot = sum(float(r[-1]) for r in rows)
print(f"traced cycle: {tot:.2f} ms in {sum(int(r[-2]) for r in rows)} marks")
for r in sorted(rows, key=lambda r: -float(r[-1])):
    name, n, ms = " ".join(r[:-2]), int(r[-2]), float(r[-1])
    print(f"  {name:34s} {n:5d} {ms:9.3f} ms {ms / tot * 100:5.1f}%  {ms / n * 1e3:8.2f} us/launch")
