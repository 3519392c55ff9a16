"""Per-GPU cost of the row-partitioned rhqr_left chain, measured with a
world of ONE real rank (NCCL communicator of size 1 / IPC mailboxes of one
rank): the same kernels and launches a rank of an N-GPU weak-scaling run
issues per column (column pass, rank-local subtree, exchange, step with the
rank-order combine), without the inter-GPU latency.  Config 2 shape."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import paper_2405_10923_b200 as P
from paper_2405_10923_b200 import _lib, workloads, dist as D
from paper_2405_10923_b200.devarray import to_device

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29617")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
ctx = _lib.context()
N, m, ell = 1 << 20, 128, 256
W = workloads.illcond_w(N, m, 7)
Wd = to_device(W, "double", align_row=m)
om = P.SRHTSketch(ell, N - m, 8)


def timeit(fn, reps=5):
    fn(); fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def trace(fn):
    _lib.lib().sqb_ctx_trace(ctx.h, 1)
    fn()
    buf = ctypes.create_string_buffer(1 << 16)
    _lib.lib().sqb_ctx_trace_read(ctx.h, buf, len(buf))
    _lib.lib().sqb_ctx_trace(ctx.h, 0)
    rows = [l.split() for l in buf.value.decode().splitlines()]
    tot = sum(float(r[-1]) for r in rows)
    for r in sorted(rows, key=lambda r: -float(r[-1]))[:6]:
        nm, n, t = " ".join(r[:-2]), int(r[-2]), float(r[-1])
        print(f"     {nm:30s} {n:5d} {t:9.3f} ms {t / tot * 100:5.1f}%  {t / n * 1e3:8.2f} us/launch")


print(f"single GPU rhqr_left: {timeit(lambda: P.rhqr_left(Wd, om)):.3f} ms")
D.init_comm()
f = lambda: D.rhqr_left_distributed(Wd, om, m, check=False)
print(f"row-partitioned chain, world 1, NCCL all-gather: {timeit(f):.3f} ms")
trace(f)
D.init_p2p(m, ell)
print(f"row-partitioned chain, world 1, peer-memory mailboxes: {timeit(f):.3f} ms")
trace(f)
D.close_p2p()
dist.destroy_process_group()
