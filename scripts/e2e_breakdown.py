"""Where the config-2 end-to-end time goes: PCIe copy rates (pinned / pageable,
one direction / both) and the phases of P.rhqr_left(host W) -> host factors."""

import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_10923_b200 as P  # noqa: E402
from paper_2405_10923_b200 import workloads  # noqa: E402
from paper_2405_10923_b200.devarray import to_device, to_numpy  # noqa: E402
from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device  # noqa: E402

GB = 1 << 30


def t_copy(dst, src, reps=5, stream=None):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def main():
    n = GB // 8
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    dev2 = torch.empty(n, dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    print(f"pinned alloc 1 GiB (first): {1e3 * (time.perf_counter() - t0):.1f} ms")
    pin2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    pin.fill_(1.0)
    pin2.fill_(1.0)
    del pin2
    t0 = time.perf_counter()
    pin2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    print(f"pinned alloc 1 GiB (cached): {1e3 * (time.perf_counter() - t0):.3f} ms")
    page = torch.from_numpy(np.ones(n))
    print(f"H2D pinned  : {GB / t_copy(dev, pin) / 1e9:.1f} GB/s")
    print(f"D2H pinned  : {GB / t_copy(pin2, dev) / 1e9:.1f} GB/s")
    print(f"H2D pageable: {GB / t_copy(dev, page, 3) / 1e9:.1f} GB/s")
    print(f"D2H pageable: {GB / t_copy(page, dev, 3) / 1e9:.1f} GB/s")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            dev.copy_(pin, non_blocking=True)
        with torch.cuda.stream(s2):
            pin2.copy_(dev2, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"bidirectional pinned: {2 * GB / dt / 1e9:.1f} GB/s aggregate ({1e3 * dt:.1f} ms per 1 GiB each way)")
    # chunked D2H (8 MiB pieces, like per-column streaming)
    ch = (8 << 20) // 8
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(0, n, ch):
        pin2[i:i + ch].copy_(dev[i:i + ch], non_blocking=True)
    torch.cuda.synchronize()
    print(f"D2H pinned 8 MiB chunks: {GB / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    del dev, dev2, pin, pin2, page

    N, m, ell = 1 << 20, 128, 256
    W = workloads.illcond_w(N, m, 7)
    om = P.SRHTSketch(ell, N - m, 8)
    Wp = torch.from_numpy(W).pin_memory()
    pol = P.PrecisionPolicy("double", "double")
    psi = _embed(om, N, m)
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Wd = to_device(Wp, "double", align_row=m)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        U, S, T, R, sg, rh, bt = rhqr_left_device(Wd, psi, "sqrt2", pol)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        Uh = to_numpy(U)
        t3 = time.perf_counter()
        _ = [to_numpy(x) for x in (S, T, R, sg, rh, bt)]
        t4 = time.perf_counter()
        print(f"iter {it}: to_device {1e3 * (t1 - t0):.1f} ms, factor {1e3 * (t2 - t1):.1f} ms, "
              f"U to_numpy {1e3 * (t3 - t2):.1f} ms, small {1e3 * (t4 - t3):.1f} ms")
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        F = P.rhqr_left(Wp, om)
        t1 = time.perf_counter()
        print(f"public rhqr_left(pinned W): {1e3 * (t1 - t0):.1f} ms")


if __name__ == "__main__":
    main()
