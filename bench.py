"""Benchmark: left-looking RHQR (BASELINE config 2) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full `rhqr_left` of W (2^20 x 128 fp64, ill-conditioned,
sigma = logspace(0, -15)) with an SRHT of ell = 256 — the configuration
BASELINE.json's metric is quoted on.  Prints ONE JSON line on rank 0.

value   effective HBM GB/s = algorithmic bytes (8 N (m^2 + 5m)/2)
        x ranks / max-over-ranks device time of the K timed steps, W resident
        in HBM (1 GiB W + 1 GiB U exceed the 126 MB L2, so no flush is needed).
e2e     the same metric through the public API with host numpy input and host
        numpy factors returned (H2D of W and D2H of U, S, T, R inside the timer).
roofline  the dominant kernel (rhqr_col_kernel, the fused GEMV + SRHT-leaf pass)
        timed per launch with CUDA events on its own stream during the timed
        steps; peak = MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle port (oracle/sketchqr_oracle.py, restating the
        reference's numpy code) on a bounded sample (2^17 rows, same m, ell).

Multi-GPU (torchrun): every rank factors its own W (replicas, weak scaling);
the row-partitioned version is the next step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(N=1 << 20, m=128, ell=256, w_seed=7, sketch_seed=8)
CPU_SAMPLE_N = 1 << 17
METRIC = "rhqr_left effective HBM GB/s (config 2: W 2^20 x 128 fp64, SRHT ell=256)"


def alg_bytes(N, m, b=8):
    return b * N * (m * m + 5 * m) / 2.0


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_run(N, m, ell, w_seed, sketch_seed):
    from oracle import sketchqr_oracle as O
    from paper_2405_10923_b200 import workloads

    W = workloads.illcond_w(N, m, w_seed)
    om = O.SRHT(ell, N - m, sketch_seed)
    t0 = time.perf_counter()
    O.rhqr_left(W, om)
    return time.perf_counter() - t0


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on the host
    cores, rank 0 only; bounded sample per step."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    N, m, ell = CPU_SAMPLE_N, CFG["m"], CFG["ell"]
    for _ in range(args.warmup):
        cpu_oracle_run(N, m, ell, CFG["w_seed"], CFG["sketch_seed"])
    ts = [cpu_oracle_run(N, m, ell, CFG["w_seed"], CFG["sketch_seed"]) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    v = alg_bytes(N, m) / t / 1e9
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: W = A diag(logspace(0,-15,128)) B, A/B orthonormalised seeded Gaussians",
        "config": {"workload": f"rhqr_left cfg2 shape, CPU sample N=2^{N.bit_length() - 1} x 128, SRHT ell=256",
                   "N": N, "m": m, "ell": ell},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"full rhqr_left on N={N} rows (config-2 m, ell, sigma); "
                                   "numpy oracle restating sketchqr (FWHT single-threaded, BLAS "
                                   f"{cores} threads)"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2405_10923_b200 as P
    from paper_2405_10923_b200 import _lib, workloads
    from paper_2405_10923_b200.devarray import to_device
    from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    N, m, ell = CFG["N"], CFG["m"], CFG["ell"]
    W = workloads.illcond_w(N, m, CFG["w_seed"] + rank)
    om = P.SRHTSketch(ell, N - m, CFG["sketch_seed"])
    psi = _embed(om, N, m)
    pol = P.DOUBLE_POLICY
    Wd = to_device(W, "double", align_row=m)
    ctx = _lib.context()
    stream = torch.cuda.current_stream()

    def step(check=False):
        return rhqr_left_device(Wd, psi, "sqrt2", pol, check=check)

    for i in range(args.warmup):
        step(check=(i == 0))
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    l0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = ctx.launches() - l0
    # roofline pass: the same K steps again with every launch of the dominant
    # kernel bracketed by CUDA events on its stream (kept out of `value`)
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    k_ms, k_bytes, k_n = ctx.profile_read()
    ctx.profile(False)
    prof_step_ms = p0.elapsed_time(p1) / args.steps
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = alg_bytes(N, m) * ws / (ms_step * 1e-3) / 1e9

    # end-to-end through the public API: host numpy in, host numpy factors out
    e2e = None
    if not args.no_e2e:
        Wp = torch.from_numpy(W).pin_memory()
        P.rhqr_left(Wp, om)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = max(2, min(args.steps, 5))
        for _ in range(reps):
            F = P.rhqr_left(Wp, om)
            _ = float(F.R[0, 0])
        dt = (time.perf_counter() - t0) / reps
        d2h = 8 * (N * m + (m + ell) * m + 2 * m * m + 3 * m)
        e2e = {"value": alg_bytes(N, m) / dt / 1e9, "unit": "GB/s", "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": 8 * N * m, "d2h_bytes_per_step": d2h,
               "note": "P.rhqr_left(pinned host W) -> host numpy U,S,T,R; wall clock incl. copies"}

    peak, peak_kind = measured_peak()
    achieved = (k_bytes / k_n) / (k_ms / k_n * 1e-3) / 1e9 if k_n else None
    prof_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = None
    try:
        with open(prof_path) as f:
            tj = json.load(f)
            traffic = {"bytes_per_launch": tj.get("rhqr_col_kernel_bytes_per_launch_c64"),
                       "alg_bytes_per_launch": tj.get("rhqr_col_kernel_alg_bytes_c64"),
                       "launch": "column c=64 (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"}
    except Exception:
        pass

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        t = cpu_oracle_run(CPU_SAMPLE_N, m, ell, CFG["w_seed"], CFG["sketch_seed"])
        cores = blas_threads()
        cpu = {"value": alg_bytes(CPU_SAMPLE_N, m) / t / 1e9, "unit": "GB/s", "cores": cores,
               "kind": "port", "seconds": t,
               "sample": f"full rhqr_left on N={CPU_SAMPLE_N} rows x 128, SRHT 256 (config-2 shape at "
                         "1/8 rows); numpy oracle port of sketchqr (FWHT single-threaded, "
                         f"BLAS {cores} threads)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: W = A diag(logspace(0,-15,128)) B, A/B orthonormalised seeded Gaussians",
            "config": {"workload": "rhqr_left cfg2: W 2^20 x 128 fp64 ill-conditioned, SRHT ell=256",
                       "N": N, "m": m, "ell": ell, "w_seed": CFG["w_seed"],
                       "sketch_seed": CFG["sketch_seed"],
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "l2": "no flush: W (1 GiB) and U (1 GiB) exceed the 126 MB L2",
                       "alg_bytes_per_step": alg_bytes(N, m)},
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "rhqr_col_kernel (fused GEMV over U[:, :c] + lazy scale + SRHT leaves)",
                         "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                         "kernel_share_of_step": (k_ms / args.steps) / prof_step_ms if prof_step_ms else None,
                         "timing": "per-launch CUDA events on the library stream over K extra steps",
                         "launches_timed": k_n},
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
