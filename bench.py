"""Benchmark: randomized Householder QR on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg3|cfg4|cfg5]

Default workload = BASELINE config 2: one step is a full `rhqr_left` of W
(2^20 x 128 fp64 per GPU, sigma = logspace(0,-15)) with an SRHT of ell = 256.
Prints ONE JSON line on rank 0.

value     effective HBM GB/s = algorithmic bytes (config 2: 8 N (m^2 + 5m)/2,
          SURVEY §8(d)) of the whole job / max-over-ranks device time of the
          K timed steps; inputs resident in HBM and larger than the 126 MB L2
          (no flush needed).
e2e       the same metric through the public API with pinned host input and
          host numpy factors returned (H2D + D2H inside the timer).
roofline  the dominant kernel (rhqr_col_kernel: fused GEMV + lazy scaling +
          SRHT leaves).  Its passes overlap their neighbours (PDL look-ahead,
          cross-pass flags), so `achieved` = the kernel's algorithmic bytes of
          one step / the step's CUDA-event time in the timed region (a lower
          bound of its rate); `serialised` = the same bytes over event pairs
          around every launch (K extra steps; that breaks the overlap).
          peak = MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the unmodified reference (baseline/_ref; the oracle port when it
          is absent) on a bounded sample of the same workload, on this host's
          cores, plus a 1-thread run.

Multi-GPU (torchrun, N > 1): config 2 runs the row-partitioned factorization
of a (N*2^20) x 128 W — one NCCL all-gather per column, bitwise identical to
one GPU (weak scaling); the other workloads run replicas.
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

if "reference" in sys.argv and os.environ.get("RANK", "0") == "0":
    # the reference arm uses every host core; torchrun exports OMP_NUM_THREADS=1
    # to its ranks, which must not reach the BLAS pools before numpy loads
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        if "WORLD_SIZE" in os.environ and os.environ.get(_v) == "1":
            os.environ[_v] = str(os.cpu_count() or 1)

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(N=1 << 20, m=128, ell=256, w_seed=7, sketch_seed=8)
CPU_SAMPLE_N = 1 << 17
METRIC = "rhqr_left effective HBM GB/s (config 2: W 2^20 x 128 fp64 per GPU, SRHT ell=256)"
DATA = "synthetic: W = A diag(logspace(0,-15,128)) B, A/B orthonormalised seeded Gaussians"


def alg_bytes(N, m, b=8):
    """rhqr_left algorithmic HBM bytes b*N*(m^2 + 5m)/2."""
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


def blas_threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def ref_module():
    """The UNMODIFIED reference package (`sketchqr`) installed into
    baseline/_ref (pip --target, git-ignored, travels to the GPU box), or None.
    The reference arm and cpu_baseline time it when present, else the oracle
    port (oracle/sketchqr_oracle.py; same algorithm, pinned to the reference's
    golden vectors)."""
    d = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(d, "sketchqr")):
        return None
    if d not in sys.path:
        sys.path.insert(0, d)
    try:
        import sketchqr
        from sketchqr import precision as RP
    except Exception:
        return None
    if "bf16" not in RP.PRECISIONS:  # config 4: runtime bf16 tag, SURVEY A.6 (source untouched)
        import ml_dtypes
        RP.PRECISIONS = RP.PRECISIONS + ("bf16",)
        RP.DTYPES["bf16"] = ml_dtypes.bfloat16
        RP.UNIT_ROUNDOFF["bf16"] = 2.0 ** -8
    return sketchqr


def cpu_kind():
    return "reference" if ref_module() is not None else "port"


def timed_sample(fn, threads=None):
    """Run one CPU sample, optionally with the BLAS pools limited."""
    if threads is None:
        return fn()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        return fn()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
class Workload:
    name = ""
    metric = METRIC
    dtype = "f64"
    data = DATA
    scaling = "weak"

    def cpu_sample(self):
        """(seconds, algorithmic bytes, description) of one oracle run."""
        raise NotImplementedError


class RHQRLeft(Workload):
    """rhqr_left on N x m per GPU (configs 1, 2, 4)."""

    def __init__(self, name, N, m, ell, tag, cpu_N, data, metric, w_kind):
        self.name, self.N, self.m, self.ell, self.tag = name, N, m, ell, tag
        self.cpu_N, self.data, self.metric, self.w_kind = cpu_N, data, metric, w_kind
        if tag == "double":  # config 4's full fp64-emulated size needs ~96 GB of host arrays
            self.full_N = N
        self.b = 8 if tag == "double" else 2
        self.dtype = {"double": "f64", "bf16": "bf16"}[tag]

    def make_w(self, rows, seed, device=False):
        from paper_2405_10923_b200 import workloads
        if self.w_kind == "illcond":
            return workloads.illcond_w(rows, self.m, seed)
        if self.w_kind == "gauss":
            return workloads.gaussian_w(rows, self.m, seed)
        import torch  # config 4: seeded device generator
        g = torch.Generator(device="cuda").manual_seed(seed)
        scales = torch.logspace(0, -8, self.m, dtype=torch.float64, device="cuda")
        W = torch.randn(self.m, rows, generator=g, device="cuda", dtype=torch.float32).t()
        return (W.to(torch.float64) * scales[None, :]).to(torch.float32).to(torch.bfloat16)

    def setup(self, ws, rank):
        import torch

        import paper_2405_10923_b200 as P
        from paper_2405_10923_b200 import dist as D
        from paper_2405_10923_b200.devarray import to_device
        from paper_2405_10923_b200.rhqr import _embed, rhqr_left_device
        self.ws = ws
        self.partitioned = ws > 1 and self.name in ("cfg2", "cfg4")
        Ng = self.N * ws if (self.partitioned and self.name == "cfg2") else self.N
        self.Ng = Ng
        m = self.m
        self.om = P.SRHTSketch(self.ell, Ng - m, CFG["sketch_seed"])
        pol = P.PrecisionPolicy("double", self.tag)
        if self.partitioned:
            rows = D.local_rows(Ng, m, self.om.n_pad, ws, rank, self.tag)
            W = self.make_w(len(rows), CFG["w_seed"] + rank)
            self.Wd = to_device(W, self.tag, align_row=m if rank == 0 else 0)
            D.init_comm()
            self.exchange = "nccl all-gather"
            mode = getattr(self, "exchange_mode", "auto")
            if mode in ("p2p", "auto"):
                # the exchange inside the step kernel (sqb_p2p_*: IPC mailboxes, NVLink stores, release/acquire
                # flags): two launches per column instead of four; "auto" falls back to NCCL when the mailboxes
                # cannot be set up (no peer access / IPC) — agreed on by every rank
                import torch.distributed as dist
                ok = 1
                try:
                    D.init_p2p(m, self.ell)
                except Exception as exc:  # noqa: BLE001
                    if mode == "p2p":
                        raise
                    ok = 0
                    sys.stderr.write(f"[bench] rank {rank}: peer-memory exchange unavailable ({exc}); using NCCL\n")
                flag = torch.tensor([ok], device="cuda")
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                if int(flag.item()) == 1 and mode == "auto":
                    # one trial factorization over the mailboxes with a short wait limit: a peer whose stores or
                    # flags never arrive (no NVLink path behind the mapping) shows up here as a timeout error on
                    # some rank, and every rank then falls back to NCCL together
                    try:
                        D.set_p2p_timeout(5000)
                        D.rhqr_left_distributed(self.Wd, self.om, m, policy=pol, check=True)
                        torch.cuda.synchronize()
                        D.set_p2p_timeout(0)
                    except Exception as exc:  # noqa: BLE001
                        ok = 0
                        sys.stderr.write(f"[bench] rank {rank}: peer-memory trial failed ({exc}); using NCCL\n")
                    flag = torch.tensor([ok], device="cuda")
                    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                if int(flag.item()) == 1:
                    self.exchange = "peer-memory mailboxes, exchange inside the step kernel (NVLink stores + release/acquire flags)"
                else:
                    try:
                        D.close_p2p()
                    except Exception:  # noqa: BLE001
                        pass
            self.step = lambda check=False: D.rhqr_left_distributed(self.Wd, self.om, m, policy=pol, check=check)
            self.W_host = None
        else:
            W = self.make_w(Ng, CFG["w_seed"] + rank)
            self.W_host = W if not isinstance(W, torch.Tensor) else None
            self.Wd = to_device(W, self.tag, align_row=m)
            psi = _embed(self.om, Ng, m)
            self.step = lambda check=False: rhqr_left_device(self.Wd, psi, "sqrt2", pol, check=check)
        self.pol = pol
        self.alg = alg_bytes(Ng, m, self.b)  # whole job
        self.roof_note = ("a fraction above 1 is possible: the peak is the measured COPY bandwidth (read + write) "
                          "and the pass is ~98% reads")
        self.kernel = "rhqr_col_kernel (fused GEMV over U[:, :c] + lazy scale + SRHT leaves)"
        if (not self.partitioned and self.tag == "double" and self.om.n_pad <= (1 << 16)
                and os.environ.get("SQB_PERSIST", "2") != "0"):
            self.kernel = ("rhqr_persist_fast_kernel (one cooperative grid for all columns: column pass on rows "
                           "held in shared memory, SRHT leaves, one grid barrier and a single-reduction step per column)")
        self.config = {"workload": f"rhqr_left {self.name}: W {Ng} x {m} {self.tag}, SRHT ell={self.ell}",
                       "N": Ng, "N_per_gpu": self.N, "m": m, "ell": self.ell, "w_seed": CFG["w_seed"],
                       "sketch_seed": CFG["sketch_seed"],
                       "parallelism": (f"row-partitioned x{ws} (1 exchange/column: {self.exchange})" if self.partitioned
                                       else (f"replicas x{ws}" if ws > 1 else "single GPU")),
                       "l2": ("no flush: W and U exceed the 126 MB L2" if self.b * Ng * m * 2 > 126e6 else
                              "no flush: the 8 MB working set is L2-resident by the config's size; the step is "
                              "bound by its chain of dependent column steps, not by memory"),
                       "alg_bytes_per_step": self.alg}
        if self.partitioned and self.name == "cfg4":
            self.scaling = "strong"

    def extra_kernels(self):
        """K1 standalone SRHT (the raw sketches Psi W of this workload, through
        sqb_sketch_apply, tile + tree kernels) timed live: algorithmic bytes
        b (N-m) m + 8 ell m over CUDA-event time, against the HBM peak."""
        import torch
        from paper_2405_10923_b200 import _lib
        from paper_2405_10923_b200.devarray import CODES, empty_colmajor, ld_of
        if self.partitioned:
            return None
        m, n = self.m, self.Ng - self.m
        Y = empty_colmajor(self.ell, m, "double")
        ctx = _lib.context()
        d = self.om.desc()
        esz = self.Wd.element_size()
        f = lambda: ctx.check(_lib.lib().sqb_sketch_apply(  # noqa: E731
            ctx.h, d, CODES[self.tag], self.Wd.data_ptr() + m * esz, ld_of(self.Wd), m, Y.data_ptr(), ld_of(Y)),
            "sqb_sketch_apply")
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record(s)
        for _ in range(reps):
            f()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        by = self.b * n * m + 8.0 * self.ell * m
        peak, _ = measured_peak()
        return {"srht_k1": {"what": f"standalone SRHT apply of W's {n} x {m} Omega rows ({self.tag}), "
                                    "srht_tma*_tile_kernel + srht_tree_kernel",
                            "ms": ms, "GB/s": by / ms / 1e6, "frac_hbm": by / ms / 1e6 / peak,
                            "alg_bytes": by}}

    def e2e(self, steps):
        import torch

        import paper_2405_10923_b200 as P
        if self.W_host is None or self.partitioned:
            return None
        N, m, ell = self.Ng, self.m, self.ell

        def run(Wp):
            # steady state: a caller holds the previous factors while the next call
            # runs; 4 warm-up calls leave enough page-locked U blocks in torch's
            # host cache that no timed call pays a cudaHostAlloc
            held = []
            for _ in range(4):
                held = held[-1:] + [P.rhqr_left(Wp, self.om, policy=self.pol)]
            torch.cuda.synchronize()
            reps = max(3, min(steps, 10))
            t0 = time.perf_counter()
            for _ in range(reps):
                F = P.rhqr_left(Wp, self.om, policy=self.pol)
                _ = float(F.R[0, 0])
                held = held[-1:] + [F]
            return (time.perf_counter() - t0) / reps

        # the reference's users hand over C-order numpy arrays; a column-major
        # (Fortran-order) W additionally lets the upload stream column groups
        # under the sweep (csrc/host_pipe.cu)
        dt_c = run(torch.from_numpy(np.ascontiguousarray(self.W_host)).pin_memory())
        dt_f = run(torch.from_numpy(np.asfortranarray(self.W_host).T).pin_memory().T)
        dt = dt_c  # headline: the C-order arrays the reference's users pass
        # the same call with an ordinary pageable (not page-locked) C-order ndarray: the upload goes through the
        # library's page-locked staging ring filled by host threads (host_pipe.cu: staged_h2d)
        dt_pg = run(np.array(self.W_host, order="C"))
        return {"value": self.alg / dt / 1e9, "unit": "GB/s", "ms_per_step": dt * 1e3,
                "ms_per_step_pageable_c_order_input": dt_pg * 1e3,
                "h2d_bytes_per_step": self.b * N * m if self.b == 8 else 8 * N * m,
                "d2h_bytes_per_step": 8 * (N * m + (m + ell) * m + 2 * m * m + 3 * m),
                "ms_per_step_c_order_input": dt_c * 1e3, "ms_per_step_f_order_input": dt_f * 1e3,
                "input_order": "C (headline; F-order reported beside it)",
                "note": ("P.rhqr_left(pinned host float64 W) -> host float64 U,S,T,R,scalars "
                         "(sqb_rhqr_left_host: H2D/D2H overlapped with the sweep); wall clock, "
                         "steady state (caller holds the previous result)")}

    def cpu_sample(self, N=None):
        from paper_2405_10923_b200 import workloads
        N, m = N or self.cpu_N, self.m
        if self.w_kind == "illcond":
            W = workloads.illcond_w(N, m, CFG["w_seed"])
        elif self.w_kind == "gauss":
            W = workloads.gaussian_w(N, m, CFG["w_seed"])
        else:
            W = workloads.scaled_gaussian_w(N, m, CFG["w_seed"])
        R = ref_module()
        if R is not None:  # sketchqr.rhqr_left (rhqr.py:254-267), stock code path
            om = R.SRHTSketch(self.ell, N - m, CFG["sketch_seed"])
            pol = R.PrecisionPolicy(high="double", low=self.tag)
            run = lambda: R.rhqr_left(W, om, policy=pol)  # noqa: E731
        else:
            from oracle import sketchqr_oracle as O
            om = O.SRHT(self.ell, N - m, CFG["sketch_seed"])
            pol = O.Policy("double", self.tag)
            run = lambda: O.rhqr_left(W, om, policy=pol)  # noqa: E731
        t0 = time.perf_counter()
        run()
        t = time.perf_counter() - t0
        return t, alg_bytes(N, m, self.b), (f"full rhqr_left on N={N} rows x {m} ({self.tag} storage), "
                                              f"SRHT {self.ell}")


class RecRHQR(Workload):
    """Config 3: rec_rhqr of gen_cmatrix(2^22, 64) with a Gaussian ell=256 sketch."""

    name = "cfg3"
    metric = "rec_rhqr effective GB/s (config 3: gen_cmatrix 2^22 x 64 fp64, Gaussian ell=256)"
    data = "synthetic: W = gen_cmatrix(2^22, 64) (experiments.py:86-98); G from per-row Philox (seeded)"

    def __init__(self, N=1 << 22, m=64, ell=256, cpu_N=1 << 19):
        self.N, self.m, self.ell, self.cpu_N = N, m, ell, cpu_N
        self.full_N = N

    def setup(self, ws, rank):
        import paper_2405_10923_b200 as P
        from paper_2405_10923_b200 import workloads
        from paper_2405_10923_b200.devarray import to_device
        N, m, ell = self.N, self.m, self.ell
        self.W_host = workloads.gen_cmatrix(N, m)
        self.Wd = to_device(self.W_host, "double", align_row=m)
        self.om = P.GaussianSketch(ell, N - m, CFG["sketch_seed"])
        self.om.desc()  # host Philox rows + upload (one-time, like the reference constructor)
        self.step = lambda check=False: P.rec_rhqr(self.Wd, self.om)
        n = N - m
        # read G (ell x n) and W, write U (sketch GEMM + reconstruction)
        self.alg = 8.0 * (ell * n + N * m + N * m)
        self.flops = 2.0 * ell * n * m
        self.kernel = ("dense_tma_kernel (FP64 DMMA split-K sketch GEMM: TMA tensor-map boxes on a 5-stage "
                       "mbarrier ring, one producer warp, 16 consumer warps)")
        # the sketch GEMM is tensor-bound (AI ~12.8 flop/B): its roofline is
        # the FP64 DMMA pipe, which MEASURED_PEAKS.json does not carry
        self.roof = {"bound": "tensor", "unit": "TFLOP/s", "scale": 1e12, "peak": 37.0,
                     "peak_source": "profiles/fp64_peak_b200.txt (register-only DMMA m16n8k16 probe, 36.8-37.1 "
                                    "TFLOP/s on this pool's B200s; MEASURED_PEAKS.json has no FP64 figure)"}
        self.config = {"workload": f"rec_rhqr cfg3: W {N} x {m} fp64 gen_cmatrix, Gaussian ell={ell}",
                       "N": N, "m": m, "ell": ell, "sketch_seed": CFG["sketch_seed"],
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                       "l2": "no flush: G (8.6 GB) and W (2.1 GB) exceed L2", "alg_bytes_per_step": self.alg,
                       "sketch_gflop": self.flops / 1e9}

    def e2e(self, steps):
        import torch

        import paper_2405_10923_b200 as P
        N, m, ell = self.N, self.m, self.ell

        def run(Wp):
            held = []  # as for rhqr_left: no timed call pays a page-locked allocation
            for _ in range(4):
                held = held[-1:] + [P.rec_rhqr(Wp, self.om)]
            torch.cuda.synchronize()
            reps = max(3, min(steps, 5))
            t0 = time.perf_counter()
            for _ in range(reps):
                F = P.rec_rhqr(Wp, self.om)
                _ = float(F.R[0, 0])
                held = held[-1:] + [F]
            return (time.perf_counter() - t0) / reps

        dt_c = run(torch.from_numpy(np.ascontiguousarray(self.W_host)).pin_memory())
        dt_f = run(torch.from_numpy(np.asfortranarray(self.W_host).T).pin_memory().T)
        dt = dt_c
        return {"value": self.alg / dt / 1e9, "unit": "GB/s", "ms_per_step": dt * 1e3,
                "h2d_bytes_per_step": 8 * N * m,
                "d2h_bytes_per_step": 8 * (N * m + (m + ell) * m + 2 * m * m + 3 * m),
                "ms_per_step_c_order_input": dt_c * 1e3, "ms_per_step_f_order_input": dt_f * 1e3,
                "input_order": "C (headline; F-order reported beside it)",
                "note": ("P.rec_rhqr(pinned host float64 W) -> host float64 U,S,T,R,scalars "
                         "(sqb_rec_rhqr_host: the sketch GEMM runs under the blocked upload; U downloads "
                         "after the reconstruction); wall clock, steady state")}

    def cpu_sample(self, N=None, precached=False):
        """precached: G built once through the reference's own row generator
        and placed in its `_cache` (sketching.py:110-117) before the timer, so
        the time is the GEMM + HQR + solve without the Philox regeneration."""
        from paper_2405_10923_b200 import workloads
        N, m = N or self.cpu_N, self.m
        W = workloads.gen_cmatrix(N, m)
        R = ref_module()
        if R is not None:  # sketchqr.rec_rhqr (rhqr.py:368-395); G regenerated per apply
            om = R.GaussianSketch(self.ell, N - m, CFG["sketch_seed"])
            if precached:
                om._cache[np.dtype(np.float64)] = om._rows(0, self.ell)
            run = lambda: R.rec_rhqr(W, om)  # noqa: E731
        else:
            from oracle import sketchqr_oracle as O
            run = lambda: O.rec_rhqr(W, O.Gaussian(self.ell, N - m, CFG["sketch_seed"],  # noqa: E731
                                                   materialize=precached))
        t0 = time.perf_counter()
        run()
        t = time.perf_counter() - t0
        n = N - m
        return t, 8.0 * (self.ell * n + 2 * N * m), (f"full rec_rhqr on gen_cmatrix({N}, {m}), Gaussian "
                                                      f"{self.ell} regenerated per apply as the reference does")


class GMRESCycle(Workload):
    """Config 5: one RHQR-GMRES(200) cycle on the 2048^2 convection-diffusion CSR."""

    name = "cfg5"
    metric = "rhqr_gmres effective GB/s per GMRES(200) cycle (config 5: 2048^2 convection-diffusion, SRHT 400)"
    data = "synthetic: 5-point -Laplace + (50,50).grad on 2048^2, b ~ N(0,1) (seeded)"

    def __init__(self, k=2048, m=200, ell=400):
        self.k, self.m, self.ell = k, m, ell

    def setup(self, ws, rank):
        import torch

        import paper_2405_10923_b200 as P
        from paper_2405_10923_b200 import workloads
        k, m = self.k, self.m
        indptr, indices, data = workloads.convection_diffusion_csr(k)
        N = k * k
        self.om = P.SRHTSketch(self.ell, N - m - 1, CFG["sketch_seed"])
        b = np.random.default_rng(11).standard_normal(N)
        nnz = int(indptr[-1])
        if ws > 1:
            # strong scaling: the row-partitioned Arnoldi over the same 2048^2
            # problem (q all-gather for the SpMV + two sketch all-gathers per step)
            import scipy.sparse

            from paper_2405_10923_b200 import dist as D
            D.init_comm()
            A = scipy.sparse.csr_matrix((data, indices, indptr), shape=(N, N))
            self.Al = D.local_operator(A, m, self.om.n_pad, ws, rank)
            r0, nr = self.Al[3], self.Al[4]
            bl = torch.from_numpy(b[r0:r0 + nr].copy()).cuda()
            x0l = torch.zeros(nr, dtype=torch.float64, device="cuda")

            def step(check=False):
                bun = D.rhqr_arnoldi_distributed(self.Al, bl, x0l, m, self.om, N)
                y, _ = P.hessenberg_lstsq(bun.H, bun.beta)
                return D.gmres_solution_local(bun, y, x0l, rank)
            self.step = step
            self.scaling = "strong"
        else:
            self.A = P.CSRMatrix(indptr, indices, data, N)
            self.b = torch.from_numpy(b).cuda()
            self.step = lambda check=False: P.rhqr_gmres(self.A, self.b, None, m, self.om)
        self.alg = float(sum(8 * N * (2 * j + 5) for j in range(1, m + 1)) + m * (12 * nnz + 12 * N))
        self.kernel = ("arn_q_kernel (streaming GEMV q = e_j - U_j coef over the Krylov reflectors; the "
                       "apply_reflectors update GEMV has the same shape)")
        self.host = (indptr, indices, data, b, N)
        self.roof_note = ("achieved can reach the measured peak: the GEMV is a read stream (the peak is a "
                          "read+write copy), and the reflector columns written moments earlier are partly "
                          "L2-resident")
        self.config = {"workload": f"rhqr_gmres cfg5: one GMRES({m}) cycle, {k}^2 grid CSR (nnz {nnz}), SRHT {self.ell}",
                       "N": N, "m": m, "ell": self.ell, "nnz": nnz,
                       "parallelism": (f"row-partitioned x{ws} (q all-gather + 2 sketch all-gathers per step)"
                                       if ws > 1 else "single GPU"),
                       "l2": "no flush: U (6.7 GB) exceeds L2", "alg_bytes_per_step": self.alg}

    def e2e(self, steps):
        import scipy.sparse
        import torch

        import paper_2405_10923_b200 as P
        if not hasattr(self, "A"):
            return None
        indptr, indices, data, b, N = self.host
        A = scipy.sparse.csr_matrix((data, indices, indptr), shape=(N, N))
        bp = torch.from_numpy(b).pin_memory()
        for _ in range(2):
            P.rhqr_gmres(A, bp, None, self.m, self.om)
        torch.cuda.synchronize()
        reps = max(3, min(steps, 5))
        t0 = time.perf_counter()
        for _ in range(reps):
            x, hist = P.rhqr_gmres(A, bp, None, self.m, self.om)
            _ = float(np.asarray(x)[0])
        dt = (time.perf_counter() - t0) / reps
        nnz = int(indptr[-1])
        return {"value": self.alg / dt / 1e9, "unit": "GB/s", "ms_per_step": dt * 1e3,
                "h2d_bytes_per_step": int(indptr.nbytes + indices.nbytes + data.nbytes + 8 * N),
                "d2h_bytes_per_step": 8 * N + 8 * (self.m + 1),
                "note": (f"P.rhqr_gmres(host scipy CSR ({nnz} nnz), pinned host b) -> host x and residual "
                         "history: the CSR upload is inside every timed call; wall clock")}

    def cpu_sample(self, N=None):
        import scipy.sparse

        from paper_2405_10923_b200 import workloads
        k, msamp = self.k, 8
        indptr, indices, data = workloads.convection_diffusion_csr(k)
        N = k * k
        A = scipy.sparse.csr_matrix((data, indices, indptr), shape=(N, N))
        b = np.random.default_rng(11).standard_normal(N)
        R = ref_module()
        if R is not None:  # sketchqr.rhqr_arnoldi (krylov.py:82-150)
            from sketchqr.krylov import rhqr_arnoldi
            om = R.SRHTSketch(self.ell, N - msamp - 1, CFG["sketch_seed"])
            run = lambda: rhqr_arnoldi(A, b, None, msamp, om, store_q=False)  # noqa: E731
        else:
            from oracle import sketchqr_oracle as O
            om = O.SRHT(self.ell, N - msamp - 1, CFG["sketch_seed"])
            run = lambda: O.rhqr_arnoldi(A, b, None, msamp, om, store_q=False)  # noqa: E731
        t0 = time.perf_counter()
        run()
        t = time.perf_counter() - t0
        nnz = A.nnz
        by = float(sum(8 * N * (2 * j + 5) for j in range(1, msamp + 1)) + msamp * (12 * nnz + 12 * N))
        return t, by, f"first {msamp} Arnoldi steps of the full-size cycle (oracle, {k}^2 grid)"


WORKLOADS = {
    "cfg3": lambda: RecRHQR(),
    "cfg5": lambda: GMRESCycle(),
    "cfg1": lambda: RHQRLeft("cfg1", 1 << 14, 32, 128, "double", 1 << 14,
                             "synthetic: W i.i.d. N(0,1) (seeded)",
                             "rhqr_left effective HBM GB/s (config 1: W 2^14 x 32 fp64, SRHT ell=128)", "gauss"),
    "cfg2": lambda: RHQRLeft("cfg2", CFG["N"], CFG["m"], CFG["ell"], "double", CPU_SAMPLE_N, DATA, METRIC,
                             "illcond"),
    "cfg4": lambda: RHQRLeft("cfg4", 1 << 24, 256, 512, "bf16", 1 << 14,
                             "synthetic: W N(0,1) x logspace(0,-8) column scales (device torch generator)",
                             "rhqr_left effective HBM GB/s (config 4: W 2^24 x 256 bf16, SRHT ell=512)",
                             "scaled"),
}


def cpu_desc(kind, cores):
    if kind == "reference":
        return (f"the unmodified reference package sketchqr 0.1.0 (baseline/_ref, numpy/scipy; FWHT "
                f"single-threaded numpy, BLAS {cores} threads)")
    return f"numpy oracle port of sketchqr (FWHT single-threaded, BLAS {cores} threads)"


def run_reference(args, wl):
    """--impl reference: the reference's own CPU implementation (sketchqr from
    baseline/_ref when installed, else the oracle port) on this host's cores,
    rank 0 only; each step a bounded sample of the workload."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    for _ in range(args.warmup):
        wl.cpu_sample()
    runs = [wl.cpu_sample() for _ in range(args.steps)]
    t = sum(r[0] for r in runs) / len(runs)
    v = runs[0][1] / t / 1e9
    cores = blas_threads()
    kind = cpu_kind()
    line = {
        "impl": "reference", "metric": wl.metric, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype, "data": wl.data,
        "config": {"workload": f"{wl.name} CPU sample: {runs[0][2]}"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": runs[0][2] + "; " + cpu_desc(kind, cores)},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measure(wl, steps, warmup, ws, local):
    """W warm-up steps, then exactly K timed steps bracketed by barrier +
    synchronize with CUDA events on the launching stream (max over ranks),
    clocks sampled meanwhile; then K more steps with every launch of the
    dominant kernel bracketed by events on the library stream (the roofline
    pass, kept out of `value`)."""
    import torch
    import torch.distributed as dist

    from paper_2405_10923_b200 import _lib
    ctx = _lib.context()
    stream = torch.cuda.current_stream()
    for i in range(warmup):
        wl.step(check=(i == 0))
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
    for _ in range(steps):
        wl.step()
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = ctx.launches() - l0
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / steps
    value = wl.alg / (ms_step * 1e-3) / 1e9
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(steps):
        wl.step()
    p1.record(stream)
    torch.cuda.synchronize()
    k_ms, k_bytes, k_n = ctx.profile_read()
    ctx.profile(False)
    return {"ms_step": ms_step, "value": value, "launches": launches, "clocks": clk, "k_ms": k_ms,
            "k_bytes": k_bytes, "k_n": k_n, "prof_step_ms": p0.elapsed_time(p1) / steps}


def other_configs(budget_s, local):
    """The other BASELINE configs (1, 3, 5, 4) measured in the same default
    run, device-timed like the headline (3 warm-up + 3 timed steps each, inputs
    resident in HBM and larger than L2 except config 1), so every config has a
    line from the driver's own bench run.  Bounded by `budget_s` of wall clock:
    a config that would start after the budget is reported as skipped."""
    import gc

    import torch
    out = {}
    t_start = time.perf_counter()
    peak, _ = measured_peak()
    for name in ("cfg1", "cfg3", "cfg5", "cfg4"):
        if time.perf_counter() - t_start > budget_s:
            out[name] = {"skipped": f"time budget of {budget_s:.0f} s used up"}
            continue
        try:
            t0 = time.perf_counter()
            w = WORKLOADS[name]()
            w.p2p = False
            w.setup(1, 0)
            t_setup = time.perf_counter() - t0
            steps = 20 if name == "cfg1" else 3
            r = measure(w, steps, 3, 1, local)
            roof = getattr(w, "roof", None) or {"bound": "hbm", "unit": "GB/s", "scale": 1e9, "peak": peak}
            ach = (r["k_bytes"] / r["k_n"]) / (r["k_ms"] / r["k_n"] * 1e-3) / roof["scale"] if r["k_n"] else None
            ach_ser = None
            if isinstance(w, RHQRLeft) and r["k_n"]:  # as the headline: kernel bytes of a step / the step's time
                ach_ser = ach
                ach = (r["k_bytes"] / steps) / (r["ms_step"] * 1e-3) / roof["scale"]
            out[name] = {"workload": w.config["workload"], "ms_per_step": r["ms_step"], "value": r["value"],
                         "unit": "GB/s", "frac_hbm_whole_step": r["value"] / peak, "steps": steps, "warmup": 3,
                         "dtype": w.dtype, "gpu_launches": r["launches"], "setup_s": t_setup,
                         "kernel": w.kernel, "kernel_bound": roof["bound"], "kernel_achieved": ach,
                         "kernel_unit": roof["unit"], "kernel_frac": (ach / roof["peak"]) if ach else None,
                         **({"kernel_achieved_serialised": ach_ser} if ach_ser else {}),
                         "clocks": r["clocks"]}
            del w
        except Exception as exc:  # informational: never lose the headline line
            out[name] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
        gc.collect()
        torch.cuda.empty_cache()
    return out


def relaunch_cmd(args_gpus, argv, port):
    """`bench.py --gpus N` (N > 1) started without torchrun re-executes itself
    as N ranks of one node (the contract's launch line)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args_gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p"],
                    help="row-partitioned runs (N > 1): per-column exchange by NCCL all-gather or in-kernel "
                         "peer-memory stores")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="default run (cfg2, 1 GPU): skip the short device-timed lines of configs 1, 3, 4, 5")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also time the CPU reference on the workload's full size (config 2: ~35-60 s)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-exec under torchrun (NCCL INIT log kept on so
        # the ranks are visible in the output)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        r = subprocess.run(relaunch_cmd(args.gpus, sys.argv[1:], free_port()), env=env)
        sys.exit(r.returncode)
    ws_env = int(os.environ.get("WORLD_SIZE", "1"))
    if ws_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    print(f"[bench] rank {os.environ.get('RANK', '0')}/{ws_env} impl={args.impl}", file=sys.stderr, flush=True)
    wl = WORKLOADS[args.workload]()
    wl.exchange_mode = args.exchange
    if args.impl == "reference":
        run_reference(args, wl)
        return
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist

    from paper_2405_10923_b200 import _lib

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl.setup(ws, rank)
    ctx = _lib.context()
    stream = torch.cuda.current_stream()
    meas = measure(wl, args.steps, args.warmup, ws, local)
    ms_step, value, launches, clk = meas["ms_step"], meas["value"], meas["launches"], meas["clocks"]
    k_ms, k_bytes, k_n, prof_step_ms = meas["k_ms"], meas["k_bytes"], meas["k_n"], meas["prof_step_ms"]

    e2e = None if args.no_e2e else wl.e2e(args.steps)
    peak, peak_kind = measured_peak()
    roof = getattr(wl, "roof", None) or {"bound": "hbm", "unit": "GB/s", "scale": 1e9, "peak": peak,
                                         "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)"}
    achieved = (k_bytes / k_n) / (k_ms / k_n * 1e-3) / roof["scale"] if k_n else None
    # RHQR sweeps: the column kernel overlaps its neighbours (PDL look-ahead,
    # cross-pass flags), and an event pair around every launch serialises
    # exactly that.  The headline figure is therefore the kernel's algorithmic
    # bytes of one step over the WHOLE step's time in the timed region — a lower
    # bound of the kernel's rate (the step also holds the other kernels); the
    # event-bracketed per-launch figure is kept under "serialised".
    serialised = None
    if isinstance(wl, RHQRLeft) and k_n and ms_step:
        serialised = {"achieved": achieved, "frac": achieved / roof["peak"],
                      "what": "event pair around every launch of the kernel over K extra steps (no overlap "
                              "between passes)", "profiled_step_ms": prof_step_ms}
        achieved = (k_bytes / args.steps) / (ms_step * 1e-3) / roof["scale"]
    traffic, traffic_detail = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f).get(wl.name)
        if tj:
            traffic = tj["bytes_per_launch"]
            traffic_detail = {"alg_bytes_per_launch": tj["alg_bytes_per_launch"], "launch": tj["launch"],
                              "source": "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum)"}
    except Exception:
        pass

    extra = None
    if rank == 0 and hasattr(wl, "extra_kernels"):
        try:
            extra = wl.extra_kernels()
        except Exception as exc:  # informational only
            extra = {"error": str(exc)[:200]}

    others = None
    if ws == 1 and args.workload == "cfg2" and not args.no_other_configs:
        others = other_configs(200.0, local)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        t, by, desc = wl.cpu_sample()
        cores = blas_threads()
        kind = cpu_kind()
        cpu = {"value": by / t / 1e9, "unit": "GB/s", "cores": cores, "kind": kind, "seconds": t,
               "sample": desc + "; " + cpu_desc(kind, cores)}
        t1, by1, _ = timed_sample(wl.cpu_sample, threads=1)  # also a 1-thread run
        cpu["one_thread"] = {"value": by1 / t1 / 1e9, "seconds": t1, "cores": 1}
        if isinstance(wl, RecRHQR):
            tp, byp, _ = wl.cpu_sample(precached=True)
            cpu["g_precached"] = {"value": byp / tp / 1e9, "seconds": tp,
                                  "what": "same sample with G pre-cached in GaussianSketch._cache"}
        if args.cpu_full and hasattr(wl, "full_N"):
            tf, byf, descf = wl.cpu_sample(N=wl.full_N)
            cpu["full_size"] = {"value": byf / tf / 1e9, "seconds": tf, "sample": descf}

    if rank == 0:
        line = {
            "metric": wl.metric, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": wl.dtype, "data": wl.data,
            "config": wl.config,
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": {"bound": roof["bound"], "achieved": achieved, "peak": roof["peak"], "unit": roof["unit"],
                         "frac": (achieved / roof["peak"]) if achieved else None, "traffic": traffic,
                         "traffic_detail": traffic_detail,
                         "kernel": wl.kernel,
                         "peak_source": roof["peak_source"],
                         "kernel_share_of_step": (k_ms / args.steps) / prof_step_ms if prof_step_ms else None,
                         "timing": ("algorithmic bytes of the kernel's launches in one step / the step's CUDA-event "
                                    "time in the timed region (pipeline intact: a lower bound of the kernel's rate)"
                                    if serialised else
                                    "per-launch CUDA events on the library stream over K extra steps"),
                         "serialised": serialised,
                         "in_pipeline": ({"achieved": value, "frac": value / roof["peak"],
                                          "what": "whole step (all kernels, PDL look-ahead intact): "
                                                  "algorithmic bytes / ms_per_step"}
                                         if roof["bound"] == "hbm" else None),
                         "profiled_step_ms": prof_step_ms,
                         "launches_timed": k_n, **({"note": wl.roof_note} if hasattr(wl, "roof_note") else {})},
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        if extra:
            line["kernels"] = extra
        if others:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
