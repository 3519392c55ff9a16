"""Stability sweeps on the device (mirror of experiments.py).

`run_factor_experiment` factors W once (left-looking methods) or once per
sampled width (rec-rhqr) with the sm_100a library and reports, per width j,
the reference's MetricRow (experiments.py:47-54): cond(Q), cond(Psi Q),
||W - QR||_F / ||W||_F, the largest column error and ||(Psi Q)^t Psi Q - I||_F,
all in double against the storage-rounded W (experiments.py:1-9).
`run_gmres_experiment` does the same for RHQR-GMRES (GmresRow, :57-63).

Everything n-dimensional stays on the device.  The prefix metrics of a
left-looking factorization are read off ONE set of full-width quantities
instead of re-materialising every prefix as the reference does
(experiments.py:189-209), which is exact algebra, not an approximation:
  * thin Q of the j-column prefix is the first j columns of the full thin Q
    (U is lower trapezoidal and T upper triangular, rhqr.py:171-178);
  * column i of W - QR involves only Q[:, :i+1] and R[:i+1, i], so per-column
    residual norms are computed once and the prefix errors are partial sums;
  * (Psi Q)^t (Psi Q) of a prefix is the leading block of the full Gram;
  * cond of a column prefix is cond of the leading block of the R factor of
    one QR of the full matrix (the orthogonal factor does not change singular
    values); the small SVDs run on the device.
The CSV writer is byte-compatible with experiments.py:318-339 (%.17g).

Methods outside the hot path (RGS/CGS/MGS, randomized Cholesky QR,
RGS-GMRES) raise NotImplementedError.
"""

from __future__ import annotations

import re
import time
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import scipy.sparse
import torch

from . import _lib
from .devarray import ld_of, to_device
from .krylov import CSRMatrix, arnoldi_q, hessenberg_lstsq, rhqr_arnoldi
from .linalg import _hqr_r, BreakdownError, gram
from .precision import PrecisionRangeError, policy_from_tag, require_device_policy
from .rhqr import (apply_reflectors_compact, householder_qr, rec_rhqr, rhqr_block, rhqr_left, rhqr_right,
                   thin_q)
from .sketching import make_sketch
from .trim import trim_rhqr_left, trim_rhqr_right, trim_thin_q
from .workloads import gen_cmatrix as _gen_cmatrix

FACTOR_ALGOS = ("rhqr-left", "rhqr-right", "rhqr-block", "rec-rhqr",
                "trim-left", "trim-right", "rgs", "blas2-rgs", "cgs", "mgs",
                "hqr", "rcholqr")
EMBEDDED_ALGOS = ("rhqr-left", "rhqr-right", "rhqr-block", "rec-rhqr")
RERUN_ALGOS = ("rec-rhqr", "rcholqr")
DEVICE_ALGOS = ("rhqr-left", "rhqr-right", "rhqr-block", "rec-rhqr", "trim-left", "trim-right", "hqr")


class MetricRow(NamedTuple):
    j: int
    cond_q: float
    cond_sq: float
    fro_rel_err: float
    max_col_rel_err: float
    orth_err: float
    status: str


class GmresRow(NamedTuple):
    j: int
    sketched_resid: float
    true_resid: float
    relation_err: float
    cond_basis: float
    status: str


@dataclass
class ExperimentConfig:
    """experiments.py:66-84 (same fields, defaults and validation)."""

    algo: str
    sketch: str = "srht"
    ell: int = 0            # 0 means the 4m default
    s: int = 8              # nonzeros per column for the sparse sign sketch
    seed: int = 0
    precision: str = "double"
    every: int = 25
    scaling: str = "sqrt2"
    block_size: int = 32
    deterministic: bool = False

    def __post_init__(self):
        if self.every < 1:
            raise ValueError("metric stride must be >= 1")
        if self.ell < 0:
            raise ValueError("sampling size must be >= 1 (0 picks the default)")


def gen_cmatrix(n, m):
    """experiments.py:86-98 (evaluated on the host in double, like the reference)."""
    return _gen_cmatrix(n, m)


def sample_widths(m, every):
    """experiments.py:101-105."""
    js = list(range(every, m + 1, every))
    if not js or js[-1] != m:
        js.append(m)
    return js


def _nan_row(j, status):
    return MetricRow(j, np.nan, np.nan, np.nan, np.nan, np.nan, status)


def _breakdown_column(exc, fallback):
    """experiments.py:178-180."""
    hit = re.search(r"column (\d+)", str(exc))
    return int(hit.group(1)) if hit else fallback


# ---------------------------------------------------------------- device metrics
def _dev64(A) -> torch.Tensor:
    return to_device(A, "double")


def _round_device(Wd, tag):
    """round_to(W, tag) (precision.py:34-51) on the device, as float64."""
    if tag == "double":
        return Wd
    Wl = to_device(Wd, tag).to(torch.float64)
    bad = torch.isfinite(Wd) & ~torch.isfinite(Wl)
    if bool(bad.any()):
        raise PrecisionRangeError(f"value {float(Wd.abs()[bad].max()):g} overflows {tag} range")
    return Wl


def _prefix_conds(A):
    """cond(A[:, :j]) for every j (index j-1), from the R factor of one QR."""
    k = A.shape[1]
    if not bool(torch.isfinite(A).all()):
        return [np.inf] * k
    # the R factor of the library's Householder QR (one CTA for a small A, the
    # tall path of csrc/hqr_tall.cu otherwise): the n-dimensional work stays in
    # the library; only the k x k SVDs of its leading blocks go to torch
    R = _hqr_r(A) if A.shape[0] > k else torch.linalg.qr(A, mode="r").R
    out = []
    for j in range(1, k + 1):
        sv = torch.linalg.svdvals(R[:j, :j])
        smin = float(sv[-1])
        out.append(np.inf if smin == 0.0 else float(sv[0]) / smin)
    return out


def _prefix_metrics(Wl, Q, R, SQ):
    """Per-width metrics of a left-looking factorization (see module doc);
    returns a function j -> MetricRow."""
    k = Q.shape[1]
    Wd, Qd, Rd = _dev64(Wl[:, :k]), _dev64(Q), _dev64(R)
    out = torch.empty(2 * k, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_residual_norms(ctx.h, Wd.data_ptr(), ld_of(Wd), Qd.data_ptr(), ld_of(Qd),
                                            Rd.data_ptr(), ld_of(Rd), Qd.shape[0], k, k, out.data_ptr()),
              "sqb_residual_norms")
    o = out.cpu().numpy()
    d2, w2 = o[:k], o[k:]
    G = gram(SQ).cpu().numpy()
    cq, csq = _prefix_conds(_dev64(Q)), _prefix_conds(_dev64(SQ))

    def row(j, status="ok"):
        wf = float(np.sqrt(w2[:j].sum()))
        dn = float(np.sqrt(d2[:j].sum()))
        colw, cold = np.sqrt(w2[:j]), np.sqrt(d2[:j])
        rel = cold / np.where(colw == 0.0, wf if wf else 1.0, colw)
        orth = float(np.linalg.norm(G[:j, :j] - np.eye(j)))
        return MetricRow(j=j, cond_q=cq[j - 1], cond_sq=csq[j - 1], fro_rel_err=dn / wf if wf else dn,
                         max_col_rel_err=float(rel.max()) if rel.size else 0.0, orth_err=orth, status=status)

    return row


# ---------------------------------------------------------------- factor sweeps
def _factor_once(Wd, config, policy, ell):
    n, m = Wd.shape
    algo = config.algo
    omega = make_sketch(config.sketch, ell, n - m, config.seed, s=config.s) if algo in EMBEDDED_ALGOS else None
    if algo in ("trim-left", "trim-right"):  # the trimmed drivers sketch all n coordinates
        omega = make_sketch(config.sketch, ell, n, config.seed, s=config.s)
        fn = trim_rhqr_left if algo == "trim-left" else trim_rhqr_right
        return fn(Wd, omega, scaling=config.scaling, policy=policy)
    if algo == "rhqr-left":
        return rhqr_left(Wd, omega, scaling=config.scaling, policy=policy)
    if algo == "rhqr-right":
        return rhqr_right(Wd, omega, scaling=config.scaling, policy=policy)
    if algo == "rhqr-block":
        return rhqr_block(Wd, omega, block_size=config.block_size, scaling=config.scaling, policy=policy)
    if algo == "rec-rhqr":
        return rec_rhqr(Wd, omega, scaling=config.scaling, policy=policy)
    return householder_qr(Wd, scaling=config.scaling, policy=policy)


def _qr_of(out, algo):
    """(Q, R, Psi Q) of a full-width factorization object (experiments.py:189-209)."""
    if algo == "hqr":
        return out.Q, out.R, out.Q
    if algo.startswith("trim"):  # experiments.py:196-199
        Q = trim_thin_q(out)
        return Q, out.R, out.omega.apply(Q)
    Q = thin_q(out)
    return Q, out.R, out.psi.apply(Q)


def run_factor_experiment(W, config):
    """experiments.py:125-142: metric rows for config.algo on the leading j
    columns of W, j = every, 2 every, ..., m.  A breakdown at column c gives
    rows with status 'breakdown@c' and NaN metrics from the first affected
    width on."""
    if config.algo not in FACTOR_ALGOS:
        raise ValueError(f"unknown algorithm {config.algo!r}")
    if config.algo not in DEVICE_ALGOS:
        raise NotImplementedError(
            f"{config.algo!r} is a comparison method outside the B200 hot path (SURVEY §2); "
            f"device algorithms: {DEVICE_ALGOS}")
    policy = policy_from_tag(config.precision)
    require_device_policy(policy)
    Wd = _dev64(W)
    n, m = Wd.shape
    ell = config.ell or 4 * m
    Wl = _round_device(Wd, policy.low)
    js = sample_widths(m, config.every)
    if config.algo in RERUN_ALGOS:
        return _rerun_sweep(Wd, Wl, config, policy, ell, js)
    return _prefix_sweep(Wd, Wl, config, policy, ell, js)


def _prefix_sweep(Wd, Wl, config, policy, ell, js):
    """experiments.py:212-235."""
    attained = Wd.shape[1]
    status = "ok"
    out = None
    while attained > 0:
        try:
            out = _factor_once(Wd[:, :attained], config, policy, ell)
            break
        except (BreakdownError, PrecisionRangeError) as exc:
            col = _breakdown_column(exc, attained)
            if status == "ok":
                status = f"breakdown@{col}"
            attained = min(col - 1, attained - 1)
    if config.algo == "rhqr-block" and out is not None:
        out = out.stacked()
    rows = []
    row = None
    if out is not None and attained > 0:
        Q, R, SQ = _qr_of(out, config.algo)
        row = _prefix_metrics(Wl, Q, R, SQ)
    for j in js:
        if j > attained:
            rows.append(_nan_row(j, status))
            continue
        rows.append(row(j))
    return rows


def _rerun_sweep(Wd, Wl, config, policy, ell, js):
    """experiments.py:238-252 (rec-rhqr depends on the whole input: refactor per width)."""
    rows = []
    for j in js:
        try:
            out = _factor_once(Wd[:, :j], config, policy, ell)
        except (BreakdownError, PrecisionRangeError) as exc:
            rows.append(_nan_row(j, f"breakdown@{_breakdown_column(exc, j)}"))
            continue
        Q, R, SQ = _qr_of(out, config.algo)
        rows.append(_prefix_metrics(Wl, Q, R, SQ)(j))
    return rows


# ---------------------------------------------------------------- GMRES sweep
class _MatVec:
    """A x for the metric pass: CSR through the library SpMV, dense through a
    device GEMV, callables as given."""

    def __init__(self, A, n):
        self.A = A
        if scipy.sparse.issparse(A):
            self.csr = CSRMatrix.from_scipy(A)
        elif isinstance(A, CSRMatrix):
            self.csr = A
        else:
            self.csr = None
            if not callable(A) or isinstance(A, (np.ndarray, torch.Tensor)):
                self.dense = _dev64(A)

    def __call__(self, x):
        if self.csr is not None:
            return self.csr.matvec(x)
        if hasattr(self, "dense"):
            return self.dense @ x
        y = self.A(x)
        return y if isinstance(y, torch.Tensor) else torch.from_numpy(np.asarray(y, dtype=np.float64)).cuda()


def _operator_fro_norm(A, n):
    """experiments.py:302-315."""
    if scipy.sparse.issparse(A):
        return float(np.sqrt(A.multiply(A).sum()))
    if isinstance(A, CSRMatrix):
        return float(torch.linalg.norm(A.data))
    if callable(A) and not isinstance(A, (np.ndarray, torch.Tensor)):
        mv = _MatVec(A, n)
        total = 0.0
        e = torch.zeros(n, dtype=torch.float64, device="cuda")
        for i in range(n):
            e[i] = 1.0
            col = mv(e)
            total += float(col @ col)
            e[i] = 0.0
        return float(np.sqrt(total))
    return float(torch.linalg.norm(_dev64(A)))


def run_gmres_experiment(A, b, m, config, x0=None):
    """experiments.py:247-299 for algo 'rhqr': per iteration j the sketched
    and true residuals, the scaled Arnoldi relation error
    ||A Q_j - Q_{j+1} H_j||_F / (||A||_F ||Q_j||_F) and cond(Q_{j+1})."""
    if config.algo == "rgs":
        raise NotImplementedError("RGS-GMRES is a comparison method outside the B200 hot path (SURVEY §2 #11)")
    if config.algo != "rhqr":
        raise ValueError(f"unknown solver {config.algo!r}")
    policy = policy_from_tag(config.precision)
    require_device_policy(policy)
    bd = _dev64(b)[:, 0]
    n = bd.shape[0]
    x0d = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None else _dev64(x0)[:, 0]
    ell = config.ell or 4 * (m + 1)
    anorm = _operator_fro_norm(A, n)
    omega = make_sketch(config.sketch, ell, n - m - 1, config.seed, s=config.s)
    Aop = CSRMatrix.from_scipy(A) if scipy.sparse.issparse(A) else A
    bundle = rhqr_arnoldi(Aop, bd, x0d, m, omega, scaling=config.scaling, policy=policy)
    k = bundle.dim
    H, beta = bundle.H, bundle.beta
    Qext = arnoldi_q(bundle, min(k + 1, bundle.U.shape[1]))
    qc = Qext.shape[1]
    mv = _MatVec(Aop, n)
    # per-column pieces of the relation error: column i of A Q - Q H involves
    # Q[:, :i+2] only (H is Hessenberg)
    r2 = np.zeros(k)
    for i in range(min(k, qc)):
        nc = min(i + 2, qc)
        r = mv(Qext[:, i]) - Qext[:, :nc] @ H[:nc, i]
        r2[i] = float(r @ r)
    qn2 = (Qext * Qext).sum(dim=0).cpu().numpy()
    conds = _prefix_conds(Qext) if qc else []
    status = "ok" if k == m else f"closed@{k}"
    rows = []
    for j in range(1, k + 1):
        y, resid = hessenberg_lstsq(H[: j + 1, :j], beta)
        pad = torch.zeros(n, dtype=torch.float64, device="cuda")
        pad[:j] = y
        x = x0d + apply_reflectors_compact(bundle.U[:, :j], bundle.S[:, :j], bundle.T[:j, :j], pad,
                                           bundle.psi, policy=policy).to(torch.float64)
        ncols = min(j + 1, qc)
        rel = float(np.sqrt(r2[:j].sum())) / (anorm * max(float(np.sqrt(qn2[:j].sum())), 1e-300))
        rows.append(GmresRow(j=j, sketched_resid=float(resid),
                             true_resid=float(torch.linalg.norm(bd - mv(x))),
                             relation_err=rel, cond_basis=conds[ncols - 1], status=status))
    return rows


# ---------------------------------------------------------------- CSV
def write_csv(path, rows, config=None, extra=None):
    """experiments.py:318-339: rows to CSV with 17 significant digits; a
    commented header echoes the config and, unless deterministic, a timestamp."""
    fields = rows[0]._fields if rows else MetricRow._fields
    with open(path, "w") as fh:
        if config is not None:
            fh.write(f"# {config}\n")
            if not config.deterministic:
                fh.write(f"# written {time.strftime('%Y-%m-%dT%H:%M:%S')}\n")
        if extra:
            fh.write(f"# {extra}\n")
        fh.write(",".join(fields) + "\n")
        for row in rows:
            cells = []
            for v in row:
                if isinstance(v, str):
                    cells.append(v)
                elif isinstance(v, (int, np.integer)):
                    cells.append(str(int(v)))
                else:
                    cells.append(f"{v:.17g}")
            fh.write(",".join(cells) + "\n")


__all__ = ["FACTOR_ALGOS", "EMBEDDED_ALGOS", "RERUN_ALGOS", "DEVICE_ALGOS", "MetricRow", "GmresRow",
           "ExperimentConfig", "gen_cmatrix", "sample_widths", "run_factor_experiment",
           "run_gmres_experiment", "write_csv"]
