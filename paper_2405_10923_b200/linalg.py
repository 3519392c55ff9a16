"""Exceptions, scaling modes and the stability diagnostics (mirror of linalg.py).

Diagnostics run on the device: the Gram matrix A^t A by the library's
`sqb_gram` kernel, its eigenvalues by cuSOLVER (torch.linalg.eigvalsh on the
k x k Gram, device-side), the residual W - QR by the library's fused
`sqb_residual_norms` kernel.  cond(Q) through the Gram is accurate for the
well-conditioned Q this package produces (squaring a cond-5 matrix loses
nothing); an ill-conditioned input switches to a device QR + SVD of R, so
the value matches the reference's SVD (linalg.py:151-160) at any cond.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from .devarray import empty_colmajor, is_device, ld_of, to_device

SCALE_SQRT2 = "sqrt2"
SCALE_UNIT = "unit"
SCALINGS = (SCALE_SQRT2, SCALE_UNIT)


class BreakdownError(RuntimeError):
    """A factorization step cannot continue (linalg.py:18-19)."""


class SingularFactorError(np.linalg.LinAlgError):
    """Triangular solve hit a zero or subnormal diagonal entry (linalg.py:35-36)."""


def check_scaling(scaling):
    if scaling not in SCALINGS:
        raise ValueError(f"unknown scaling {scaling!r}, expected one of {SCALINGS}")


def scaling_code(scaling) -> int:
    check_scaling(scaling)
    return _lib.SQB_SCALE_SQRT2 if scaling == SCALE_SQRT2 else _lib.SQB_SCALE_UNIT


def sign(v):
    """linalg.py:200-202: sign(0) = +1."""
    return 1.0 if v >= 0.0 else -1.0


class DenseMatrix:
    """linalg.py:40-72: a host matrix tagged with the format its float64 entries
    honour (rounded on construction).  Every entry point of this package takes
    it wherever it takes an ndarray (it converts through __array__)."""

    def __init__(self, data, precision="double"):
        from .precision import round_to
        a = np.array(data, dtype=np.float64, ndmin=2)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-D array, got shape {a.shape}")
        self.precision = precision
        self.data = np.asfortranarray(round_to(a, precision))

    rows = property(lambda self: self.data.shape[0])
    cols = property(lambda self: self.data.shape[1])
    shape = property(lambda self: self.data.shape)

    def __array__(self, dtype=None, copy=None):
        return np.array(self.data, dtype=np.float64 if dtype is None else dtype, copy=bool(copy) or None)

    def __eq__(self, other):
        return (isinstance(other, DenseMatrix) and self.precision == other.precision
                and np.array_equal(self.data, other.data))

    def __repr__(self):
        return f"DenseMatrix(data={self.data!r}, precision={self.precision!r})"


def as_array(M):
    """linalg.py:75-79 (device tensors are left as they are)."""
    if isinstance(M, torch.Tensor):
        return M
    if isinstance(M, DenseMatrix):
        return M.data
    return np.asarray(M, dtype=np.float64)


def cast_precision(M, tag):
    """linalg.py:82-89: M rounded to `tag` as a DenseMatrix (idempotent)."""
    return DenseMatrix(as_array(M), tag)


def _dev64(A) -> torch.Tensor:
    return to_device(A, "double")


def gram(A) -> torch.Tensor:
    """A^t A (fp64, k x k) on the device."""
    Ad = _dev64(A)
    N, k = Ad.shape
    G = empty_colmajor(k, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_gram(ctx.h, Ad.data_ptr(), ld_of(Ad), N, k, G.data_ptr(), ld_of(G)), "sqb_gram")
    return G


# Gram eigenvalues resolve sigma_min to ~u * cond^2 relative; above this
# lambda_min / lambda_max ratio (cond < 1e4) that is <= 1e-8 and the fast
# path is kept, below it (or lambda_min <= 0) the QR + SVD path runs.
_GRAM_RATIO_MIN = 1e-8


def _hqr_r(Ad) -> torch.Tensor:
    """R factor of the library's Householder QR (baselines.py:33-89; one CTA
    for a small matrix, the tall multi-CTA path of csrc/hqr_tall.cu
    otherwise) — the reduction LAPACK's gesdd applies to a tall matrix before
    its SVD, without leaving the library for the n-dimensional work.  A column
    exactly dependent on its predecessors (HQR breakdown) makes M singular to
    working precision: sigma_min = 0."""
    from .devarray import empty_colmajor as _ec
    N, k = Ad.shape
    U = _ec(N, k, "double")
    T = _ec(k, k, "double")
    R = _ec(k, k, "double")
    scal = torch.empty(3 * k, dtype=torch.float64, device=Ad.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_householder_qr(ctx.h, 0, Ad.data_ptr(), ld_of(Ad), N, k, U.data_ptr(), ld_of(U),
                                            T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R), scal.data_ptr(),
                                            scal.data_ptr() + 8 * k, scal.data_ptr() + 16 * k), "sqb_householder_qr")
    code, col, _ = ctx.status()
    if code != 0:
        R = torch.triu(R)
        R[col - 1:, col - 1:] = 0.0  # the trailing block was never reduced
    return R


def cond_number(M, exact: bool = False):
    """linalg.py:151-160: 2-norm condition number; +inf if sigma_min == 0.

    The reference takes float64 SVD values.  Here a well-conditioned M (the
    factors' Q, cond ~ 1-10) is measured through its Gram matrix (library
    `sqb_gram` + a k x k eigvalsh), where squaring loses nothing; whenever the
    Gram ratio shows cond >~ 1e4 (lambda_min <= 0 included) the value is the
    float64 SVD of the R factor of a device Householder QR of M — the same
    numbers as the reference's SVD (LAPACK's gesdd also reduces a tall matrix
    by QR first), e.g. 1e15 on config 2's W where the Gram route underflows.
    `exact=True` skips the Gram probe."""
    Ad = _dev64(M)
    if Ad.numel() == 0:
        return np.inf
    if not bool(torch.isfinite(Ad).all()):
        return np.inf
    if not exact:
        ev = torch.linalg.eigvalsh(gram(Ad))
        lmin, lmax = float(ev[0]), float(ev[-1])
        if lmax > 0.0 and lmin > _GRAM_RATIO_MIN * lmax:
            return float(np.sqrt(lmax) / np.sqrt(lmin))
    N, k = Ad.shape
    B = _hqr_r(Ad) if N > k else Ad
    sv = torch.linalg.svdvals(B)
    smax, smin = float(sv[0]), float(sv[-1])
    if smin == 0.0:
        return np.inf
    return smax / smin


def orthogonality_error(Q):
    """linalg.py:193-197: ||Q^t Q - I||_F."""
    G = gram(Q)
    k = G.shape[0]
    return float(torch.linalg.norm(G - torch.eye(k, dtype=G.dtype, device=G.device)))


class FactorizationErrors(NamedTuple):
    fro_rel_err: float
    max_col_rel_err: float
    flagged_columns: tuple


def factorization_errors(W, Q, R):
    """linalg.py:169-190: relative residuals of W ~ Q R (Frobenius, per column)."""
    Wd, Qd, Rd = _dev64(W), _dev64(Q), _dev64(R)
    N, k = Qd.shape
    out = torch.empty(2 * Rd.shape[1], dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_residual_norms(ctx.h, Wd.data_ptr(), ld_of(Wd), Qd.data_ptr(), ld_of(Qd),
                                            Rd.data_ptr(), ld_of(Rd), N, k, Rd.shape[1], out.data_ptr()),
              "sqb_residual_norms")
    o = out.cpu().numpy()
    d2, w2 = o[: Rd.shape[1]], o[Rd.shape[1]:]
    wf = float(np.sqrt(w2.sum()))
    dn = float(np.sqrt(d2.sum()))
    fro = dn / wf if wf else dn
    colw = np.sqrt(w2)
    cold = np.sqrt(d2)
    zero = colw == 0.0
    rel = cold / np.where(zero, wf if wf else 1.0, colw)
    return FactorizationErrors(fro, float(rel.max()) if rel.size else 0.0,
                               tuple(np.nonzero(zero)[0].tolist()))


__all__ = ["SCALE_SQRT2", "SCALE_UNIT", "SCALINGS", "BreakdownError", "SingularFactorError",
           "check_scaling", "sign", "cond_number", "orthogonality_error", "factorization_errors",
           "FactorizationErrors", "gram", "is_device"]
