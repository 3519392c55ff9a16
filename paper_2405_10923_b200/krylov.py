"""RHQR-Arnoldi and GMRES (mirror of krylov.py) on the sm_100a library.

The whole Arnoldi run (krylov.py:82-150) is one library call
(`sqb_rhqr_arnoldi`): the per-step kernels are enqueued back to back and a
closed Krylov space is detected on the device, so the host synchronises once.
Operators (krylov.py:28-35): scipy sparse matrices and `CSRMatrix` run the
library's CSR SpMV; dense arrays the DMMA GEMV; a Python callable (a numpy
closure, a scipy LinearOperator, ...) is called through a C callback on the
library's stream.  As in the reference (krylov.py:28-35) it receives the
vector in the caller's form: a float64 numpy vector when the caller passed
host operands, a CUDA float64 tensor when it passed device tensors; it may
return either.  An exception raised by the callable propagates unchanged.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse
import torch

from . import _lib
from .devarray import CODES, empty_colmajor, is_device, ld_of, to_device, to_numpy, tag_of_torch
from .linalg import SCALE_SQRT2, check_scaling, scaling_code
from .precision import DOUBLE_POLICY, require_device_policy
from .rhqr import _embed, _out, apply_reflectors_compact, raise_status
from .sketching import EmbeddedSketch


class CSRMatrix:
    """A square fp64 CSR matrix resident on the device (int64 indptr, int32
    indices).  Built from scipy sparse or raw arrays."""

    def __init__(self, indptr, indices, data, n=None):
        ip = np.asarray(indptr, dtype=np.int64)
        self.n = int(n if n is not None else ip.shape[0] - 1)
        self.indptr = torch.from_numpy(ip).cuda()
        self.indices = torch.from_numpy(np.asarray(indices, dtype=np.int32)).cuda()
        self.data = torch.from_numpy(np.asarray(data, dtype=np.float64)).cuda()
        self.shape = (self.n, self.n)
        self.nnz = int(self.data.shape[0])

    @classmethod
    def from_scipy(cls, A):
        A = scipy.sparse.csr_matrix(A)
        A.sort_indices()
        return cls(A.indptr, A.indices, A.data, A.shape[0])

    def matvec(self, x):
        """y = A x for a CUDA vector (library SpMV)."""
        xd = to_device(x, "double")
        y = empty_colmajor(self.n, 1, "double")
        ctx = _lib.context()
        ctx.check(_lib.lib().sqb_csr_spmv(ctx.h, CODES["double"], self.n, self.indptr.data_ptr(),
                                          self.indices.data_ptr(), self.data.data_ptr(), xd.data_ptr(),
                                          None, y.data_ptr()), "sqb_csr_spmv")
        return y[:, 0]


class _Operator:
    """Device form of A for sqb_rhqr_arnoldi (keeps buffers alive)."""

    def __init__(self, A, n, tag, host=False):
        self.keep = []
        self.exc = None  # exception raised by a Python matvec, re-raised after the library call
        self.desc = _lib.OperatorDesc(n=n)
        if isinstance(A, CSRMatrix) or scipy.sparse.issparse(A):
            M = A if isinstance(A, CSRMatrix) else CSRMatrix.from_scipy(A)
            self.keep.append(M)
            self.desc.kind = _lib.SQB_OP_CSR
            self.desc.indptr, self.desc.indices, self.desc.data = (
                M.indptr.data_ptr(), M.indices.data_ptr(), M.data.data_ptr())
        elif callable(A) and not isinstance(A, (np.ndarray, torch.Tensor)):
            xbuf = empty_colmajor(n, 1, tag)
            ybuf = torch.empty(n, dtype=torch.float64, device="cuda")

            def _cb(user, stream):
                try:
                    x = xbuf[:, 0].to(torch.float64)
                    y = A(x.cpu().numpy() if host else x)
                    y = y if isinstance(y, torch.Tensor) else torch.from_numpy(
                        np.ascontiguousarray(np.asarray(y, dtype=np.float64)))
                    if y.numel() != n:
                        raise ValueError(f"matvec returned {y.numel()} values, expected {n}")
                    ybuf.copy_(y.reshape(-1).to(device=ybuf.device, dtype=torch.float64))
                    return 0
                except BaseException as e:  # kept and re-raised by the caller
                    self.exc = e
                    return 1

            cb = _lib.MATVEC_CB(_cb)
            self.keep += [xbuf, ybuf, cb]
            self.desc.kind = _lib.SQB_OP_CALLBACK
            self.desc.cb = cb
            self.desc.xbuf, self.desc.ybuf = xbuf.data_ptr(), ybuf.data_ptr()
        else:
            Ad = A if is_device(A) else torch.from_numpy(np.ascontiguousarray(np.asarray(A, dtype=np.float64)))
            Ad = Ad.to(device="cuda", dtype=torch.float64).contiguous()  # row-major
            self.keep.append(Ad)
            self.desc.kind = _lib.SQB_OP_DENSE
            self.desc.A, self.desc.lda = Ad.data_ptr(), Ad.stride(0)


@dataclass
class KrylovBundle:
    """krylov.py:38-61."""

    U: object
    S: object
    T: object
    H: object
    psi: EmbeddedSketch
    beta: float
    scaling: str
    Q_cols: object = None
    breakdown: int = None
    y: object = None
    resid_history: object = None

    @property
    def dim(self):
        return self.H.shape[1]


def _lo_tag(U):
    return tag_of_torch(U.dtype) if is_device(U) else "double"


def arnoldi_q(bundle, cols=None):
    """krylov.py:64-79: basis columns q_1..q_cols from the compact form."""
    host = not is_device(bundle.U)
    tag = _lo_tag(bundle.U)
    Ud = to_device(bundle.U, tag)
    N, r = Ud.shape
    c = r if cols is None else cols
    if not 0 <= c <= r:
        raise ValueError(f"have {r} reflectors, cannot build {c} columns")
    Sd, Td = to_device(bundle.S, "double"), to_device(bundle.T, "double")
    Q = empty_colmajor(N, c, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_arnoldi_q(ctx.h, CODES[tag], Ud.data_ptr(), ld_of(Ud), N, r, Td.data_ptr(),
                                       ld_of(Td), Sd.data_ptr(), ld_of(Sd), c, Q.data_ptr(), ld_of(Q)),
              "sqb_arnoldi_q")
    return _out(Q, host)


def rhqr_arnoldi(A, b, x0, m, omega, scaling=SCALE_SQRT2, policy=None, store_q=True, happy_tol=None,
                 _host=None):
    """krylov.py:82-150: Krylov basis of (A, b - A x0) through randomized
    Householder QR; omega sketches the trailing n-m-1 coordinates."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(b)                     # form of the returned bundle
    op_host = host if _host is None else _host  # form a Python matvec receives
    tag = policy.low
    bd = to_device(b, "double")[:, 0]
    n = bd.shape[0]
    x0 = np.zeros(n) if x0 is None else x0
    x0d = to_device(x0, tag)
    psi = _embed(omega, n, m + 1)
    if happy_tol is None:
        happy_tol = 32.0 * policy.u_high
    mt = m + 1
    od = psi.out_dim
    op = _Operator(A, n, tag, host=op_host)
    U = empty_colmajor(n, mt, tag)
    S = empty_colmajor(od, mt, "double")
    T = empty_colmajor(mt, mt, "double")
    H = empty_colmajor(mt, m, "double")
    Q = empty_colmajor(n, m, "double") if store_q else None
    beta = torch.zeros(1, dtype=torch.float64, device="cuda")
    attained = C.c_int(-1)
    ctx = _lib.context()
    _check_op(ctx, op, _lib.lib().sqb_rhqr_arnoldi(
        ctx.h, psi.omega.desc(), C.byref(op.desc), m, scaling_code(scaling), CODES[tag], float(happy_tol),
        bd.data_ptr(), x0d.data_ptr(), U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T),
        H.data_ptr(), ld_of(H), Q.data_ptr() if store_q else None, ld_of(Q) if store_q else 1,
        beta.data_ptr(), C.byref(attained)), "sqb_rhqr_arnoldi")
    raise_status(ctx, "rhqr_arnoldi")
    closed = None if attained.value < 0 else attained.value
    k = m if closed is None else closed
    r = mt if closed is None else closed
    return KrylovBundle(U=_out(U[:, :r], host), S=_out(S[:, :r], host), T=_out(T[:r, :r], host),
                        H=_out(H[: k + 1, :k], host), psi=psi, beta=float(beta.item()), scaling=scaling,
                        Q_cols=_out(Q[:, :k], host) if store_q else None, breakdown=closed)


def hessenberg_lstsq(H, beta, history=False):
    """krylov.py:153-190: min ||beta e1 - H y|| by Givens rotations (device)."""
    host = not is_device(H)
    Hd = to_device(H, "double")
    p, k = Hd.shape
    y = torch.zeros(max(k, 1), dtype=torch.float64, device="cuda")
    hist = torch.zeros(k + 1, dtype=torch.float64, device="cuda")
    resid = torch.zeros(1, dtype=torch.float64, device="cuda")
    work = torch.empty(p * max(k, 1) + p, dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_hessenberg_lstsq(ctx.h, Hd.data_ptr(), ld_of(Hd), p, k, float(beta), y.data_ptr(),
                                              hist.data_ptr(), resid.data_ptr(), work.data_ptr()),
              "sqb_hessenberg_lstsq")
    yk = y[:k]
    out = (_out(yk, host), float(resid.item()))
    return out + (_out(hist, host),) if history else out


def rhqr_gmres(A, b, x0, m, omega, scaling=SCALE_SQRT2, policy=None, happy_tol=None, _host=None):
    """krylov.py:193-222: GMRES in the sketched norm; returns (x, resid_history)."""
    policy = policy or DOUBLE_POLICY
    host = (not is_device(b)) if _host is None else _host
    bd = to_device(b, "double")[:, 0]
    n = bd.shape[0]
    x0d = torch.zeros(n, dtype=torch.float64, device="cuda") if x0 is None else to_device(x0, "double")[:, 0]
    bun = rhqr_arnoldi(A, bd, x0d, m, omega, scaling=scaling, policy=policy, store_q=False, happy_tol=happy_tol,
                       _host=host)
    k = bun.dim
    y, _, hist = hessenberg_lstsq(bun.H, bun.beta, history=True)
    if k and bool((torch.diagonal(bun.H)[:k] == 0.0).any()):
        warnings.warn("Hessenberg system is rank deficient; dependent coordinates were zeroed", RuntimeWarning)
    bun.y = y
    bun.resid_history = hist
    if k == 0:
        x = x0d.clone()
        return (to_numpy(x), to_numpy(hist)) if host else (x, hist)
    pad = torch.zeros(n, dtype=torch.float64, device="cuda")
    pad[:k] = y
    corr = apply_reflectors_compact(bun.U[:, :k], bun.S[:, :k], bun.T[:k, :k], pad, bun.psi, policy=policy)
    x = x0d + corr.to(torch.float64)
    return (to_numpy(x), to_numpy(hist)) if host else (x, hist)


def rhqr_gmres_restarted(A, b, x0, m, omega, tol=1e-8, max_cycles=1000, scaling=SCALE_SQRT2, policy=None):
    """Restarted GMRES(m) with a relative-residual stop ||b - A x|| <= tol ||b||.
    Not in the reference (SPEC.md:546, :552 have neither restart nor
    tolerance); each cycle is exactly `rhqr_gmres` reusing the same Omega."""
    host = not is_device(b)
    op = A if isinstance(A, CSRMatrix) or callable(A) else None
    Aop = CSRMatrix.from_scipy(A) if scipy.sparse.issparse(A) else (op if op is not None else A)
    bd = to_device(b, "double")[:, 0]
    x = torch.zeros_like(bd) if x0 is None else to_device(x0, "double")[:, 0].clone()
    bnorm = float(torch.linalg.norm(bd))
    hists = []
    for cyc in range(max_cycles):
        x, h = rhqr_gmres(Aop, bd, x, m, omega, scaling=scaling, policy=policy, _host=host)
        x = to_device(x, "double")[:, 0] if host else x
        h = to_device(h, "double")[:, 0] if host else h
        hists.append(h)
        r = bd - (Aop.matvec(x) if isinstance(Aop, CSRMatrix) else _dense_matvec(Aop, x, host))
        if float(torch.linalg.norm(r)) <= tol * bnorm:
            break
    return (to_numpy(x), [to_numpy(h) for h in hists]) if host else (x, hists)


def _check_op(ctx, op, rc, what):
    """A failed Python matvec surfaces as its own exception, not as a status code."""
    if op.exc is not None:
        exc, op.exc = op.exc, None
        raise exc
    ctx.check(rc, what)


def _dense_matvec(A, x, host=False):
    if callable(A) and not isinstance(A, (np.ndarray, torch.Tensor)):
        y = A(x.cpu().numpy() if host else x)
        return y if isinstance(y, torch.Tensor) else torch.from_numpy(np.asarray(y, dtype=np.float64)).cuda()
    Ad = A if is_device(A) else torch.from_numpy(np.asarray(A, dtype=np.float64)).cuda()
    return Ad @ x


__all__ = ["CSRMatrix", "KrylovBundle", "arnoldi_q", "rhqr_arnoldi", "hessenberg_lstsq", "rhqr_gmres",
           "rhqr_gmres_restarted"]
