"""Randomized Householder QR (mirror of rhqr.py) on the sm_100a library.

Every numerical step runs on the device (see csrc/rhqr_left.cu,
csrc/compact.cu); this module only validates arguments exactly as the
reference does, moves operands across the boundary and maps device status
words to the reference's exceptions.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from .devarray import (CODES, empty_colmajor, host_f64, is_device, ld_of, pinned_f64, to_device, to_numpy,
                       tag_of_torch)
from .linalg import (SCALE_SQRT2, SCALE_UNIT, BreakdownError, SingularFactorError, check_scaling,
                     scaling_code)
from .precision import DOUBLE_POLICY, PrecisionRangeError, require_device_policy
from .sketching import EmbeddedSketch


@dataclass
class HouseholderStep:
    """rhqr.py:38-48."""

    j: int
    u: object
    s: object
    sigma: float
    rho: float
    beta: float


@dataclass
class RHQRFactors:
    """rhqr.py:143-168: W = Q R with Q = [I;0] - U T U1^t."""

    U: object
    S: object
    T: object
    R: object
    psi: EmbeddedSketch
    scaling: str
    sigmas: object
    rhos: object
    betas: object

    @property
    def cols(self):
        return self.U.shape[1]

    def prefix(self, j):
        return RHQRFactors(U=self.U[:, :j], S=self.S[:, :j], T=self.T[:j, :j], R=self.R[:j, :j],
                           psi=self.psi, scaling=self.scaling, sigmas=self.sigmas[:j],
                           rhos=self.rhos[:j], betas=self.betas[:j])


def _embed(omega, n, m):
    """rhqr.py:202-216 (same checks and messages)."""
    if isinstance(omega, EmbeddedSketch):
        if omega.n != n or omega.m != m:
            raise ValueError(
                f"embedding is {omega.out_dim}x{omega.n} with identity block "
                f"{omega.m}, expected input {n} and block {m}")
        if omega.omega.ell < m:
            raise ValueError("sampling size below column count")
        return omega
    if omega.n != n - m:
        raise ValueError(f"sketch takes {omega.n} coordinates, expected n-m={n - m}")
    if omega.ell < m:
        raise ValueError("sampling size below column count")
    return EmbeddedSketch(m, omega)


def raise_status(ctx, what="factorization", tag=None):
    """Map the device status word to the reference's exceptions."""
    code, col, val = ctx.status()
    if code == _lib.SQB_OK:
        return
    if code == _lib.SQB_ERR_RANGE:  # round_to on the device (precision.py:45-50)
        raise PrecisionRangeError(f"value {val:g} overflows {tag} range")
    if code == _lib.SQB_ERR_BREAKDOWN:
        if what == "rec_rhqr":
            if val == -1.0:  # rhqr.py:388-391
                raise BreakdownError(f"reconstruction factor has zero diagonal at column {col}")
            raise BreakdownError(f"column {col} exactly dependent on its predecessors")  # baselines.py:62
        if val == 0.0:
            raise BreakdownError(f"sketched tail annihilated at column {col}")
        raise BreakdownError(f"reflector scale degenerated at column {col} (rho={val:.3e})")
    if code == _lib.SQB_ERR_SINGULAR:
        raise SingularFactorError(f"triangular factor has zero or subnormal diagonal at index {col - 1}")
    if code == _lib.SQB_ERR_NONFINITE:  # scipy's check_finite in the reference's triangular solves
        raise ValueError("array must not contain infs or NaNs")
    if code == _lib.SQB_ERR_NCCL and col < 0:  # p2p_wait (csrc/p2p.cuh): a peer's flag never arrived
        raise _lib.SketchQRError(f"{what}: peer-memory exchange {int(val)} timed out waiting for rank {-col - 1}")
    raise _lib.SketchQRError(f"{what}: device status {code} at column {col}")


def _out(t, host):
    return to_numpy(t) if host else t


def _shape2(A):
    return tuple(A.shape) if is_device(A) else np.shape(np.asarray(A))


def rhqr_left_device(Wd, psi, scaling, policy, check=True):
    """Device-resident core: Wd is a column-major CUDA tensor in the low dtype
    with row m 16-byte aligned.  Returns device factors."""
    N, m = Wd.shape
    tag = policy.low
    od = psi.out_dim
    U = empty_colmajor(N, m, tag, align_row=m)
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_rhqr_left(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[tag], Wd.data_ptr(), N, m, ld_of(Wd),
        U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
        scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m), "sqb_rhqr_left")
    if check:
        raise_status(ctx, "rhqr_left")
    return U, S, T, R, scal[:m], scal[m:2 * m], scal[2 * m:]


def rhqr_left(W, omega, scaling=SCALE_SQRT2, policy=None):
    """rhqr.py:254-267: left-looking randomized Householder QR of a tall W."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    n, m = _shape2(W)
    psi = _embed(omega, n, m)
    if host:
        return _rhqr_left_host(W, psi, scaling, policy)
    Wd = to_device(W, policy.low, align_row=m)  # round_to(W, low) (rhqr.py:264)
    U, S, T, R, sg, rh, bt = rhqr_left_device(Wd, psi, scaling, policy)
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host), psi=psi,
                       scaling=scaling, sigmas=_out(sg, host), rhos=_out(rh, host),
                       betas=_out(bt, host))


def _rhqr_left_host(W, psi, scaling, policy):
    """Host operands (numpy / CPU tensor): one sqb_rhqr_left_host call, which
    uploads W, rounds it to the storage format on the device and overlaps
    both PCIe directions with the sweep (csrc/host_pipe.cu).  The float64
    factors come back as column-major (Fortran-order) ndarrays; U lives in
    page-locked memory so its column groups stream back during the sweep."""
    Wa, layout, ldw = host_f64(W)
    n, m = Wa.shape
    od = psi.out_dim
    U = pinned_f64(n, m)
    S = np.empty((m, od)).T
    T = np.empty((m, m)).T
    R = np.empty((m, m)).T
    scal = np.empty(3 * m)
    ctx = _lib.context()
    p = lambda a: a.ctypes.data  # noqa: E731
    ctx.check(_lib.lib().sqb_rhqr_left_host(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[policy.low], p(Wa), n, m, ldw, layout,
        p(U), n, p(S), od, p(T), m, p(R), m, p(scal), p(scal[m:]), p(scal[2 * m:])), "sqb_rhqr_left_host")
    raise_status(ctx, "rhqr_left", policy.low)
    return RHQRFactors(U=U, S=S, T=T, R=R, psi=psi, scaling=scaling, sigmas=scal[:m], rhos=scal[m:2 * m],
                       betas=scal[2 * m:])


def rhqr_right(W, omega, scaling=SCALE_SQRT2, policy=None):
    """rhqr.py:270-301: right-looking variant — rank-1 update of the trailing
    block, which is re-sketched wholesale at every step; T recovered from S."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    n, m = _shape2(W)
    psi = _embed(omega, n, m)
    tag = policy.low
    Wd = to_device(W, tag, align_row=m)
    od = psi.out_dim
    U = empty_colmajor(n, m, tag, align_row=m)
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_rhqr_right(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[tag], Wd.data_ptr(), n, m, ld_of(Wd),
        U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
        scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m), "sqb_rhqr_right")
    raise_status(ctx, "rhqr_right")
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host), psi=psi,
                       scaling=scaling, sigmas=_out(scal[:m], host), rhos=_out(scal[m:2 * m], host),
                       betas=_out(scal[2 * m:], host))


def rec_rhqr(W, omega, scaling=SCALE_SQRT2, policy=None):
    """rhqr.py:368-395: one sketch of W, Householder QR of the sketch in the
    high precision, triangular reconstruction of the n-dimensional reflectors."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    n, m = _shape2(W)
    psi = _embed(omega, n, m)
    if host:
        return _rec_rhqr_host(W, psi, scaling, policy)
    tag = policy.low
    Wd = to_device(W, tag, align_row=m)
    od = psi.out_dim
    U = empty_colmajor(n, m, tag, align_row=m)
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_rec_rhqr(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[tag], Wd.data_ptr(), n, m, ld_of(Wd),
        U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
        scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m), "sqb_rec_rhqr")
    raise_status(ctx, "rec_rhqr")
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host), psi=psi,
                       scaling=scaling, sigmas=_out(scal[:m], host), rhos=_out(scal[m:2 * m], host),
                       betas=_out(scal[2 * m:], host))


def _rec_rhqr_host(W, psi, scaling, policy):
    """Host operands: one sqb_rec_rhqr_host call — the Gaussian sketch GEMM
    runs under the blocked upload of W (csrc/host_pipe.cu); float64 factors
    come back as column-major ndarrays, U in page-locked memory."""
    Wa, layout, ldw = host_f64(W)
    n, m = Wa.shape
    od = psi.out_dim
    U = pinned_f64(n, m)
    S = np.empty((m, od)).T
    T = np.empty((m, m)).T
    R = np.empty((m, m)).T
    scal = np.empty(3 * m)
    ctx = _lib.context()
    p = lambda a: a.ctypes.data  # noqa: E731
    ctx.check(_lib.lib().sqb_rec_rhqr_host(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[policy.low], p(Wa), n, m, ldw, layout,
        p(U), n, p(S), od, p(T), m, p(R), m, p(scal), p(scal[m:]), p(scal[2 * m:])), "sqb_rec_rhqr_host")
    raise_status(ctx, "rec_rhqr", policy.low)
    return RHQRFactors(U=U, S=S, T=T, R=R, psi=psi, scaling=scaling, sigmas=scal[:m], rhos=scal[m:2 * m],
                       betas=scal[2 * m:])


def rh_vector(w, y, j, scaling=SCALE_SQRT2, policy=None):
    """rhqr.py:51-97: reflector eliminating entries j+1.. of y = Psi w."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(w)
    yd = to_device(y, "double")
    od = yd.shape[0]
    if not 0 <= j - 1 < od:
        raise ValueError(f"elimination index {j} outside sketch of length {od}")
    wd = to_device(w, policy.low)
    n = wd.shape[0]
    u = empty_colmajor(n, 1, policy.low)
    s = empty_colmajor(od, 1, "double")
    scal = torch.empty(5, dtype=torch.float64, device=wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_rh_vector(ctx.h, scaling_code(scaling), CODES[policy.low], wd.data_ptr(), n,
                                       yd.data_ptr(), od, j, u.data_ptr(), s.data_ptr(), scal.data_ptr()),
              "sqb_rh_vector")
    raise_status(ctx, "rh_vector")
    sc = scal.cpu().numpy()
    return HouseholderStep(j=j, u=_out(u[:, 0], host), s=_out(s[:, 0], host), sigma=float(sc[0]),
                           rho=float(sc[1]), beta=float(sc[2]))


def apply_reflectors_compact(U, S, T, X, psi, transpose_t=False, policy=None):
    """rhqr.py:100-119: (I - U T S^t Psi) X, or the reversed product."""
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(X)
    tag = policy.low
    Xs = _shape2(X)
    vec = len(Xs) == 1
    N = Xs[0]
    m = psi.m
    Ud = to_device(U if not vec or np.ndim(U) == 2 else U, tag)
    if Ud.dim() == 1:
        Ud = Ud[:, None]
    r = Ud.shape[1] if np.prod(_shape2(U)) else 0
    Sd = to_device(S, "double") if r else empty_colmajor(psi.out_dim, 1, "double")
    Td = to_device(T, "double") if r else empty_colmajor(1, 1, "double")
    Xd = to_device(X, tag, align_row=m)
    k = Xd.shape[1]
    Out = empty_colmajor(N, k, tag, align_row=m)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_apply_reflectors(
        ctx.h, psi.omega.desc(), m, CODES[tag], Ud.data_ptr(), ld_of(Ud), N, r, Sd.data_ptr(), ld_of(Sd),
        Td.data_ptr(), ld_of(Td), 1 if transpose_t else 0, Xd.data_ptr(), ld_of(Xd), k,
        Out.data_ptr(), ld_of(Out)), "sqb_apply_reflectors")
    res = Out[:, 0] if vec else Out
    if host:
        return to_numpy(res)
    return res


class QRResult(NamedTuple):
    """baselines.py:25-29."""

    Q: object
    R: object
    method: str
    aux: dict


def householder_qr(A, scaling=SCALE_SQRT2, policy=None):
    """baselines.py:33-89: left-looking Householder QR with compact T of a small
    (p x m) matrix, one CTA on the device (the sketch-space QR of recRHQR)."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    if policy.low != "double" or policy.high != "double":
        raise NotImplementedError("householder_qr in a low-precision policy is a comparison method outside the B200 "
                                  "hot path (the device Householder QR is the float64 sketch-space QR of recRHQR)")
    host = not is_device(A)
    Ad = to_device(A, "double")
    p, m = Ad.shape
    if p < m:
        raise ValueError(f"need p >= m, got {p} x {m}")
    U = empty_colmajor(p, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_householder_qr(ctx.h, scaling_code(scaling), Ad.data_ptr(), ld_of(Ad), p, m,
                                            U.data_ptr(), ld_of(U), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
                                            scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m),
              "sqb_householder_qr")
    raise_status(ctx, "rec_rhqr")
    Q = thin_q(RHQRFactors(U=U, S=U, T=T, R=R, psi=None, scaling=scaling, sigmas=None, rhos=None, betas=None))
    aux = {"U": _out(U, host), "T": _out(T, host), "sigmas": _out(scal[:m], host),
           "rhos": _out(scal[m:2 * m], host), "betas": _out(scal[2 * m:], host)}
    return QRResult(Q=_out(Q, host), R=_out(R, host), method="householder", aux=aux)


def _round_high(X, policy, host):
    """The reference solves in policy.high (linalg.py:108-116): the float64
    device solution rounded once to that format (exactly representable, as the
    reference's output is; a no-op for the double policy)."""
    if policy is None or policy.high == "double":
        return X
    from .precision import round_to
    if host:
        return round_to(X, policy.high)
    from .devarray import TORCH_DTYPES
    return X.to(TORCH_DTYPES[policy.high]).to(torch.float64)


def upper_tri_solve(R, B, policy=None):
    """linalg.py:102-116: R X = B by back substitution (device)."""
    host = not (is_device(R) or is_device(B))
    Rd = to_device(R, "double")
    vec = (B.dim() == 1) if is_device(B) else (np.ndim(B) == 1)
    Bd = to_device(B, "double")
    m, k = Bd.shape
    X = empty_colmajor(m, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_upper_tri_solve(ctx.h, Rd.data_ptr(), ld_of(Rd), m, Bd.data_ptr(), ld_of(Bd), k,
                                             X.data_ptr(), ld_of(X)), "sqb_upper_tri_solve")
    raise_status(ctx, "upper_tri_solve")
    out = X[:, 0] if vec else X
    return _round_high(_out(out, host), policy, host)


def right_tri_solve(B, R, policy=None):
    """linalg.py:119-129: X R = B for upper-triangular R.  R^t X^t = B^t is a
    lower-triangular system; reversing the index order turns it into the
    upper-triangular one the device solves (J R^t J is upper, J the flip)."""
    host = not (is_device(R) or is_device(B))
    vec = (B.dim() == 1) if is_device(B) else (np.ndim(B) == 1)
    Rd = to_device(R, "double")
    Bd = to_device(B, "double")              # a vector arrives as the column B^t
    Bt = Bd if vec else Bd.t()
    Rf = torch.flip(Rd, (0, 1)).t()
    Xf = upper_tri_solve(Rf, torch.flip(Bt, (0,)).contiguous())
    Xt = torch.flip(Xf, (0,))
    out = Xt[:, 0] if vec else Xt.t()
    return _round_high(_out(out, host), policy, host)


def lsq_via_implicit_q(factors, b, policy=None):
    """rhqr.py:191-199: argmin_x ||Psi(W x - b)|| through the compact form."""
    policy = policy or DOUBLE_POLICY
    c = apply_reflectors_compact(factors.U, factors.S, factors.T, b, factors.psi, transpose_t=True, policy=policy)
    m = factors.R.shape[1]
    return upper_tri_solve(factors.R, c[:m], policy=policy)


def t_factor_from_sketches(S, policy=None):
    """rhqr.py:122-132: T of the compact form from S = Psi U alone
    (S^t S = T^{-1} + T^{-t}); Gram + back substitution on the device."""
    policy = policy or DOUBLE_POLICY
    host = not is_device(S)
    Sd = to_device(S, "double")
    if Sd.dim() == 1:
        Sd = Sd[:, None]
    od, k = Sd.shape
    T = empty_colmajor(k, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_t_factor(ctx.h, Sd.data_ptr(), ld_of(Sd), od, k, T.data_ptr(), ld_of(T)),
              "sqb_t_factor")
    raise_status(ctx, "upper_tri_solve")
    return _out(T, host)


@dataclass
class BlockPanel:
    """rhqr.py:304-309: one panel of the blocked sweep."""

    U: object
    S: object
    T: object
    offset: int


@dataclass
class BlockRHQRFactors:
    """rhqr.py:312-331: panel-compact output of rhqr_block; stacked() merges
    the panels into one compact form (the global T rebuilt from S)."""

    panels: list
    R: object
    psi: EmbeddedSketch
    scaling: str
    sigmas: object
    rhos: object
    betas: object

    def stacked(self):
        dev = is_device(self.panels[0].U)
        cat = (lambda xs: torch.cat(xs, dim=1)) if dev else (lambda xs: np.concatenate(xs, axis=1))
        U = cat([p.U for p in self.panels])
        S = cat([p.S for p in self.panels])
        return RHQRFactors(U=U, S=S, T=t_factor_from_sketches(S), R=self.R, psi=self.psi,
                           scaling=self.scaling, sigmas=self.sigmas, rhos=self.rhos, betas=self.betas)


def rhqr_block_device(Wd, psi, block_size, scaling, policy, check=True):
    """Device core of rhqr_block: returns U, S, the block-diagonal panel T's,
    R and the scalars as device tensors."""
    N, m = Wd.shape
    tag = policy.low
    od = psi.out_dim
    U = empty_colmajor(N, m, tag, align_row=m)
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_rhqr_block(
        ctx.h, psi.omega.desc(), scaling_code(scaling), CODES[tag], Wd.data_ptr(), N, m, ld_of(Wd), block_size,
        U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
        scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m), "sqb_rhqr_block")
    if check:
        raise_status(ctx, "rhqr_block")
    return U, S, T, R, scal[:m], scal[m:2 * m], scal[2 * m:]


def rhqr_block(W, omega, block_size=32, scaling=SCALE_SQRT2, policy=None):
    """rhqr.py:334-365: blocked left-looking sweep.  Earlier panels are applied
    compactly (one re-sketch per panel), then the panel is factored in place;
    a final panel narrower than block_size is processed as-is."""
    check_scaling(scaling)
    if block_size < 1:
        raise ValueError("block_size must be positive")
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    n, m = _shape2(W)
    psi = _embed(omega, n, m)
    Wd = to_device(W, policy.low, align_row=m)
    U, S, T, R, sg, rh, bt = rhqr_block_device(Wd, psi, int(block_size), scaling, policy)
    panels = []
    for j0 in range(0, m, block_size):
        j1 = min(j0 + block_size, m)
        panels.append(BlockPanel(U=_out(U[:, j0:j1], host), S=_out(S[:, j0:j1], host),
                                 T=_out(T[j0:j1, j0:j1], host), offset=j0))
    return BlockRHQRFactors(panels=panels, R=_out(R, host), psi=psi, scaling=scaling, sigmas=_out(sg, host),
                            rhos=_out(rh, host), betas=_out(bt, host))


def _lo_tag(U):
    return tag_of_torch(U.dtype) if is_device(U) else "double"


def thin_q(factors):
    """rhqr.py:171-178: Q = [I;0] - U T U1^t in float64."""
    host = not is_device(factors.U)
    tag = _lo_tag(factors.U)
    Ud = to_device(factors.U, tag)
    Td = to_device(factors.T, "double")
    N, k = Ud.shape
    Q = empty_colmajor(N, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_thin_q(ctx.h, CODES[tag], Ud.data_ptr(), ld_of(Ud), N, k, Td.data_ptr(),
                                    ld_of(Td), Q.data_ptr(), ld_of(Q)), "sqb_thin_q")
    return _out(Q, host)


def sketch_q(factors):
    """rhqr.py:181-188: Psi Q = [I;0] - S T U1^t without n-dimensional data."""
    host = not is_device(factors.U)
    tag = _lo_tag(factors.U)
    k = factors.U.shape[1]
    Ud = to_device(factors.U[:k], tag)
    Td = to_device(factors.T, "double")
    Sd = to_device(factors.S, "double")
    od = Sd.shape[0]
    Q = empty_colmajor(od, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_sketch_q(ctx.h, CODES[tag], Ud.data_ptr(), ld_of(Ud), k, Td.data_ptr(),
                                      ld_of(Td), Sd.data_ptr(), ld_of(Sd), od, Q.data_ptr(), ld_of(Q)),
              "sqb_sketch_q")
    return _out(Q, host)


__all__ = ["HouseholderStep", "RHQRFactors", "QRResult", "householder_qr", "upper_tri_solve",
           "BlockPanel", "BlockRHQRFactors", "rhqr_block", "rhqr_right", "t_factor_from_sketches",
           "lsq_via_implicit_q", "rh_vector", "rhqr_left", "rec_rhqr", "apply_reflectors_compact",
           "thin_q", "sketch_q", "SCALE_SQRT2", "SCALE_UNIT", "raise_status", "_embed", "right_tri_solve"]
_ = C
