"""Trimmed randomized Householder QR (mirror of trim.py) on the sm_100a library.

The reflector for column j sketches only coordinates j..n of its input, so
the sampling size ell may be smaller than the column count m.  The operator
is wrapped so its m leading columns sketch to unit vectors
(`normalize_leading_columns`, trim.py:51-77); the factorization then keeps
two compact-form triangles (T in creation order, T~ reversed) and the
strictly lower table L[i, k] = <Omega u_i, Omega e_k>.

`trim_rhqr_left` / `trim_rhqr_right` run the whole column sweep on the
device (csrc/trim.cu: column-scaled K1 sketches, single-CTA sketch-space
kernels, a streaming GEMV or rank-1 update); this module validates arguments exactly as the
reference does, builds the wrapper (a one-time sketch construction, like the
SRHT's signs), moves operands across the boundary and maps device status
words to the reference's exceptions.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .devarray import CODES, empty_colmajor, is_device, ld_of, to_device, to_numpy
from .linalg import SCALE_SQRT2, BreakdownError, check_scaling, scaling_code
from .precision import DOUBLE_POLICY, require_device_policy
from .sketching import SketchOperator, SRHTSketch, _columns, _device_input, _dtype_tag


class ColumnScaledSketch(SketchOperator):
    """sketching.py:216-235: rescale the m leading input coordinates (in the
    arithmetic dtype), then apply the base operator; `unit_column_sketches`
    caches the ell x m unit sketches of the leading columns."""

    kind = "colscaled"

    def __init__(self, base, scales, m, unit_column_sketches):
        super().__init__(base.ell, base.n, base.seed)
        self.base = base
        self.m = int(m)
        self.scales = np.asarray(scales, dtype=np.float64)
        self.unit_column_sketches = unit_column_sketches

    def desc(self):
        return self.base.desc()

    def device_scales(self):
        dev = torch.cuda.current_device()
        key = ("scales", dev)
        t = self._dev.get(key)
        if t is None:
            t = self._dev[key] = torch.from_numpy(np.ascontiguousarray(self.scales[: self.m])).to(
                device=f"cuda:{dev}")
        return t

    def apply(self, X, dtype=np.float64):
        """sketching.py:230-235 (through sqb_colscaled_apply)."""
        X2, vec = _columns(X, self.n)
        tag = _dtype_tag(dtype)
        Xd = _device_input(X2, tag)
        k = Xd.shape[1]
        Y = empty_colmajor(self.ell, k, "double")
        sc = self.device_scales()
        ctx = _lib.context()
        ctx.check(_lib.lib().sqb_colscaled_apply(ctx.h, self.desc(), sc.data_ptr(), self.m, CODES[tag],
                                                 Xd.data_ptr(), ld_of(Xd), k, Y.data_ptr(), ld_of(Y)),
                  "sqb_colscaled_apply")
        out = Y[:, 0] if vec else Y
        return out if is_device(X) else to_numpy(out)


def _srht_unit_columns(omega, m):
    """Omega e_k, k < m, of an SRHT in closed form: the FWHT of a one-hot
    vector adds only exact zeros, so every entry is
    sign_k (-1)^popcount(idx_i & k) fl(fl(1 * scale) n_pad^-1/2) — bitwise
    the reference's sketching.py:149-155 on I[:, :m] (tests pin it)."""
    a = np.float64(np.float64(1.0) * np.float64(omega.scale)) * np.float64(omega.n_pad ** -0.5)
    k = np.arange(m, dtype=np.int64)
    x = np.asarray(omega.indices, dtype=np.int64)[:, None] & k[None, :]
    par = np.zeros_like(x)
    while np.any(x):
        par ^= x & 1
        x >>= 1
    return (np.where(par == 1, -1.0, 1.0) * np.asarray(omega.signs[:m], dtype=np.float64)[None, :]) * a


def normalize_leading_columns(omega, m, chunk=256):
    """trim.py:51-77: wrap omega so its first m columns sketch to unit norm.
    The unit sketches of an SRHT come in closed form; any other operator
    sketches identity blocks on the device, `chunk` columns at a time."""
    if isinstance(omega, ColumnScaledSketch) and omega.m >= m:
        return omega
    n = omega.n
    if m > n:
        raise ValueError(f"cannot normalize {m} leading columns of {n} inputs")
    if isinstance(omega, SRHTSketch):
        cols = _srht_unit_columns(omega, m)
    else:
        cols = np.empty((omega.ell, m))
        for k0 in range(0, m, chunk):
            k1 = min(k0 + chunk, m)
            eye_blk = np.zeros((n, k1 - k0))
            eye_blk[np.arange(k0, k1), np.arange(k1 - k0)] = 1.0
            cols[:, k0:k1] = omega.apply(eye_blk)
    norms = np.linalg.norm(cols, axis=0)
    if np.any(norms == 0.0):
        dead = int(np.argmin(norms)) + 1
        raise ValueError(f"leading column {dead} sketches to zero")
    scales = np.ones(n)
    scales[:m] = 1.0 / norms
    return ColumnScaledSketch(omega, scales, m, cols / norms)


@dataclass
class TrimStep:
    """trim.py:36-47: one trimmed reflector (elimination index j, 1-based; tail
    vector v of length n-j+1; its sketch s = Omega [0; v]; the scalars)."""

    j: int
    v: object
    s: object
    sigma: float
    rho: float
    beta: float


def trim_rh_vector(w_tail, omega, j, scaling=SCALE_SQRT2, policy=None):
    """trim.py:79-146: the reflector of the trimmed elimination at column j, on
    the device: the two sketches Omega [0; w_tail] and Omega [0; v] through
    the operator's kernels, the scalars in float64 (the column sweep's
    trim_tail / trim_finish kernels compute the same quantities in place;
    this is the single-step form the reference exposes)."""
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    from .devarray import TORCH_DTYPES
    host = not is_device(w_tail)
    lo_t = TORCH_DTYPES[policy.low]
    wt = to_device(w_tail, "double")[:, 0]
    n = omega.n
    jj = j - 1
    if not 0 <= jj < n:
        raise ValueError(f"elimination index {j} outside {n} coordinates")
    if wt.shape[0] != n - jj:
        raise ValueError(f"tail has {wt.shape[0]} entries, expected {n - jj}")
    lo_np = _np_lo(policy.low)
    x = torch.zeros(n, dtype=torch.float64, device=wt.device)
    x[jj:] = wt
    z = omega.apply(x, dtype=lo_np)
    rho = float(torch.linalg.norm(z))
    if rho == 0.0:
        raise BreakdownError(f"sketched tail annihilated at column {j}")
    w0 = float(wt[0])
    sigma = 1.0 if w0 >= 0.0 else -1.0
    v = wt.clone()
    v[0] += sigma * rho
    v = v.to(lo_t).to(torch.float64)  # round_to(v, low)
    x[jj:] = v
    vs = omega.apply(x, dtype=lo_np)
    nv = float(torch.linalg.norm(vs))
    u_high = 2.0 ** -53  # sketch-space arithmetic is float64 on the device
    if nv <= 8.0 * u_high * (rho + rho):
        raise BreakdownError(f"sketched reflector vector cancelled at column {j} "
                             f"(degenerate sketch geometry, norm {nv:.3e})")
    beta = 2.0 / (nv * nv)
    if scaling == SCALE_SQRT2:
        f = float(np.sqrt(beta))
        v = v * f
        vs = vs * f
        beta = 1.0
    else:
        piv = float(vs[0])
        if abs(piv) <= 8.0 * u_high * nv:
            raise BreakdownError(f"unit scaling pivot vanished at column {j} (sketched entry {piv:.3e})")
        v = v / piv
        vs = vs / piv
        beta = beta * piv * piv
    v = v.to(lo_t).to(torch.float64)
    o = (lambda t: to_numpy(t)) if host else (lambda t: t)
    return TrimStep(j=j, v=o(v), s=o(vs), sigma=sigma, rho=rho, beta=float(beta))


def _np_lo(tag):
    from .precision import DTYPES
    return DTYPES[tag]


def t_tilde_from_factors(S, E, U, policy=None):
    """trim.py:179-196: the reversed-product triangle from S, E and U's leading
    block: A = L U[:m] - tril(S^t S, -1) - diag(S^t S) / 2 is lower triangular
    and T~^t = -A^{-1} (device products and the device triangular solve)."""
    from .rhqr import upper_tri_solve
    host = not is_device(S)
    Sd = to_device(S, "double")
    m = Sd.shape[1]
    Ed = to_device(E, "double")[:, :m]
    Ud = (U if is_device(U) else torch.from_numpy(np.ascontiguousarray(np.asarray(U, dtype=np.float64)[:m])).cuda())
    Ud = Ud[:m].to(torch.float64)
    G = Sd.t() @ Sd
    L = torch.tril(Sd.t() @ Ed, -1)
    A = L @ Ud - torch.tril(G, -1) - torch.diag(torch.diagonal(G) / 2.0)
    X = upper_tri_solve(A.t().contiguous(), torch.eye(m, dtype=torch.float64, device=Sd.device))
    out = -X
    return to_numpy(out) if host else out


@dataclass
class TrimFactors:
    """trim.py:149-186: W = (I - U T ut((Omega U)^t Omega)) [R; 0]."""

    U: object
    S: object
    T: object
    T_tilde: object
    R: object
    L: object
    E: object
    omega: ColumnScaledSketch
    scaling: str
    sigmas: object
    rhos: object
    betas: object

    @property
    def cols(self):
        return self.U.shape[1]

    def prefix(self, j):
        """trim.py:175-186."""
        return TrimFactors(
            U=self.U[:, :j], S=self.S[:, :j], T=self.T[:j, :j], T_tilde=self.T_tilde[:j, :j],
            R=self.R[:j, :j], L=self.L[:j, :j], E=self.E[:, :j], omega=self.omega, scaling=self.scaling,
            sigmas=self.sigmas[:j], rhos=self.rhos[:j], betas=self.betas[:j])


def _trim_setup(W, omega, m):
    """trim.py:228-235."""
    if (W.dim() if is_device(W) else np.ndim(W)) != 2:
        raise ValueError("W must be a matrix")
    omega = normalize_leading_columns(omega, m)
    if omega.n != W.shape[0]:
        raise ValueError(f"sketch takes {omega.n} coordinates, W has {W.shape[0]} rows")
    return omega


def _raise_trim_status(ctx):
    code, col, val = ctx.status()
    if code == _lib.SQB_OK:
        return
    if code == _lib.SQB_ERR_BREAKDOWN:
        j, kind = col & 0xFFFFFF, col >> 24
        if kind == 0:
            raise BreakdownError(f"sketched tail annihilated at column {j}")
        if kind == 1:
            raise BreakdownError(f"sketched reflector vector cancelled at column {j} "
                                 f"(degenerate sketch geometry, norm {val:.3e})")
        raise BreakdownError(f"unit scaling pivot vanished at column {j} (sketched entry {val:.3e})")
    if code == _lib.SQB_ERR_SINGULAR:
        from .linalg import SingularFactorError
        raise SingularFactorError("triangular factor has zero or subnormal diagonal")
    if code == _lib.SQB_ERR_NONFINITE:  # scipy's check_finite in the reference's triangular solves
        raise ValueError("array must not contain infs or NaNs")
    raise _lib.SketchQRError(f"trimmed factorization: device status {code} at column {col}")


def trim_rhqr_left(W, omega, scaling=SCALE_SQRT2, policy=None):
    """trim.py:272-325: left-looking trimmed factorization maintaining both
    triangles; column j is transformed by the reversed compact form
    w -= U T~^t (S^t (Omega w) - L w_head), then reflected from its tail."""
    return _trim_run("sqb_trim_rhqr_left", W, omega, scaling, policy)


def trim_rhqr_right(W, omega, scaling=SCALE_SQRT2, policy=None):
    """trim.py:238-269: right-looking trimmed factorization; each reflector
    updates the trailing columns through the masked sketch, and T, T~ and L
    are assembled from S and E after the sweep."""
    return _trim_run("sqb_trim_rhqr_right", W, omega, scaling, policy)


def _trim_run(entry, W, omega, scaling, policy):
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    if not host and W.dim() != 2 or host and np.ndim(W) != 2:
        raise ValueError("W must be a matrix")
    n, m = tuple(W.shape)
    omega = _trim_setup(W, omega, m)
    tag = policy.low
    Wd = to_device(W, tag)
    E = omega.unit_column_sketches[:, :m]
    Ed = to_device(np.ascontiguousarray(E), "double")
    sc = omega.device_scales()
    ell = omega.ell
    U = empty_colmajor(n, m, tag)
    S = empty_colmajor(ell, m, "double")
    T = empty_colmajor(m, m, "double")
    Tt = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    L = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device=Wd.device)
    ctx = _lib.context()
    ctx.check(getattr(_lib.lib(), entry)(
        ctx.h, omega.desc(), sc.data_ptr(), omega.m, Ed.data_ptr(), ld_of(Ed), scaling_code(scaling), CODES[tag],
        Wd.data_ptr(), n, m, ld_of(Wd), U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T),
        Tt.data_ptr(), ld_of(Tt), R.data_ptr(), ld_of(R), L.data_ptr(), ld_of(L), scal.data_ptr(),
        scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m), entry)
    _raise_trim_status(ctx)
    o = (lambda t: to_numpy(t)) if host else (lambda t: t)
    return TrimFactors(U=o(U), S=o(S), T=o(T), T_tilde=o(Tt), R=o(R), L=o(L),
                       E=np.array(E) if host else Ed, omega=omega, scaling=scaling, sigmas=o(scal[:m]),
                       rhos=o(scal[m:2 * m]), betas=o(scal[2 * m:]))


def trim_thin_q(factors):
    """trim.py:211-225: Q = [I_m; 0] - U T triu(S^t E) in float64."""
    host = not is_device(factors.U)
    Ud = factors.U if not host else to_device(factors.U, "double")
    tag = {torch.float64: "double", torch.float32: "single", torch.float16: "half",
           torch.bfloat16: "bf16"}[Ud.dtype]
    Ud = to_device(Ud, tag)
    Td = to_device(factors.T, "double")
    Sd = to_device(factors.S, "double")
    Ed = to_device(factors.E, "double")
    N, k = Ud.shape
    Q = empty_colmajor(N, k, "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_trim_thin_q(ctx.h, CODES[tag], Ud.data_ptr(), ld_of(Ud), N, k, Td.data_ptr(),
                                         ld_of(Td), Sd.data_ptr(), ld_of(Sd), Ed.data_ptr(), ld_of(Ed),
                                         Sd.shape[0], Q.data_ptr(), ld_of(Q)), "sqb_trim_thin_q")
    return to_numpy(Q) if host else Q
