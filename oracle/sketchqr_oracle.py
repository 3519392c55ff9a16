"""CPU oracle for the RHQR hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package's
(`sketchqr`, arXiv 2405.10923) algorithms on the hot path.  It exists so
that the parity tests, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg have a checker that travels to the GPU
box (the reference tree does not).  The product package
(`paper_2405_10923_b200`) never imports it: every product computation runs in
the sm_100a CUDA library and fails loudly when that library is missing.

Pinning: the restatement is checked against golden vectors produced by the
reference itself (`tests/golden/make_golden.py` imports
/root/reference/pkg/src/sketchqr in the build container and records its
outputs); `tests/test_oracle_golden.py` asserts bitwise equality for the
sketches and tight tolerances for the BLAS-dependent factors.

Every function cites the reference file:line it restates.  Paths are relative
to /root/reference/pkg/src/sketchqr/.

Emulation model (precision.py:1-7): arrays are float64 carrying values that
are exactly representable in the low format; each elementary op is done in
the native numpy dtype (round-to-nearest-even).  A "bf16" tag is added here
(ml_dtypes.bfloat16, u = 2^-8) — the reference has no bf16, SURVEY A.6 shows
the identical injection.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.linalg

try:  # bf16 storage is an extension of the reference's precision tags
    import ml_dtypes

    _BF16 = np.dtype(ml_dtypes.bfloat16)
except Exception:  # pragma: no cover - ml_dtypes ships in the image
    _BF16 = None

# --------------------------------------------------------------------------
# precision.py:12-109
# --------------------------------------------------------------------------
TAG_DTYPE = {"half": np.dtype(np.float16), "single": np.dtype(np.float32),
             "double": np.dtype(np.float64)}
TAG_U = {"half": 2.0 ** -11, "single": 2.0 ** -24, "double": 2.0 ** -53}
if _BF16 is not None:
    TAG_DTYPE["bf16"] = _BF16
    TAG_U["bf16"] = 2.0 ** -8


class BreakdownError(RuntimeError):
    """linalg.py:18-19."""


class PrecisionRangeError(ArithmeticError):
    """precision.py:25-26."""


def round_to(a, tag):
    """precision.py:34-51: round to `tag`, raise on finite overflow."""
    a = np.asarray(a, dtype=np.float64)
    if tag == "double":
        return a.copy()
    with np.errstate(over="ignore"):
        r = a.astype(TAG_DTYPE[tag])
    bad = np.isfinite(a) & ~np.isfinite(r.astype(np.float64))
    if bad.any():
        raise PrecisionRangeError(f"value {np.abs(a[bad]).max():g} overflows {tag} range")
    return r.astype(np.float64)


@dataclass(frozen=True)
class Policy:
    """precision.py:54-98 (high for sketch-space, low for n-dimensional)."""

    high: str = "double"
    low: str = "double"

    @property
    def hi(self):
        return TAG_DTYPE[self.high]

    @property
    def lo(self):
        return TAG_DTYPE[self.low]

    @property
    def u_high(self):
        return TAG_U[self.high]

    @property
    def u_low(self):
        return TAG_U[self.low]


DOUBLE = Policy()


def policy_from_tag(tag):
    """precision.py:104-109 ('mixed' = half storage, double coefficients)."""
    if tag == "mixed":
        return Policy("double", "half")
    if tag == "mixed_bf16":
        return Policy("double", "bf16")
    return Policy(tag, tag)


def sign(v):
    """linalg.py:200-202: sign(0) = +1."""
    return 1.0 if v >= 0.0 else -1.0


def _cast(a, dt):
    a = np.asarray(a)
    return a if a.dtype == dt else a.astype(dt)


# --------------------------------------------------------------------------
# sketching.py
# --------------------------------------------------------------------------
def fwht(x):
    """sketching.py:21-43.  Butterfly stages h = 1, 2, 4, ... with
    (a + b, a - b) on the pair (i, i + h), then one multiply by n^-1/2
    rounded to x's dtype.  Arithmetic stays in x's dtype."""
    a = np.array(x, copy=True)
    n = a.shape[0]
    if n == 0 or n & (n - 1):
        raise ValueError(f"length {n} is not a power of two")
    vec = a.ndim == 1
    a = a.reshape(n, -1)
    k = a.shape[1]
    h = 1
    while h < n:
        v = a.reshape(n // (2 * h), 2, h, k)
        lo = v[:, 0].copy()
        hi = v[:, 1].copy()
        v[:, 0] = lo + hi
        v[:, 1] = lo - hi
        h <<= 1
    a = a * a.dtype.type(n ** -0.5)
    return a[:, 0] if vec else a


def _cols(X, n):
    """sketching.py:46-53."""
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    if vec:
        X = X[:, None]
    if X.shape[0] != n:
        raise ValueError(f"operand has {X.shape[0]} rows, operator expects {n}")
    return X, vec


class SRHT:
    """sketching.py:128-155.  sqrt(n_pad/ell) * P * H * diag(signs), zero pad."""

    kind = "srht"

    def __init__(self, ell, n, seed):
        if ell < 1 or n < 1:
            raise ValueError(f"invalid sketch dimensions {ell} x {n}")
        self.ell, self.n, self.seed = int(ell), int(n), int(seed)
        self.n_pad = 1 << (self.n - 1).bit_length()
        if self.ell > self.n_pad:
            raise ValueError(f"ell={ell} exceeds padded length {self.n_pad}")
        g = np.random.Generator(np.random.Philox(key=[self.seed, (1 << 40) + 1]))
        self.signs = (g.integers(0, 2, self.n_pad) * 2 - 1).astype(np.float64)
        self.indices = g.permutation(self.n_pad)[: self.ell].copy()
        self.scale = float(np.sqrt(self.n_pad / self.ell))

    def apply(self, X, dtype=np.float64):
        """sketching.py:72-76 + 149-155: scale, signs, pad, fwht, gather."""
        X, vec = _cols(X, self.n)
        dt = np.dtype(dtype)
        buf = np.zeros((self.n_pad, X.shape[1]), dtype=dt)
        buf[: self.n] = X.astype(dt) * dt.type(self.scale)
        buf[: self.n] *= self.signs[: self.n, None].astype(dt)
        Y = fwht(buf)[self.indices].astype(np.float64)
        return Y[:, 0] if vec else Y


class Gaussian:
    """sketching.py:82-125.  Row i from Philox(key=[seed, i]), scaled by
    ell^-1/2.  fp16 applies accumulate in fp32 (sketching.py:111)."""

    kind = "gauss"

    def __init__(self, ell, n, seed, materialize=True):
        if ell < 1 or n < 1:
            raise ValueError(f"invalid sketch dimensions {ell} x {n}")
        self.ell, self.n, self.seed = int(ell), int(n), int(seed)
        self.G = self.rows(0, self.ell) if materialize else None

    def rows(self, i0, i1):
        G = np.empty((i1 - i0, self.n))
        for i in range(i0, i1):
            G[i - i0] = np.random.Generator(
                np.random.Philox(key=[self.seed, i])).standard_normal(self.n)
        G *= self.ell ** -0.5
        return G

    def apply(self, X, dtype=np.float64):
        X, vec = _cols(X, self.n)
        dt = np.dtype(dtype)
        acc = np.dtype(np.float32) if dt == np.float16 else dt
        G = self.G if self.G is not None else self.rows(0, self.ell)
        Y = (G.astype(acc) @ X.astype(acc)).astype(dt).astype(np.float64)
        return Y[:, 0] if vec else Y


class Identity:
    """sketching.py:186-195."""

    kind = "identity"

    def __init__(self, n):
        self.ell = self.n = int(n)
        self.seed = 0

    def apply(self, X, dtype=np.float64):
        X, vec = _cols(X, self.n)
        Y = X.astype(np.dtype(dtype)).astype(np.float64)
        return Y[:, 0] if vec else Y


class Embedded:
    """sketching.py:238-260: Psi = [I_m; Omega], top block bitwise."""

    def __init__(self, m, omega):
        self.m = int(m)
        self.omega = omega
        self.n = self.m + omega.n
        self.out_dim = self.m + omega.ell

    def apply(self, X, dtype=np.float64):
        X, vec = _cols(X, self.n)
        Y = np.concatenate([X[: self.m].copy(),
                            self.omega.apply(X[self.m:], dtype=dtype)], axis=0)
        return Y[:, 0] if vec else Y


def embed(omega, n, m):
    """rhqr.py:202-216."""
    if isinstance(omega, Embedded):
        if omega.n != n or omega.m != m:
            raise ValueError("embedding shape mismatch")
        if omega.omega.ell < m:
            raise ValueError("sampling size below column count")
        return omega
    if omega.n != n - m:
        raise ValueError(f"sketch takes {omega.n} coordinates, expected n-m={n - m}")
    if omega.ell < m:
        raise ValueError("sampling size below column count")
    return Embedded(m, omega)


# --------------------------------------------------------------------------
# rhqr.py
# --------------------------------------------------------------------------
@dataclass
class Step:
    """rhqr.py:38-48."""

    j: int
    u: np.ndarray
    s: np.ndarray
    sigma: float
    rho: float
    beta: float


def rh_vector(w, y, j, scaling="sqrt2", policy=DOUBLE):
    """rhqr.py:51-97."""
    w = np.asarray(w, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    p = j - 1
    if not 0 <= p < y.shape[0]:
        raise ValueError(f"elimination index {j} outside sketch of length {y.shape[0]}")
    hi = policy.hi.type
    rho = float(round_to(np.linalg.norm(y[p:]), policy.high))
    if rho == 0.0:
        raise BreakdownError(f"sketched tail annihilated at column {j}")
    sg = sign(y[p])
    gamma = float(hi(y[p] + sg * rho))
    beta = float(hi(1.0 / (rho * sg * gamma)))
    if not np.isfinite(beta):
        raise BreakdownError(f"reflector scale degenerated at column {j} (rho={rho:.3e})")
    u = np.zeros(w.shape[0])
    u[p:] = w[p:]
    u[p] += sg * rho
    s = np.zeros(y.shape[0])
    s[p:] = y[p:]
    s[p] = gamma
    if scaling == "sqrt2":
        f = float(hi(np.sqrt(beta)))
        u *= f
        s *= f
        beta = 1.0
    else:
        u /= gamma
        s /= gamma
        beta = float(hi(sg * gamma / rho))
    return Step(j, round_to(u, policy.low), round_to(s, policy.high), sg, rho, beta)


def extend_t(T, S, s_new, beta, c, hi=np.float64):
    """rhqr.py:135-140."""
    if c:
        v = _cast(S[:, :c], hi).T @ _cast(s_new, hi)
        col = _cast(T[:c, :c], hi) @ v
        T[:c, c] = (hi(-beta) * col).astype(np.float64)
    T[c, c] = beta


def apply_reflectors_compact(U, S, T, X, psi, transpose_t=False, policy=DOUBLE):
    """rhqr.py:100-119."""
    lo, hi = policy.lo, policy.hi
    X = np.asarray(X, dtype=np.float64)
    vec = X.ndim == 1
    Xc = X[:, None] if vec else X
    Y = psi.apply(Xc, dtype=lo)
    C = _cast(np.asarray(S), hi).T @ _cast(Y, hi)
    C = _cast(np.asarray(T).T if transpose_t else np.asarray(T), hi) @ C
    out = (_cast(Xc, lo) - _cast(np.asarray(U), lo) @ _cast(C, lo)).astype(np.float64)
    return out[:, 0] if vec else out


@dataclass
class Factors:
    """rhqr.py:143-168."""

    U: np.ndarray
    S: np.ndarray
    T: np.ndarray
    R: np.ndarray
    psi: Embedded
    scaling: str
    sigmas: np.ndarray
    rhos: np.ndarray
    betas: np.ndarray

    def prefix(self, j):
        return Factors(self.U[:, :j], self.S[:, :j], self.T[:j, :j], self.R[:j, :j],
                       self.psi, self.scaling, self.sigmas[:j], self.rhos[:j],
                       self.betas[:j])


def thin_q(F):
    """rhqr.py:171-178."""
    U = np.asarray(F.U)
    k = U.shape[1]
    Q = -U @ (np.asarray(F.T) @ U[:k, :k].T)
    Q[:k] += np.eye(k)
    return Q


def sketch_q(F):
    """rhqr.py:181-188."""
    U = np.asarray(F.U)
    k = U.shape[1]
    Q = -np.asarray(F.S) @ (np.asarray(F.T) @ U[:k, :k].T)
    Q[:k] += np.eye(k)
    return Q


def upper_tri_solve(R, B, policy=DOUBLE):
    """linalg.py:102-116 (double/single path through LAPACK)."""
    d = np.abs(np.diagonal(R))
    if np.any(d < np.finfo(policy.hi).tiny):
        raise np.linalg.LinAlgError("triangular factor has zero or subnormal diagonal")
    return scipy.linalg.solve_triangular(np.asarray(R, dtype=policy.hi),
                                         np.asarray(B, dtype=policy.hi),
                                         lower=False).astype(np.float64)


def right_tri_solve(B, R, policy=DOUBLE):
    """linalg.py:119-129: X R = B via the transposed lower solve."""
    d = np.abs(np.diagonal(R))
    if np.any(d < np.finfo(policy.hi).tiny):
        raise np.linalg.LinAlgError("triangular factor has zero or subnormal diagonal")
    X = scipy.linalg.solve_triangular(np.asarray(R, dtype=policy.hi).T,
                                      np.asarray(B, dtype=policy.hi).T, lower=True).T
    return X.astype(np.float64)


def lsq_via_implicit_q(F, b, policy=DOUBLE):
    """rhqr.py:191-199."""
    c = apply_reflectors_compact(F.U, F.S, F.T, b, F.psi, transpose_t=True, policy=policy)
    m = F.R.shape[1]
    return upper_tri_solve(F.R, c[:m], policy=policy)


def left_sweep(Wl, psi, offset, scaling, policy):
    """rhqr.py:219-251: the hot loop."""
    lo, hi = policy.lo, policy.hi
    n, b = Wl.shape
    U = np.zeros((n, b))
    S = np.zeros((psi.out_dim, b))
    T = np.zeros((b, b))
    R = np.zeros((offset + b, b))
    sig, rho, bet = np.zeros(b), np.zeros(b), np.zeros(b)
    for c in range(b):
        j = offset + c + 1
        w = Wl[:, c].astype(np.float64)
        if c:
            y = psi.apply(w, dtype=lo)
            g = _cast(S[:, :c], hi).T @ _cast(y, hi)
            coef = _cast(T[:c, :c].T, hi) @ g
            w = (_cast(w, lo) - _cast(U[:, :c], lo) @ _cast(coef, lo)).astype(np.float64)
        y = psi.apply(w, dtype=lo)
        st = rh_vector(w, y, j, scaling, policy)
        U[:, c] = st.u
        S[:, c] = st.s
        extend_t(T, S, st.s, st.beta, c, hi.type)
        R[: j - 1, c] = w[: j - 1]
        R[j - 1, c] = -st.sigma * st.rho
        sig[c], rho[c], bet[c] = st.sigma, st.rho, st.beta
    return U, S, T, R, sig, rho, bet


def rhqr_left(W, omega, scaling="sqrt2", policy=DOUBLE):
    """rhqr.py:254-267."""
    W = np.asarray(W, dtype=np.float64)
    n, m = W.shape
    psi = embed(omega, n, m)
    Wl = round_to(W, policy.low)
    U, S, T, R, sg, rh, bt = left_sweep(Wl, psi, 0, scaling, policy)
    return Factors(U, S, T, R, psi, scaling, sg, rh, bt)


def t_factor_from_sketches(S, policy=DOUBLE):
    """rhqr.py:122-132: S^t S = T^{-1} + T^{-t}; T^{-1} = triu(G, 1) + diag(G)/2."""
    Sh = _cast(np.asarray(S), policy.hi)
    G = (Sh.T @ Sh).astype(np.float64)
    Tinv = np.triu(G, 1) + np.diag(np.diagonal(G) / 2.0)
    return upper_tri_solve(Tinv, np.eye(G.shape[0]), policy=policy)


@dataclass
class BlockPanel:
    """rhqr.py:304-309."""

    U: np.ndarray
    S: np.ndarray
    T: np.ndarray
    offset: int


@dataclass
class BlockFactors:
    """rhqr.py:312-331 (BlockRHQRFactors)."""

    panels: list
    R: np.ndarray
    psi: Embedded
    scaling: str
    sigmas: np.ndarray
    rhos: np.ndarray
    betas: np.ndarray

    def stacked(self):
        U = np.concatenate([p.U for p in self.panels], axis=1)
        S = np.concatenate([p.S for p in self.panels], axis=1)
        return Factors(U, S, t_factor_from_sketches(S), self.R, self.psi, self.scaling,
                       self.sigmas, self.rhos, self.betas)


def rhqr_block(W, omega, block_size=32, scaling="sqrt2", policy=DOUBLE):
    """rhqr.py:334-365: earlier panels applied compactly (one re-sketch per
    panel, coefficients in high, update in low), then the panel is swept."""
    if block_size < 1:
        raise ValueError("block_size must be positive")
    lo, hi = policy.lo, policy.hi
    W = np.asarray(W, dtype=np.float64)
    n, m = W.shape
    psi = embed(omega, n, m)
    Wl = round_to(W, policy.low)
    panels = []
    R = np.zeros((m, m))
    sig, rho, bet = np.zeros(m), np.zeros(m), np.zeros(m)
    for j0 in range(0, m, block_size):
        j1 = min(j0 + block_size, m)
        X = Wl[:, j0:j1].copy()
        for p in panels:
            Y = psi.apply(X, dtype=lo)
            coef = _cast(p.T.T, hi) @ (_cast(p.S, hi).T @ _cast(Y, hi))
            X = (_cast(X, lo) - _cast(p.U, lo) @ _cast(coef, lo)).astype(np.float64)
        U, S, T, Rp, sg, rh, bt = left_sweep(X, psi, j0, scaling, policy)
        R[:j1, j0:j1] = Rp
        sig[j0:j1], rho[j0:j1], bet[j0:j1] = sg, rh, bt
        panels.append(BlockPanel(U, S, T, j0))
    return BlockFactors(panels, R, psi, scaling, sig, rho, bet)


def rhqr_right(W, omega, scaling="sqrt2", policy=DOUBLE):
    """rhqr.py:270-301: rank-1 update of the trailing block, re-sketched
    wholesale at every step; T recovered from S afterwards."""
    lo, hi = policy.lo, policy.hi
    W = np.asarray(W, dtype=np.float64)
    n, m = W.shape
    psi = embed(omega, n, m)
    Wl = round_to(W, policy.low)
    U = np.zeros((n, m))
    S = np.zeros((psi.out_dim, m))
    R = np.zeros((m, m))
    sig, rho, bet = np.zeros(m), np.zeros(m), np.zeros(m)
    for c in range(m):
        Y = psi.apply(Wl[:, c:], dtype=lo)
        st = rh_vector(Wl[:, c], Y[:, 0], c + 1, scaling, policy)
        U[:, c] = st.u
        S[:, c] = st.s
        R[:c, c] = Wl[:c, c]
        R[c, c] = -st.sigma * st.rho
        sig[c], rho[c], bet[c] = st.sigma, st.rho, st.beta
        if c + 1 < m:
            coef = hi.type(st.beta) * (_cast(st.s, hi) @ _cast(Y[:, 1:], hi))
            tail = _cast(Wl[:, c + 1:], lo) - np.outer(_cast(st.u, lo), _cast(coef, lo))
            Wl[:, c + 1:] = tail.astype(np.float64)
    T = t_factor_from_sketches(S, policy=policy)
    return Factors(U, S, T, R, psi, scaling, sig, rho, bet)


def householder_qr(A, scaling="sqrt2", policy=DOUBLE):
    """baselines.py:33-89: left-looking HQR with compact T (used by recRHQR)."""
    lo, hi = policy.lo, policy.hi
    A = np.asarray(A, dtype=np.float64)
    p, m = A.shape
    if p < m:
        raise ValueError(f"need p >= m, got {p} x {m}")
    Al = round_to(A, policy.low)
    U = np.zeros((p, m))
    T = np.zeros((m, m))
    R = np.zeros((m, m))
    sig, rho_a, bet = np.zeros(m), np.zeros(m), np.zeros(m)
    for c in range(m):
        w = Al[:, c].astype(np.float64)
        if c:
            coef = _cast(T[:c, :c].T, hi) @ (_cast(U[:, :c], hi).T @ _cast(w, hi))
            w = (_cast(w, lo) - _cast(U[:, :c], lo) @ _cast(coef, lo)).astype(np.float64)
        rho = float(round_to(np.linalg.norm(w[c:]), policy.high))
        if rho == 0.0:
            raise BreakdownError(f"column {c + 1} exactly dependent on its predecessors")
        sg = sign(w[c])
        gamma = float(hi.type(w[c] + sg * rho))
        beta = float(hi.type(1.0 / (rho * sg * gamma)))
        u = np.zeros(p)
        u[c:] = w[c:]
        u[c] = gamma
        if scaling == "sqrt2":
            u *= float(hi.type(np.sqrt(beta)))
            beta = 1.0
        else:
            u /= gamma
            beta = float(hi.type(sg * gamma / rho))
        u = round_to(u, policy.low)
        U[:, c] = u
        if c:
            col = _cast(T[:c, :c], hi) @ (_cast(U[:, :c], hi).T @ _cast(u, hi))
            T[:c, c] = (hi.type(-beta) * col).astype(np.float64)
        T[c, c] = beta
        R[:c, c] = w[:c]
        R[c, c] = -sg * rho
        sig[c], rho_a[c], bet[c] = sg, rho, beta
    Q = -U @ (T @ U[:m, :m].T)
    Q[:m] += np.eye(m)
    return Q, R, {"U": U, "T": T, "sigmas": sig, "rhos": rho_a, "betas": bet}


def rec_rhqr(W, omega, scaling="sqrt2", policy=DOUBLE):
    """rhqr.py:368-395."""
    W = np.asarray(W, dtype=np.float64)
    n, m = W.shape
    psi = embed(omega, n, m)
    Wl = round_to(W, policy.low)
    Z = psi.apply(Wl, dtype=policy.lo)
    _, Rz, aux = householder_qr(Z, scaling=scaling, policy=Policy(policy.high, policy.high))
    S, T = aux["U"], aux["T"]
    hi = policy.hi
    M = np.triu(_cast(T.T, hi) @ (_cast(S, hi).T @ _cast(Z, hi))).astype(np.float64)
    d = np.abs(np.diagonal(M))
    if np.any(d < np.finfo(np.float64).tiny):
        raise BreakdownError(
            f"reconstruction factor has zero diagonal at column {int(np.argmin(d)) + 1}")
    U2 = right_tri_solve(Wl[m:], M, policy=policy)
    U = np.concatenate([S[:m], round_to(U2, policy.low)], axis=0)
    return Factors(U, S, T, Rz, psi, scaling, aux["sigmas"], aux["rhos"], aux["betas"])


# --------------------------------------------------------------------------
# krylov.py
# --------------------------------------------------------------------------
def as_operator(A):
    """krylov.py:28-35."""
    if callable(A):
        return A
    return lambda v: A @ v


@dataclass
class Krylov:
    """krylov.py:38-61."""

    U: np.ndarray
    S: np.ndarray
    T: np.ndarray
    H: np.ndarray
    psi: Embedded
    beta: float
    scaling: str
    Q_cols: np.ndarray = None
    breakdown: int = None
    y: np.ndarray = None
    resid_history: np.ndarray = None

    @property
    def dim(self):
        return self.H.shape[1]


def rhqr_arnoldi(A, b, x0, m, omega, scaling="sqrt2", policy=DOUBLE,
                 store_q=True, happy_tol=None):
    """krylov.py:82-150."""
    lo, hi = policy.lo, policy.hi
    mv = as_operator(A)
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    psi = embed(omega, n, m + 1)
    if happy_tol is None:
        happy_tol = 32.0 * policy.u_high
    r = m + 1
    U = np.zeros((n, r))
    S = np.zeros((psi.out_dim, r))
    T = np.zeros((r, r))
    Hc = np.zeros((m + 1, m))
    Q = np.zeros((n, m))
    beta = 0.0
    closed = None
    w = round_to(b - mv(round_to(x0, policy.low)), policy.low).astype(np.float64)
    z = psi.apply(w, dtype=lo)
    for j in range(1, r + 1):
        zt = z.astype(np.float64)
        tail = float(np.linalg.norm(zt[j - 1:]))
        if tail <= happy_tol * float(np.linalg.norm(zt)):
            closed = j - 1
            if j >= 2:
                sg = 1.0 if zt[j - 1] >= 0 else -1.0
                Hc[: j - 1, j - 2] = w[: j - 1]
                Hc[j - 1, j - 2] = -sg * tail
            break
        st = rh_vector(w, z, j, scaling, policy)
        U[:, j - 1] = st.u
        S[:, j - 1] = st.s
        extend_t(T, S, st.s, st.beta, j - 1, hi.type)
        if j == 1:
            beta = -st.sigma * st.rho
        else:
            Hc[: j - 1, j - 2] = w[: j - 1]
            Hc[j - 1, j - 2] = -st.sigma * st.rho
        if j <= m:
            coef = _cast(T[:j, :j], hi) @ _cast(S[j - 1, :j], hi)
            q = -(_cast(U[:, :j], lo) @ _cast(coef, lo)).astype(np.float64)
            q[j - 1] += 1.0
            Q[:, j - 1] = q
            w = round_to(mv(round_to(q, policy.low)), policy.low).astype(np.float64)
            w = apply_reflectors_compact(U[:, :j], S[:, :j], T[:j, :j], w, psi,
                                         transpose_t=True, policy=policy)
            z = psi.apply(w, dtype=lo)
    k = m if closed is None else closed
    nr = r if closed is None else closed
    return Krylov(U[:, :nr], S[:, :nr], T[:nr, :nr], Hc[: k + 1, :k].copy(), psi, beta,
                  scaling, Q[:, :k].copy() if store_q else None, closed)


def hessenberg_lstsq(H, beta, history=False):
    """krylov.py:153-190: Givens QR of the Hessenberg, skip zero subcolumns."""
    R = np.array(H, dtype=np.float64)
    p, k = R.shape
    g = np.zeros(p)
    g[0] = float(beta)
    hist = np.zeros(k + 1)
    hist[0] = abs(float(beta))
    for j in range(k):
        a, t = R[j, j], R[j + 1, j]
        r = float(np.hypot(a, t))
        cs, sn = (1.0, 0.0) if r == 0.0 else (a / r, t / r)
        r1 = R[j, j:k].copy()
        r2 = R[j + 1, j:k].copy()
        R[j, j:k] = cs * r1 + sn * r2
        R[j + 1, j:k] = -sn * r1 + cs * r2
        g[j], g[j + 1] = cs * g[j] + sn * g[j + 1], -sn * g[j] + cs * g[j + 1]
        hist[j + 1] = abs(g[j + 1])
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        if R[i, i] == 0.0:
            continue
        y[i] = (g[i] - R[i, i + 1: k] @ y[i + 1:]) / R[i, i]
    res = float(abs(g[k])) if p > k else 0.0
    return (y, res, hist) if history else (y, res)


def rhqr_gmres(A, b, x0, m, omega, scaling="sqrt2", policy=DOUBLE, happy_tol=None):
    """krylov.py:193-222."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    bun = rhqr_arnoldi(A, b, x0, m, omega, scaling, policy, store_q=False,
                       happy_tol=happy_tol)
    k = bun.dim
    y, _, hist = hessenberg_lstsq(bun.H, bun.beta, history=True)
    if k and np.any(np.diagonal(bun.H)[:k] == 0.0):
        warnings.warn("Hessenberg system is rank deficient; dependent "
                      "coordinates were zeroed", RuntimeWarning)
    bun.y, bun.resid_history = y, hist
    if k == 0:
        return x0.copy(), hist
    pad = np.zeros(n)
    pad[:k] = y
    corr = apply_reflectors_compact(bun.U[:, :k], bun.S[:, :k], bun.T[:k, :k], pad,
                                    bun.psi, policy=policy)
    return x0 + corr, hist


# --------------------------------------------------------------------------
# linalg.py diagnostics, experiments.py generator
# --------------------------------------------------------------------------
def cond_number(M):
    """linalg.py:151-160."""
    A = np.asarray(M, dtype=np.float64)
    if not np.all(np.isfinite(A)):
        return np.inf
    sv = np.linalg.svd(A, compute_uv=False)
    return np.inf if sv[-1] == 0.0 else float(sv[0] / sv[-1])


def orthogonality_error(Q):
    """linalg.py:193-197."""
    Q = np.asarray(Q, dtype=np.float64)
    G = Q.T @ Q
    return float(np.linalg.norm(G - np.eye(G.shape[0])))


def factorization_errors(W, Q, R):
    """linalg.py:169-190 -> (fro_rel_err, max_col_rel_err, flagged)."""
    W, Q, R = (np.asarray(a, dtype=np.float64) for a in (W, Q, R))
    D = W - Q @ R
    wf = np.linalg.norm(W)
    fro = float(np.linalg.norm(D) / wf) if wf else float(np.linalg.norm(D))
    cw = np.linalg.norm(W, axis=0)
    cd = np.linalg.norm(D, axis=0)
    zero = cw == 0.0
    rel = cd / np.where(zero, wf if wf else 1.0, cw)
    return fro, (float(rel.max()) if rel.size else 0.0), tuple(np.nonzero(zero)[0].tolist())


def gen_cmatrix(n, m):
    """experiments.py:86-98 (config 3 input)."""
    if n < 2 or m < 2:
        raise ValueError("need n >= 2 and m >= 2")
    x = np.arange(n) / (n - 1.0)
    mu = np.arange(m) / (m - 1.0)
    return np.sin(10.0 * (mu[None, :] + x[:, None])) / (
        np.cos(100.0 * (mu[None, :] - x[:, None])) + 1.1)


# --------------------------------------------------------------------------
# trim.py (+ sketching.py:216-235): trimmed RHQR, SURVEY §8(f)4
# --------------------------------------------------------------------------
class ColumnScaled:
    """sketching.py:216-235: rescale the m leading input coordinates (in the
    arithmetic dtype), then apply the base operator.  `E` caches the unit
    sketches of the leading columns."""

    kind = "colscaled"

    def __init__(self, base, scales, m, E):
        self.base, self.m = base, int(m)
        self.ell, self.n, self.seed = base.ell, base.n, base.seed
        self.scales = np.asarray(scales, dtype=np.float64)
        self.E = E

    def apply(self, X, dtype=np.float64):
        X, vec = _cols(X, self.n)
        dt = np.dtype(dtype)
        Xs = X.astype(dt) * self.scales[:, None].astype(dt)
        Y = self.base.apply(Xs.astype(np.float64), dtype=dt)
        Y = np.asarray(Y, dtype=np.float64)
        return Y[:, 0] if vec else Y


def srht_unit_columns(omega, m):
    """Omega e_k for k < m in closed form (SRHT only): the FWHT of a one-hot
    vector adds only exact zeros, so entry i is
    sign_k * (-1)^popcount(idx_i & k) * fl(fl(1 * scale) * n_pad^-1/2)
    — bitwise what sketching.py:149-155 computes for I[:, :m]."""
    a = np.float64(np.float64(1.0) * np.float64(omega.scale)) * np.float64(omega.n_pad ** -0.5)
    k = np.arange(m, dtype=np.int64)
    par = np.zeros((omega.ell, m), dtype=np.int64)
    x = omega.indices[:, None] & k[None, :]
    while np.any(x):
        par ^= x & 1
        x >>= 1
    return (np.where(par == 1, -1.0, 1.0) * omega.signs[:m][None, :]) * a


def normalize_leading_columns(omega, m, chunk=256):
    """trim.py:51-77."""
    if isinstance(omega, ColumnScaled) and omega.m >= m:
        return omega
    n = omega.n
    if m > n:
        raise ValueError(f"cannot normalize {m} leading columns of {n} inputs")
    cols = np.empty((omega.ell, m))
    for k0 in range(0, m, chunk):
        k1 = min(k0 + chunk, m)
        eye = np.zeros((n, k1 - k0))
        eye[np.arange(k0, k1), np.arange(k1 - k0)] = 1.0
        cols[:, k0:k1] = omega.apply(eye)
    norms = np.linalg.norm(cols, axis=0)
    if np.any(norms == 0.0):
        raise ValueError(f"leading column {int(np.argmin(norms)) + 1} sketches to zero")
    scales = np.ones(n)
    scales[:m] = 1.0 / norms
    return ColumnScaled(omega, scales, m, cols / norms)


@dataclass
class TrimStep:
    """trim.py:37-48."""

    j: int
    v: np.ndarray
    s: np.ndarray
    sigma: float
    rho: float
    beta: float


def trim_rh_vector(w_tail, omega, j, scaling="sqrt2", policy=DOUBLE):
    """trim.py:80-146: the reflector of the tail w[j-1:], sketched with the
    j-1 leading coordinates zeroed."""
    lo, hi = policy.lo, policy.hi.type
    w_tail = np.asarray(w_tail, dtype=np.float64)
    n, p = omega.n, j - 1
    if not 0 <= p < n:
        raise ValueError(f"elimination index {j} outside {n} coordinates")
    if w_tail.shape[0] != n - p:
        raise ValueError(f"tail has {w_tail.shape[0]} entries, expected {n - p}")
    x = np.zeros(n)
    x[p:] = w_tail
    z = omega.apply(x, dtype=lo)
    zn = float(np.linalg.norm(z))
    rho = float(round_to(zn, policy.high))
    if rho == 0.0:
        raise BreakdownError(f"sketched tail annihilated at column {j}")
    sg = sign(w_tail[0])
    v = w_tail.copy()
    v[0] += sg * rho
    v = round_to(v, policy.low)
    x[p:] = v
    vs = omega.apply(x, dtype=lo)
    nv = float(round_to(np.linalg.norm(vs), policy.high))
    if nv <= 8.0 * policy.u_high * (zn + rho):
        raise BreakdownError(f"sketched reflector vector cancelled at column {j} "
                             f"(degenerate sketch geometry, norm {nv:.3e})")
    beta = float(hi(2.0 / (nv * nv)))
    if scaling == "sqrt2":
        f = float(hi(np.sqrt(beta)))
        v, vs, beta = v * f, vs * f, 1.0
    else:
        piv = float(vs[0])
        if abs(piv) <= 8.0 * policy.u_high * nv:
            raise BreakdownError(f"unit scaling pivot vanished at column {j} (sketched entry {piv:.3e})")
        v, vs = v / piv, vs / piv
        beta = float(hi(beta * piv * piv))
    return TrimStep(j, round_to(v, policy.low), round_to(vs, policy.high), sg, rho, beta)


@dataclass
class TrimFactors:
    """trim.py:149-186."""

    U: np.ndarray
    S: np.ndarray
    T: np.ndarray
    T_tilde: np.ndarray
    R: np.ndarray
    L: np.ndarray
    E: np.ndarray
    omega: ColumnScaled
    scaling: str
    sigmas: np.ndarray
    rhos: np.ndarray
    betas: np.ndarray


def _trim_setup(W, omega, m):
    """trim.py:228-235."""
    W = np.asarray(W, dtype=np.float64)
    if W.ndim != 2:
        raise ValueError("W must be a matrix")
    omega = normalize_leading_columns(omega, m)
    if omega.n != W.shape[0]:
        raise ValueError(f"sketch takes {omega.n} coordinates, W has {W.shape[0]} rows")
    return W, omega


def t_tilde_from_factors(S, E, U, policy=DOUBLE):
    """trim.py:189-208: T~^t = -A^{-1}, A = corr - tril(G, -1) - diag(G)/2."""
    hi = policy.hi
    S = np.asarray(S)
    m = S.shape[1]
    Sh = _cast(S, hi)
    G = (Sh.T @ Sh).astype(np.float64)
    Lt = np.tril((Sh.T @ _cast(np.asarray(E)[:, :m], hi)).astype(np.float64), -1)
    corr = (_cast(Lt, hi) @ _cast(np.asarray(U)[:m], hi)).astype(np.float64)
    A = corr - np.tril(G, -1) - np.diag(np.diagonal(G) / 2.0)
    return -upper_tri_solve(A.T, np.eye(m), policy=policy)


def trim_thin_q(F):
    """trim.py:211-225: Q = [I;0] - U T triu(S^t E)."""
    U = np.asarray(F.U)
    k = U.shape[1]
    M = np.triu(np.asarray(F.S).T @ np.asarray(F.E)[:, :k])
    Q = -U @ (np.asarray(F.T) @ M)
    Q[:k] += np.eye(k)
    return Q


def trim_rhqr_left(W, omega, scaling="sqrt2", policy=DOUBLE):
    """trim.py:272-325: column c is transformed by the reversed compact form
    w -= U T~^t (S^t (Omega w) - L w_head), then reflected from its tail."""
    lo, hi = policy.lo, policy.hi
    n, m = np.asarray(W).shape
    W, omega = _trim_setup(W, omega, m)
    E = omega.E[:, :m].copy()
    Wl = round_to(W, policy.low)
    U = np.zeros((n, m))
    S = np.zeros((omega.ell, m))
    R = np.zeros((m, m))
    T = np.zeros((m, m))
    Tt = np.zeros((m, m))
    L = np.zeros((m, m))
    sg, rh, bt = [], [], []
    for c in range(m):
        w = Wl[:, c].copy()
        if c:
            z = omega.apply(w, dtype=lo)
            h = (_cast(S[:, :c], hi).T @ _cast(z, hi)).astype(np.float64)
            h -= (_cast(L[:c, :c], hi) @ _cast(w[:c], hi)).astype(np.float64)
            coef = (_cast(Tt[:c, :c], hi).T @ _cast(h, hi)).astype(np.float64)
            w = (_cast(w, lo) - _cast(U[:, :c], lo) @ _cast(coef, lo)).astype(np.float64)
        st = trim_rh_vector(w[c:], omega, c + 1, scaling, policy)
        U[c:, c] = st.v
        S[:, c] = st.s
        R[:c, c] = w[:c]
        R[c, c] = -st.sigma * st.rho
        lrow = (_cast(E[:, :c], hi).T @ _cast(st.s, hi)).astype(np.float64)
        L[c, :c] = lrow
        extend_t(T, S, st.s, st.beta, c, hi=hi.type)
        if c:
            g = (_cast(S[:, :c], hi).T @ _cast(st.s, hi)).astype(np.float64)
            g -= (_cast(U[:c, :c], hi).T @ _cast(lrow, hi)).astype(np.float64)
            Tt[:c, c] = (hi.type(-st.beta) * (_cast(Tt[:c, :c], hi) @ _cast(g, hi))).astype(np.float64)
        Tt[c, c] = st.beta
        sg.append(st.sigma)
        rh.append(st.rho)
        bt.append(st.beta)
    return TrimFactors(U, S, T, Tt, R, L, E, omega, scaling, np.array(sg), np.array(rh), np.array(bt))


def trim_rhqr_right(W, omega, scaling="sqrt2", policy=DOUBLE):
    """trim.py:238-269: right-looking, trailing columns updated through the
    masked sketch; T, T~ and L assembled after the sweep."""
    lo, hi = policy.lo, policy.hi
    n, m = np.asarray(W).shape
    W, omega = _trim_setup(W, omega, m)
    Wl = round_to(W, policy.low)
    U = np.zeros((n, m))
    S = np.zeros((omega.ell, m))
    R = np.zeros((m, m))
    sg, rh, bt = [], [], []
    for c in range(m):
        w = Wl[:, c]
        st = trim_rh_vector(w[c:], omega, c + 1, scaling, policy)
        U[c:, c] = st.v
        S[:, c] = st.s
        R[:c, c] = w[:c]
        R[c, c] = -st.sigma * st.rho
        sg.append(st.sigma)
        rh.append(st.rho)
        bt.append(st.beta)
        if c + 1 < m:
            Y = Wl[:, c + 1:]
            masked = Y.copy()
            masked[:c] = 0.0
            X = omega.apply(masked, dtype=lo)
            coef = (hi.type(st.beta) * (_cast(st.s, hi) @ _cast(X, hi))).astype(np.float64)
            Wl[:, c + 1:] = (_cast(Y, lo) - np.outer(_cast(U[:, c], lo), _cast(coef, lo))).astype(np.float64)
    E = omega.E[:, :m].copy()
    T = t_factor_from_sketches(S, policy=policy)
    Tt = t_tilde_from_factors(S, E, U, policy=policy)
    L = np.tril((_cast(S, hi).T @ _cast(E, hi)).astype(np.float64), -1)
    return TrimFactors(U, S, T, Tt, R, L, E, omega, scaling, np.array(sg), np.array(rh), np.array(bt))


def rhqr_left_bytes(N, m, elem_bytes=8):
    """Algorithmic HBM bytes of left-looking RHQR:
    b*N*(m^2 + 5m)/2 — read U[:, :c] and read+write w_c per column, plus the
    single raw-sketch pass over W."""
    return elem_bytes * N * (m * m + 5 * m) / 2.0


__all__ = [n for n in dir() if not n.startswith("_")]
_ = math  # keep math importable for callers that time the oracle
