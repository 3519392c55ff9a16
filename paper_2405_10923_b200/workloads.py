"""Seeded synthetic inputs for the BASELINE configs.

These are host-side input generators, exactly as in the reference
(`experiments.py:86-98` builds config 3's W with numpy in double); they are
not part of the factorization.  Device sin/cos would differ from glibc by an
ulp, so W is always generated on the host and uploaded.

Config 5's convection-diffusion operator is not in the reference
(SPEC.md:546, :552); it is a build-side definition documented in DESIGN.md.
"""

from __future__ import annotations

import hashlib

import numpy as np


def sha256(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gen_cmatrix(n: int, m: int) -> np.ndarray:
    """experiments.py:86-98: W_ij = sin(10(mu_j + x_i)) / (cos(100(mu_j - x_i)) + 1.1),
    x = i/(n-1), mu = j/(m-1), evaluated in double."""
    if n < 2 or m < 2:
        raise ValueError("need n >= 2 and m >= 2")
    x = np.arange(n) / (n - 1.0)
    mu = np.arange(m) / (m - 1.0)
    num = np.sin(10.0 * (mu[None, :] + x[:, None]))
    den = np.cos(100.0 * (mu[None, :] - x[:, None])) + 1.1
    return num / den


def gaussian_w(n: int, m: int, seed: int) -> np.ndarray:
    """Config 1: i.i.d. N(0,1) entries."""
    return np.random.default_rng(seed).standard_normal((n, m))


def illcond_w(n: int, m: int, seed: int, smin_exp: float = -15.0) -> np.ndarray:
    """Config 2: W = A diag(sigma) B with A (n x m), B (m x m) orthonormalised
    Gaussians and sigma log-spaced from 1 to 10^smin_exp."""
    g = np.random.default_rng(seed)
    A = np.linalg.qr(g.standard_normal((n, m)))[0]
    B = np.linalg.qr(g.standard_normal((m, m)))[0]
    return A @ np.diag(np.logspace(0, smin_exp, m)) @ B


def scaled_gaussian_w(n: int, m: int, seed: int, smin_exp: float = -8.0) -> np.ndarray:
    """Config 4: N(0,1) with column scales log-spaced 1 .. 10^smin_exp."""
    return np.random.default_rng(seed).standard_normal((n, m)) * np.logspace(0, smin_exp, m)[None, :]


def convection_diffusion_csr(k: int, vel=(50.0, 50.0)):
    """Config 5: -Laplace(u) + v . grad(u) on the unit square, k x k interior
    grid, h = 1/(k+1), central differences, Dirichlet boundary.  Returns CSR
    arrays (indptr int64, indices int32, data float64) in natural row order
    (row r = i*k + j).  Per row the entries are sorted by column."""
    h = 1.0 / (k + 1)
    vx, vy = vel
    c = 4.0 / (h * h)
    west = -1.0 / (h * h) - vx / (2.0 * h)
    east = -1.0 / (h * h) + vx / (2.0 * h)
    south = -1.0 / (h * h) - vy / (2.0 * h)
    north = -1.0 / (h * h) + vy / (2.0 * h)
    N = k * k
    ii, jj = np.divmod(np.arange(N, dtype=np.int64), k)
    cols, vals, rows = [], [], []
    # column order within a row: r-k, r-1, r, r+1, r+k (sorted)
    for di, dj, v in ((-1, 0, south), (0, -1, west), (0, 0, c), (0, 1, east), (1, 0, north)):
        ok = (ii + di >= 0) & (ii + di < k) & (jj + dj >= 0) & (jj + dj < k)
        r = np.nonzero(ok)[0]
        rows.append(r)
        cols.append(r + di * k + dj)
        vals.append(np.full(r.shape[0], v))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    indptr = np.zeros(N + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    return indptr, cols.astype(np.int32), vals.astype(np.float64)


def rhqr_left_bytes(N: int, m: int, elem_bytes: int = 8) -> float:
    """Algorithmic HBM bytes of one left-looking RHQR:
    b*N*(m^2 + 5m)/2 = per column c read U[:, :c], read + write w_c, plus one
    raw-sketch pass over W."""
    return elem_bytes * N * (m * m + 5 * m) / 2.0
