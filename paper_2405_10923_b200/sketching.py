"""Sketch operators (mirror of sketching.py): the operator state is generated
on the host with exactly the reference's numpy calls (so signs, indices and
Gaussian entries are bit-identical for the same seed) and kept resident on
the device; `apply` runs the sm_100a kernels (K1 SRHT, bit-exact; K2 DMMA
dense GEMM).

Array convention of the whole package: numpy in -> numpy out (the
reference's float64 ndarrays), torch CUDA tensors in -> torch CUDA tensors
out (device-resident fast path).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib
from .devarray import CODES, require_cuda, empty_colmajor, is_device, ld_of, to_device, to_numpy, tag_of_torch
from .precision import DOUBLE_POLICY, tag_of_dtype


def _columns(X, n):
    """sketching.py:46-53: 1-D -> column, row-count check (ValueError)."""
    if is_device(X):
        vec = X.dim() == 1
        X2 = X[:, None] if vec else X
    else:
        X2 = np.asarray(X, dtype=np.float64)
        vec = X2.ndim == 1
        if vec:
            X2 = X2[:, None]
    if X2.shape[0] != n:
        raise ValueError(f"operand has {X2.shape[0]} rows, operator expects {n}")
    return X2, vec


def _dtype_tag(dtype) -> str:
    return tag_of_dtype(np.dtype(dtype))


def _device_input(X2, tag, align_row=0):
    """Sketch input in the arithmetic dtype: X.astype(dtype) (sketching.py:152).
    Host arrays are cast with numpy (no range check, like astype)."""
    require_cuda()
    if is_device(X2):
        return to_device(X2, tag, align_row)
    with np.errstate(over="ignore"):
        A = np.asarray(X2, dtype=np.float64).astype(np.dtype(_np_dtype(tag)))
    if tag == "bf16":
        src = torch.from_numpy(np.ascontiguousarray(A).view(np.int16)).view(torch.bfloat16)
    else:
        src = torch.from_numpy(np.ascontiguousarray(A))
    out = empty_colmajor(A.shape[0], A.shape[1], tag, align_row)
    out.copy_(src.cuda())
    return out


def _np_dtype(tag):
    from .precision import DTYPES

    return DTYPES[tag]


class SketchOperator:
    """sketching.py:56-79: seeded linear map R^n -> R^ell, applied columnwise."""

    kind = None

    def __init__(self, ell, n, seed):
        if ell < 1 or n < 1:
            raise ValueError(f"invalid sketch dimensions {ell} x {n}")
        self.ell = int(ell)
        self.n = int(n)
        self.seed = int(seed)
        self._dev = {}

    @property
    def shape(self):
        return (self.ell, self.n)

    # -- device side -------------------------------------------------------
    def _device_state(self):
        raise NotImplementedError

    def desc(self) -> _lib.SketchDesc:
        """sqb_sketch descriptor for the current CUDA device."""
        dev = torch.cuda.current_device()
        st = self._dev.get(dev)
        if st is None:
            st = self._dev[dev] = self._device_state()
        return st["desc"]

    def apply(self, X, dtype=np.float64):
        """sketching.py:72-76: returns ell x k float64 (ell for a vector)."""
        X2, vec = _columns(X, self.n)
        tag = _dtype_tag(dtype)
        Xd = _device_input(X2, tag)
        k = Xd.shape[1]
        Y = empty_colmajor(self.ell, k, "double")
        ctx = _lib.context()
        d = self.desc()
        ctx.check(_lib.lib().sqb_sketch_apply(ctx.h, d, CODES[tag], Xd.data_ptr(), ld_of(Xd), k,
                                              Y.data_ptr(), ld_of(Y)), "sqb_sketch_apply")
        out = Y[:, 0] if vec else Y
        return out if is_device(X) else to_numpy(out)


class SRHTSketch(SketchOperator):
    """sketching.py:128-155: sqrt(n_pad/ell) * (row subset) * H * diag(signs),
    zero padded to n_pad.  Memory O(n_pad + ell) on the device: one sign BIT
    per coordinate and the ell ordered indices."""

    kind = "srht"

    def __init__(self, ell, n, seed):
        super().__init__(ell, n, seed)
        self.n_pad = 1 << (self.n - 1).bit_length()
        if self.ell > self.n_pad:
            raise ValueError(f"ell={ell} exceeds padded length {self.n_pad}")
        # the reference's exact RNG calls (sketching.py:144-147)
        rng = np.random.Generator(np.random.Philox(key=[self.seed, (1 << 40) + 1]))
        self.signs = (rng.integers(0, 2, self.n_pad) * 2 - 1).astype(np.float64)
        self.indices = rng.permutation(self.n_pad)[: self.ell].copy()
        self.scale = float(np.sqrt(self.n_pad / self.ell))

    def sign_bits(self) -> np.ndarray:
        """Packed sign bits (little-endian bit order, bit set <=> -1) as uint32."""
        b = np.packbits(self.signs < 0, bitorder="little")
        pad = (-b.shape[0]) % 4
        if pad:
            b = np.concatenate([b, np.zeros(pad, np.uint8)])
        return b.view(np.uint32)

    def _device_state(self):
        bits = torch.from_numpy(self.sign_bits().view(np.int32).copy()).cuda()
        idx = torch.from_numpy(self.indices.astype(np.int64)).cuda()
        d = _lib.SketchDesc(kind=_lib.SQB_SKETCH_SRHT, ell=self.ell, n=self.n, n_pad=self.n_pad,
                            scale=self.scale, sign_bits=bits.data_ptr(), indices=idx.data_ptr())
        return {"desc": d, "bits": bits, "idx": idx}


class _FullHadamard(SRHTSketch):
    """The SRHT with all signs +1, every row kept in order and scale 1: its
    apply IS the normalized Walsh-Hadamard transform (the K1 kernels, same
    butterfly order and rounding as fwht, sketching.py:21-43)."""

    def __init__(self, n):
        SketchOperator.__init__(self, n, n, 0)
        self.n_pad = n
        self.signs = np.ones(n)
        self.indices = np.arange(n, dtype=np.int64)
        self.scale = 1.0


_hadamard_ops = {}


def fwht(x):
    """sketching.py:21-43: normalized fast Walsh-Hadamard transform along axis 0
    in x's own dtype (float64, float32, float16 or a CUDA tensor), on the
    device through the SRHT kernels."""
    dev = is_device(x)
    a = x if dev else np.asarray(x)
    n = a.shape[0] if a.ndim else 0
    if n == 0 or n & (n - 1):
        raise ValueError(f"length {n} is not a power of two")
    if dev:
        dt = None
        tag = tag_of_torch(a.dtype)
    else:
        if a.dtype.kind != "f":
            a = a.astype(np.float64)
        dt = a.dtype
        try:
            tag = tag_of_dtype(dt)
        except ValueError:
            raise TypeError(f"fwht on the device supports float64/float32/float16, not {dt}") from None
    if n == 1:
        return a.clone() if dev else a.copy()
    if n > 1 << 18:  # every row is kept: the leaf table grows as n^2 / tile
        raise ValueError("the device fwht is a validation utility (n <= 2^18); SRHTSketch.apply is the transform")
    op = _hadamard_ops.get(n)
    if op is None:
        if len(_hadamard_ops) > 8:
            _hadamard_ops.clear()
        op = _hadamard_ops[n] = _FullHadamard(n)
    shape = a.shape
    a2 = a.reshape(n, -1)
    y = op.apply(a2 if dev else a2.astype(np.float64), dtype=_np_dtype(tag))
    y = y.reshape(shape)
    return y.to(a.dtype) if dev else y.astype(dt)


def check_embedding(op, Q, orth_tol=1e-12):
    """sketching.py:286-298: max(sigma_max - 1, 1 - sigma_min) of op applied to
    a float64-orthonormal basis Q (ValueError if Q is not orthonormal)."""
    from .linalg import orthogonality_error
    err = orthogonality_error(Q)
    if err > orth_tol:
        raise ValueError(f"basis is not orthonormal: ||Q^tQ - I|| = {err:.3e}")
    Y = op.apply(Q)
    sv = torch.linalg.svdvals(Y if is_device(Y) else torch.from_numpy(np.ascontiguousarray(Y)).cuda())
    return float(max(float(sv[0]) - 1.0, 1.0 - float(sv[-1])))


def _philox_rows(seed, n, i0, i1, out, scale):
    for i in range(i0, i1):
        g = np.random.Generator(np.random.Philox(key=[seed, i]))
        g.standard_normal(n, out=out[i])
        out[i] *= scale


class GaussianSketch(SketchOperator):
    """sketching.py:82-125: dense N(0, 1/ell), row i from Philox(key=[seed, i]).

    The reference caches G only when ell*n <= 2^23 and otherwise regenerates
    it in row blocks on every apply; here G is generated once on the host
    (rows in parallel — they are independent streams, so the matrix is
    identical) and kept resident in HBM, where the DMMA GEMM reads it."""

    kind = "gauss"
    _CACHE_ENTRIES = 1 << 23

    def __init__(self, ell, n, seed, threads=None):
        super().__init__(ell, n, seed)
        self._threads = threads or min(32, os.cpu_count() or 1)
        self._cache = {}

    def matrix(self) -> np.ndarray:
        G = self._cache.get(np.dtype(np.float64))
        if G is None:
            G = np.empty((self.ell, self.n))
            c = self.ell ** -0.5
            t = max(1, min(self._threads, self.ell))
            bounds = np.linspace(0, self.ell, t + 1).astype(int)
            with ThreadPoolExecutor(t) as ex:
                list(ex.map(lambda a: _philox_rows(self.seed, self.n, a[0], a[1], G, c),
                            zip(bounds[:-1], bounds[1:])))
            self._cache[np.dtype(np.float64)] = G
        return G

    def _device_state(self):
        G = torch.from_numpy(self.matrix()).cuda()
        d = _lib.SketchDesc(kind=_lib.SQB_SKETCH_DENSE, ell=self.ell, n=self.n, G=G.data_ptr(),
                            ldg=G.stride(0))
        return {"desc": d, "G": G}

    def desc(self):
        # the reference test suite clears _cache to force regeneration; drop the
        # device copy with it so both views stay consistent
        if not self._cache:
            self._dev.clear()
        return super().desc()


class MatrixSketch(SketchOperator):
    """sketching.py:198-213: an explicit ell x n matrix through the operator API."""

    kind = "matrix"

    def __init__(self, matrix):
        matrix = np.asarray(matrix, dtype=np.float64)
        if matrix.ndim != 2:
            raise ValueError("sketch matrix must be two dimensional")
        super().__init__(matrix.shape[0], matrix.shape[1], 0)
        self.matrix = matrix

    def _device_state(self):
        G = torch.from_numpy(np.ascontiguousarray(self.matrix)).cuda()
        d = _lib.SketchDesc(kind=_lib.SQB_SKETCH_DENSE, ell=self.ell, n=self.n, G=G.data_ptr(),
                            ldg=G.stride(0))
        return {"desc": d, "G": G}


class IdentitySketch(SketchOperator):
    """sketching.py:186-195: ell = n pass-through (test oracle operator)."""

    kind = "identity"

    def __init__(self, n):
        super().__init__(n, n, 0)

    def _device_state(self):
        d = _lib.SketchDesc(kind=_lib.SQB_SKETCH_IDENTITY, ell=self.ell, n=self.n)
        return {"desc": d}


class EmbeddedSketch:
    """sketching.py:238-260: Psi = [I_m; Omega]; the top block is a bitwise copy."""

    def __init__(self, m, omega):
        self.m = int(m)
        self.omega = omega
        self.n = self.m + omega.n
        self.out_dim = self.m + omega.ell

    @property
    def shape(self):
        return (self.out_dim, self.n)

    def apply(self, X, dtype=np.float64):
        X2, vec = _columns(X, self.n)
        tag = _dtype_tag(dtype)
        same = is_device(X2) and tag_of_torch(X2.dtype) == tag
        if tag != "double" and not same:
            # sketching.py:257-259: the top block is a bitwise copy of the float64
            # operand; only the Omega part is cast to the arithmetic dtype
            bottom = self.omega.apply(X2[self.m:], dtype=dtype)
            if is_device(X2):
                Y = torch.cat([X2[: self.m].to(torch.float64), bottom], dim=0)
            else:
                Y = np.concatenate([np.asarray(X2[: self.m], dtype=np.float64), bottom], axis=0)
            return Y[:, 0] if vec else Y
        Xd = _device_input(X2, tag, align_row=self.m)
        k = Xd.shape[1]
        Y = empty_colmajor(self.out_dim, k, "double")
        ctx = _lib.context()
        ctx.check(_lib.lib().sqb_embedded_apply(ctx.h, self.omega.desc(), self.m, CODES[tag],
                                                Xd.data_ptr(), ld_of(Xd), k, Y.data_ptr(), ld_of(Y)),
                  "sqb_embedded_apply")
        out = Y[:, 0] if vec else Y
        return out if is_device(X) else to_numpy(out)


def make_sketch(kind, ell, n, seed, s=8):
    """sketching.py:263-271."""
    if kind in ("gauss", "gaussian"):
        return GaussianSketch(ell, n, seed)
    if kind == "srht":
        return SRHTSketch(ell, n, seed)
    if kind in ("sparse", "sparse_sign"):
        raise NotImplementedError("sparse-sign sketches are outside the B200 hot path (SURVEY §2 #4)")
    raise ValueError(f"unknown sketch kind {kind!r}")


def apply_sketch(omega, X, policy=None):
    """sketching.py:274-277."""
    policy = policy or DOUBLE_POLICY
    return omega.apply(X, dtype=policy.low_dtype)


def apply_psi(psi, X, policy=None):
    """sketching.py:280-283."""
    policy = policy or DOUBLE_POLICY
    return psi.apply(X, dtype=policy.low_dtype)
