"""Row-partitioned RHQR across GPUs (one process per GPU).

Partition: rank p of P owns the Omega coordinates
[p n_pad/P, (p+1) n_pad/P) — whole SRHT tiles — and rank 0 additionally the
m identity-block rows.  Each column needs exactly one exchange, an NCCL
all-gather of an (ell + m)-vector; the top log2(P) levels of the SRHT tree are
completed in rank order, so every rank's S, T, R, sigmas, rhos, betas are
bitwise identical to the single-GPU factorization (and to the reference).

    import torch.distributed as dist
    dist.init_process_group("nccl")
    init_comm()                                   # NCCL communicator for the library
    Wl = W[local_rows(N, m, omega, P, p)]         # this rank's rows
    F = rhqr_left_distributed(Wl, omega, m)       # F.U holds the local rows of U
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .devarray import CODES, empty_colmajor, is_device, ld_of, to_device, to_numpy
from .linalg import SCALE_SQRT2, check_scaling, scaling_code
from .precision import DOUBLE_POLICY, require_device_policy
from .rhqr import RHQRFactors, _embed, _out, raise_status
from .sketching import EmbeddedSketch

TILE_LOG = {"double": 12, "single": 13, "half": 13, "bf16": 13}


def omega_span(n_pad: int, nranks: int, tag: str = "double") -> int:
    """Omega coordinates per rank; must be a whole number of SRHT tiles."""
    if nranks < 1 or nranks & (nranks - 1) or nranks > 8:
        raise ValueError("nranks must be a power of two <= 8")
    tile = min(1 << TILE_LOG[tag], n_pad)
    span = n_pad // nranks
    if span < tile or span % tile:
        raise ValueError(f"n_pad={n_pad} too small for {nranks} ranks (needs n_pad/P >= {tile})")
    return span


def local_rows(N: int, m: int, n_pad: int, nranks: int, rank: int, tag: str = "double"):
    """Global row indices of W held by `rank`: identity rows (rank 0) then its
    Omega rows (global row = m + Omega coordinate; padding rows do not exist)."""
    span = omega_span(n_pad, nranks, tag)
    n = N - m
    e0 = rank * span
    e1 = min(n, e0 + span)
    omega_rows = np.arange(m + e0, m + max(e0, e1))
    if rank == 0:
        return np.concatenate([np.arange(m), omega_rows])
    return omega_rows


def init_comm(group=None):
    """Create the library's NCCL communicator over the torch process group."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = [None]
    if rank == 0:
        uid = C.create_string_buffer(128)
        if _lib.lib().sqb_nccl_unique_id(uid, 128) != _lib.SQB_OK:
            raise _lib.SketchQRError("ncclGetUniqueId failed")
        buf[0] = uid.raw
    dist.broadcast_object_list(buf, src=0, group=group)
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_ctx_init_comm(ctx.h, buf[0], world, rank), "sqb_ctx_init_comm")
    return ctx


def rhqr_left_distributed(W_local, omega, m, scaling=SCALE_SQRT2, policy=None, check=True):
    """This rank's part of rhqr_left (rhqr.py:254-267) on the row partition."""
    return _distributed("sqb_rhqr_left_dist", W_local, omega, m, scaling, policy, check)


def rec_rhqr_distributed(W_local, omega, m, scaling=SCALE_SQRT2, policy=None, check=True):
    """This rank's part of rec_rhqr (rhqr.py:368-395) on the row partition:
    one all-gather of the sketch partials, then a local triangular solve."""
    return _distributed("sqb_rec_rhqr_dist", W_local, omega, m, scaling, policy, check)


def _distributed(entry, W_local, omega, m, scaling, policy, check):
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    host = not is_device(W_local)
    tag = policy.low
    mrow = m if rank == 0 else 0
    Wd = to_device(W_local, tag, align_row=mrow)
    rows = Wd.shape[0]
    n_local = rows - mrow
    od = m + omega.ell
    U = empty_colmajor(rows, m, tag, align_row=mrow)
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device="cuda")
    utop = torch.empty(m * m, dtype=torch.float64, device="cuda")
    ctx = _lib.context()
    args = [ctx.h, omega.desc(), scaling_code(scaling), CODES[tag], Wd.data_ptr(), n_local, m, ld_of(Wd),
            U.data_ptr(), ld_of(U), S.data_ptr(), ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R),
            scal.data_ptr(), scal.data_ptr() + 8 * m, scal.data_ptr() + 16 * m]
    if entry == "sqb_rhqr_left_dist":
        args.append(utop.data_ptr())
    ctx.check(getattr(_lib.lib(), entry)(*args), entry)
    if check:
        raise_status(ctx, "rec_rhqr" if entry == "sqb_rec_rhqr_dist" else "rhqr_left_distributed")
    del world
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host),
                       psi=EmbeddedSketch(m, omega),
                       scaling=scaling, sigmas=_out(scal[:m], host), rhos=_out(scal[m:2 * m], host),
                       betas=_out(scal[2 * m:], host))


def rhqr_left_virtual(W, omega, nranks, scaling=SCALE_SQRT2, policy=None):
    """The multi-GPU algorithm with `nranks` virtual ranks on ONE device (the
    all-gather becomes device copies).  Returns factors with U reassembled in
    global row order — bitwise equal to rhqr_left by construction."""
    return _virtual("sqb_rhqr_left_virtual", W, omega, nranks, scaling, policy)


def rec_rhqr_virtual(W, omega, nranks, scaling=SCALE_SQRT2, policy=None):
    """Row-partitioned rec_rhqr with `nranks` virtual ranks on one device."""
    return _virtual("sqb_rec_rhqr_virtual", W, omega, nranks, scaling, policy)


def _virtual(entry, W, omega, nranks, scaling, policy):
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    host = not is_device(W)
    tag = policy.low
    N, m = tuple(W.shape) if is_device(W) else np.shape(W)
    psi = _embed(omega, N, m)
    parts, Us, rows_list = [], [], []
    for p in range(nranks):
        rows = local_rows(N, m, omega.n_pad, nranks, p, tag)
        rows_list.append(rows)
        src = W[torch.as_tensor(rows, device=W.device)] if is_device(W) else np.asarray(W)[rows]
        mrow = m if p == 0 else 0
        parts.append(to_device(src, tag, align_row=mrow) if len(rows) else empty_colmajor(0, m, tag))
        Us.append(empty_colmajor(max(len(rows), 1), m, tag, align_row=mrow))
    od = psi.out_dim
    S = empty_colmajor(od, m, "double")
    T = empty_colmajor(m, m, "double")
    R = empty_colmajor(m, m, "double")
    scal = torch.empty(3 * m, dtype=torch.float64, device="cuda")
    scratch = torch.empty(max(1, (nranks - 1) * (od * m + 3 * m * m + 3 * m)), dtype=torch.float64, device="cuda")
    Wp = (C.c_void_p * nranks)(*[t.data_ptr() for t in parts])
    Wl = (C.c_int64 * nranks)(*[ld_of(t) for t in parts])
    Up = (C.c_void_p * nranks)(*[t.data_ptr() for t in Us])
    Ul = (C.c_int64 * nranks)(*[ld_of(t) for t in Us])
    ctx = _lib.context()
    ctx.check(getattr(_lib.lib(), entry)(
        ctx.h, omega.desc(), scaling_code(scaling), CODES[tag], nranks, Wp, Wl, Up, Ul, m, S.data_ptr(),
        ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R), scal.data_ptr(), scal.data_ptr() + 8 * m,
        scal.data_ptr() + 16 * m, scratch.data_ptr()), entry)
    raise_status(ctx, "rec_rhqr" if entry == "sqb_rec_rhqr_virtual" else "rhqr_left_virtual")
    U = empty_colmajor(N, m, tag)
    for rows, Ut in zip(rows_list, Us):
        if len(rows):
            U[torch.as_tensor(rows, device=U.device)] = Ut[: len(rows)]
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host), psi=psi,
                       scaling=scaling, sigmas=_out(scal[:m], host), rhos=_out(scal[m:2 * m], host),
                       betas=_out(scal[2 * m:], host))


_ = to_numpy
