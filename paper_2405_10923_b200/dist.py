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


def p2p_slot_count(m: int, ell: int) -> int:
    """Doubles per mailbox slot: the raw-sketch exchange moves m (m + ell)."""
    return m * (m + ell)


def init_p2p(m: int, ell: int, group=None):
    """In-kernel peer-memory exchange (sqb_p2p_*): allocate this rank's mailbox,
    all-gather the CUDA IPC handles over the torch process group and map every
    peer's mailbox.  The row-partitioned factorizations then store their
    per-column partials straight into the peers' memory (no NCCL launch on the
    per-column path).  Needs peer access between the GPUs (NVLink/NVSwitch)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = _lib.context()
    # every step that can fail locally is followed by a collective on its
    # outcome, so a failure on one rank raises on all of them instead of
    # leaving the others inside a collective
    h = C.create_string_buffer(64)
    err = None
    try:
        ctx.check(_lib.lib().sqb_p2p_mailbox(ctx.h, world, p2p_slot_count(m, ell), h), "sqb_p2p_mailbox")
    except Exception as exc:  # noqa: BLE001
        err = repr(exc)
    handles = [None] * world
    dist.all_gather_object(handles, None if err else h.raw, group=group)
    if any(x is None for x in handles):
        close_p2p()
        raise RuntimeError(f"peer-memory mailbox allocation failed on a rank ({err or 'another rank'})")
    table = C.create_string_buffer(b"".join(handles), 64 * world)
    try:
        ctx.check(_lib.lib().sqb_p2p_open(ctx.h, rank, table), "sqb_p2p_open")
    except Exception as exc:  # noqa: BLE001
        err = repr(exc)
    oks = [None] * world
    dist.all_gather_object(oks, err is None, group=group)
    if not all(oks):
        close_p2p()
        raise RuntimeError(f"peer-memory mailboxes could not be mapped on a rank ({err or 'another rank'})")
    return ctx


def set_p2p_timeout(ms: int):
    """Bound the in-kernel wait for a peer's flag (default 20 s): past it the
    call fails with SketchQRError naming the silent rank instead of hanging."""
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_p2p_set_timeout_ms(ctx.h, int(ms)), "sqb_p2p_set_timeout_ms")


def close_p2p():
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_p2p_close(ctx.h), "sqb_p2p_close")


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


def rhqr_left_virtual(W, omega, nranks, scaling=SCALE_SQRT2, policy=None, exchange="copy"):
    """The multi-GPU algorithm with `nranks` virtual ranks on ONE device (the
    all-gather becomes device copies, or with exchange="p2p" the peer-memory
    mailboxes of sqb_p2p_*).  Returns factors with U reassembled in global row
    order — bitwise equal to rhqr_left by construction."""
    return _virtual("sqb_rhqr_left_virtual", W, omega, nranks, scaling, policy, exchange)


def rec_rhqr_virtual(W, omega, nranks, scaling=SCALE_SQRT2, policy=None, exchange="copy"):
    """Row-partitioned rec_rhqr with `nranks` virtual ranks on one device."""
    return _virtual("sqb_rec_rhqr_virtual", W, omega, nranks, scaling, policy, exchange)


def _virtual(entry, W, omega, nranks, scaling, policy, exchange="copy"):
    if exchange not in ("copy", "p2p"):
        raise ValueError(f"unknown exchange {exchange!r}")
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
    if exchange == "p2p":
        ctx.check(_lib.lib().sqb_p2p_virtual(ctx.h, nranks, p2p_slot_count(m, omega.ell)), "sqb_p2p_virtual")
    try:
        ctx.check(getattr(_lib.lib(), entry)(
            ctx.h, omega.desc(), scaling_code(scaling), CODES[tag], nranks, Wp, Wl, Up, Ul, m, S.data_ptr(),
            ld_of(S), T.data_ptr(), ld_of(T), R.data_ptr(), ld_of(R), scal.data_ptr(), scal.data_ptr() + 8 * m,
            scal.data_ptr() + 16 * m, scratch.data_ptr()), entry)
        raise_status(ctx, "rec_rhqr" if entry == "sqb_rec_rhqr_virtual" else "rhqr_left_virtual")
    finally:
        if exchange == "p2p":
            ctx.check(_lib.lib().sqb_p2p_close(ctx.h), "sqb_p2p_close")
    U = empty_colmajor(N, m, tag)
    for rows, Ut in zip(rows_list, Us):
        if len(rows):
            U[torch.as_tensor(rows, device=U.device)] = Ut[: len(rows)]
    return RHQRFactors(U=_out(U, host), S=_out(S, host), T=_out(T, host), R=_out(R, host), psi=psi,
                       scaling=scaling, sigmas=_out(scal[:m], host), rhos=_out(scal[m:2 * m], host),
                       betas=_out(scal[2 * m:], host))


_ = to_numpy


# ---------------------------------------------------------------- RHQR-Arnoldi / GMRES
def krylov_partition(n: int, m: int, n_pad: int, nranks: int, tag: str = "double"):
    """Row ranges of the row-partitioned Arnoldi: rank 0 owns the m+1
    identity-block rows and its Omega coordinates, rank p > 0 the Omega
    coordinates [p span, (p+1) span) — each a contiguous range [row0, row0+rows).
    Returns (row0s, rows, seg) with seg = the per-rank slot of the gathered
    vectors (m+1+span)."""
    mt = m + 1
    span = omega_span(n_pad, nranks, tag)
    row0s, rows = [], []
    for p in range(nranks):
        r = local_rows(n, mt, n_pad, nranks, p, tag)
        row0s.append(int(r[0]) if len(r) else n)
        rows.append(len(r))
    return row0s, rows, mt + span


def _gather_positions(cols: np.ndarray, m: int, span: int, seg: int) -> np.ndarray:
    """Global vector index -> position in the gathered [rank][seg] layout."""
    mt = m + 1
    cols = np.asarray(cols, dtype=np.int64)
    e = cols - mt
    q = np.where(cols < mt + span, 0, e // span)
    local = np.where(q == 0, cols, e - q * span)
    return q * seg + local


def local_operator_host(A, m: int, n_pad: int, nranks: int, rank: int, tag: str = "double"):
    """This rank's CSR rows of a global scipy sparse A with the column
    indices remapped to the gathered layout (host arrays): (indptr int64,
    indices int32, data float64, row0, rows, seg)."""
    import scipy.sparse
    A = scipy.sparse.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    row0s, rows, seg = krylov_partition(n, m, n_pad, nranks, tag)
    r0, nr = row0s[rank], rows[rank]
    B = A[r0:r0 + nr]
    span = omega_span(n_pad, nranks, tag)
    idx = _gather_positions(B.indices, m, span, seg).astype(np.int32)
    return B.indptr.astype(np.int64), idx, B.data.astype(np.float64), r0, nr, seg


def gather_layout(x, m: int, n_pad: int, nranks: int, tag: str = "double"):
    """A global vector in the gathered [rank][seg] layout (what the per-step
    all-gather of q produces on every rank)."""
    n = len(x)
    row0s, rows, seg = krylov_partition(n, m, n_pad, nranks, tag)
    out = np.zeros(nranks * seg, dtype=np.asarray(x).dtype)
    for p in range(nranks):
        out[p * seg:p * seg + rows[p]] = x[row0s[p]:row0s[p] + rows[p]]
    return out


def halo_ranges(indices, seg: int, nranks: int, rank: int):
    """[lo, hi) of every rank's segment that this rank's remapped CSR column
    indices reference (its own segment: (0, 0), it is copied locally) — the
    halo of the row-partitioned SpMV; for the 5-point stencil
    one grid row at the end of the previous rank and the start of the next."""
    idx = np.asarray(indices, dtype=np.int64)
    out = np.zeros((nranks, 2), dtype=np.int64)
    if idx.size:
        owner = idx // seg
        for p in range(nranks):
            if p == rank:
                continue
            sel = idx[owner == p]
            if sel.size:
                out[p] = (int(sel.min()) - p * seg, int(sel.max()) - p * seg + 1)
    return out


def set_halo(table):
    """Install a [P][P][2] halo table on the library context (None clears)."""
    ctx = _lib.context()
    if table is None:
        ctx.check(_lib.lib().sqb_ctx_set_halo(ctx.h, 0, None), "sqb_ctx_set_halo")
        return
    t = np.ascontiguousarray(np.asarray(table, dtype=np.int64))
    ctx.check(_lib.lib().sqb_ctx_set_halo(ctx.h, int(t.shape[0]), t.ctypes.data), "sqb_ctx_set_halo")


def local_operator(A, m: int, n_pad: int, nranks: int, rank: int, tag: str = "double"):
    """local_operator_host, uploaded (what sqb_rhqr_arnoldi_dist expects)."""
    ip, ix, dv, r0, nr, seg = local_operator_host(A, m, n_pad, nranks, rank, tag)
    return (torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), torch.from_numpy(dv).cuda(), r0, nr, seg)


def _arnoldi_bufs(rows, mrow, m, od, tag, x0_local):
    mt = m + 1
    # U is streamed from local row 0 by the GEMVs (16-byte aligned there)
    return dict(U=empty_colmajor(max(rows, 1), mt, tag), S=empty_colmajor(od, mt, "double"),
                T=empty_colmajor(mt, mt, "double"), H=empty_colmajor(mt, m, "double"),
                beta=torch.zeros(1, dtype=torch.float64, device="cuda"),
                Utop=empty_colmajor(mt, mt, tag), x0=to_device(x0_local, tag))


def rhqr_arnoldi_virtual(A, b, x0, m, omega, nranks, scaling=SCALE_SQRT2, policy=None, happy_tol=None,
                         halo=True):
    """The row-partitioned RHQR-Arnoldi with `nranks` virtual ranks on one
    device; returns rank 0's sketch-space factors (bitwise those of one GPU)
    and U reassembled in global row order.  halo=True exchanges only the
    entries of q each rank's rows reference (each rank gets its own gathered
    buffer, so a wrong range changes the result); False all-gathers q."""
    from .krylov import KrylovBundle
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    tag = policy.low
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    mt = m + 1
    psi = _embed(omega, n, mt)
    od = psi.out_dim
    happy_tol = 32.0 * policy.u_high if happy_tol is None else happy_tol
    row0s, rows, seg = krylov_partition(n, m, omega.n_pad, nranks, tag)
    keep, bufs = [], []
    table = np.zeros((nranks, nranks, 2), dtype=np.int64)
    for p in range(nranks):
        ip, ix, dv, r0, nr, _ = local_operator(A, m, omega.n_pad, nranks, p, tag)
        table[p] = halo_ranges(ix.cpu().numpy(), seg, nranks, p)
        bl = torch.from_numpy(b[r0:r0 + nr].copy()).cuda() if nr else torch.zeros(1, dtype=torch.float64, device="cuda")
        bf = _arnoldi_bufs(nr, mt if p == 0 else 0, m, od, tag, x0[r0:r0 + nr] if nr else np.zeros(1))
        keep += [ip, ix, dv, bl]
        bufs.append((ip, ix, dv, bl, bf))
    P_ = nranks
    arr = lambda ctype, xs: (ctype * P_)(*xs)  # noqa: E731
    attained = C.c_int(-1)
    ctx = _lib.context()
    set_halo(table if halo else None)
    try:
        rc = _lib.lib().sqb_rhqr_arnoldi_virtual(
        ctx.h, omega.desc(), m, scaling_code(scaling), CODES[tag], float(happy_tol), P_,
        arr(C.c_int64, rows), arr(C.c_int64, row0s), seg,
        arr(C.c_void_p, [x[0].data_ptr() for x in bufs]), arr(C.c_void_p, [x[1].data_ptr() for x in bufs]),
        arr(C.c_void_p, [x[2].data_ptr() for x in bufs]), arr(C.c_void_p, [x[3].data_ptr() for x in bufs]),
        arr(C.c_void_p, [x[4]["x0"].data_ptr() for x in bufs]), arr(C.c_void_p, [x[4]["U"].data_ptr() for x in bufs]),
        arr(C.c_int64, [ld_of(x[4]["U"]) for x in bufs]), arr(C.c_void_p, [x[4]["S"].data_ptr() for x in bufs]),
        ld_of(bufs[0][4]["S"]), arr(C.c_void_p, [x[4]["T"].data_ptr() for x in bufs]), ld_of(bufs[0][4]["T"]),
        arr(C.c_void_p, [x[4]["H"].data_ptr() for x in bufs]), ld_of(bufs[0][4]["H"]),
        arr(C.c_void_p, [x[4]["beta"].data_ptr() for x in bufs]),
        arr(C.c_void_p, [x[4]["Utop"].data_ptr() for x in bufs]), C.byref(attained))
    finally:
        set_halo(None)
    ctx.check(rc, "sqb_rhqr_arnoldi_virtual")
    raise_status(ctx, "rhqr_arnoldi")
    closed = None if attained.value < 0 else attained.value
    k = m if closed is None else closed
    r = mt if closed is None else closed
    U = empty_colmajor(n, mt, tag)
    for p, (_, _, _, _, bf) in enumerate(bufs):
        if rows[p]:
            U[row0s[p]:row0s[p] + rows[p]] = bf["U"][: rows[p]]
    b0 = bufs[0][4]
    return KrylovBundle(U=to_numpy(U[:, :r]), S=to_numpy(b0["S"][:, :r]), T=to_numpy(b0["T"][:r, :r]),
                        H=to_numpy(b0["H"][: k + 1, :k]), psi=psi, beta=float(b0["beta"].item()), scaling=scaling,
                        Q_cols=None, breakdown=closed)


def rhqr_arnoldi_distributed(A_local, b_local, x0_local, m, omega, n, scaling=SCALE_SQRT2, policy=None,
                             happy_tol=None, halo=True):
    """This rank's part of rhqr_arnoldi (krylov.py:82-150) on the row
    partition (one process per GPU, NCCL).  A_local = local_operator(...)
    output; b_local / x0_local are this rank's rows.  Returns a KrylovBundle
    whose U holds the local rows; S, T, H, beta are replicated."""
    import torch.distributed as dist
    from .krylov import KrylovBundle
    check_scaling(scaling)
    policy = policy or DOUBLE_POLICY
    require_device_policy(policy)
    tag = policy.low
    rank = dist.get_rank()
    ip, ix, dv, r0, nr, seg = A_local
    mt = m + 1
    psi = _embed(omega, n, mt)
    od = psi.out_dim
    happy_tol = 32.0 * policy.u_high if happy_tol is None else happy_tol
    bl = to_device(b_local, "double")[:, 0]
    bf = _arnoldi_bufs(nr, mt if rank == 0 else 0, m, od, tag,
                       x0_local if x0_local is not None else np.zeros(max(nr, 1)))
    attained = C.c_int(-1)
    ctx = _lib.context()
    table = None
    if halo:  # every rank's halo ranges, gathered once (host, tiny)
        mine = halo_ranges(ix.cpu().numpy(), seg, dist.get_world_size(), rank)
        rows_all = [None] * dist.get_world_size()
        dist.all_gather_object(rows_all, mine.tolist())
        table = np.asarray(rows_all, dtype=np.int64)
    set_halo(table)
    try:
        rc = _lib.lib().sqb_rhqr_arnoldi_dist(
        ctx.h, omega.desc(), m, scaling_code(scaling), CODES[tag], float(happy_tol), nr, r0, seg, ip.data_ptr(),
        ix.data_ptr(), dv.data_ptr(), bl.data_ptr(), bf["x0"].data_ptr(), bf["U"].data_ptr(), ld_of(bf["U"]),
        bf["S"].data_ptr(), ld_of(bf["S"]), bf["T"].data_ptr(), ld_of(bf["T"]), bf["H"].data_ptr(), ld_of(bf["H"]),
        None, 1, bf["beta"].data_ptr(), bf["Utop"].data_ptr(), C.byref(attained))
    finally:
        set_halo(None)
    ctx.check(rc, "sqb_rhqr_arnoldi_dist")
    raise_status(ctx, "rhqr_arnoldi")
    closed = None if attained.value < 0 else attained.value
    k = m if closed is None else closed
    r = mt if closed is None else closed
    return KrylovBundle(U=bf["U"][:nr, :r], S=bf["S"][:, :r], T=bf["T"][:r, :r], H=bf["H"][: k + 1, :k], psi=psi,
                        beta=float(bf["beta"].item()), scaling=scaling, Q_cols=None, breakdown=closed)


def gmres_solution_local(bundle, y, x0_local, rank, policy=None):
    """x_local = x0_local + this rank's rows of the compact-form correction
    (krylov.py:214-222).  The padded coefficient vector lives in the identity
    rows (rank 0), so Psi pad = [pad[:m+1]; 0] is known on every rank without
    communication (an SRHT of zeros is +0); each rank updates its own rows
    (sqb_compact_update)."""
    policy = policy or DOUBLE_POLICY
    tag = policy.low
    k = bundle.dim
    x0d = to_device(x0_local, "double")[:, 0]
    if k == 0:
        return x0d.clone()
    U = to_device(bundle.U[:, :k], tag)
    rows = U.shape[0]
    od = bundle.S.shape[0]
    yv = torch.as_tensor(y, device="cuda", dtype=torch.float64).reshape(-1)[:k]
    Y = torch.zeros(od, dtype=torch.float64, device="cuda")
    Y[:k] = yv  # Psi pad, top block: a bitwise copy of pad[:m+1]
    X = empty_colmajor(rows, 1, tag, zero=True)
    if rank == 0:
        X[:k, 0] = yv.to(X.dtype)
    Out = empty_colmajor(rows, 1, tag)
    S = to_device(bundle.S[:, :k], "double")
    T = to_device(bundle.T[:k, :k], "double")
    ctx = _lib.context()
    ctx.check(_lib.lib().sqb_compact_update(ctx.h, CODES[tag], Y.data_ptr(), od, S.data_ptr(), ld_of(S),
                                            T.data_ptr(), ld_of(T), 0, k, U.data_ptr(), ld_of(U), rows,
                                            X.data_ptr(), Out.data_ptr()), "sqb_compact_update")
    return x0d + Out[:, 0].to(torch.float64)


def rhqr_gmres_virtual(A, b, x0, m, omega, nranks, scaling=SCALE_SQRT2, policy=None):
    """rhqr_gmres (krylov.py:193-222) on the row-partitioned Arnoldi with
    virtual ranks: each rank's solution rows from its own U rows."""
    from .krylov import hessenberg_lstsq
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    bun = rhqr_arnoldi_virtual(A, b, x0, m, omega, nranks, scaling=scaling, policy=policy)
    y, _, hist = hessenberg_lstsq(bun.H, bun.beta, history=True)
    tag = (policy or DOUBLE_POLICY).low
    row0s, rows, _ = krylov_partition(n, m, omega.n_pad, nranks, tag)
    x = np.empty(n)
    for p in range(nranks):
        if not rows[p]:
            continue
        sl = slice(row0s[p], row0s[p] + rows[p])
        part = type(bun)(U=bun.U[sl], S=bun.S, T=bun.T, H=bun.H, psi=bun.psi, beta=bun.beta, scaling=bun.scaling)
        x[sl] = to_numpy(gmres_solution_local(part, y, x0[sl], p, policy))
    return x, hist
