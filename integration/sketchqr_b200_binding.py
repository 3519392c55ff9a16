"""Reference-side binding of libsketchqr_b200.so — the file a maintainer of the
reference `sketchqr` package would add to dispatch its hot path to the B200
library.  It uses ctypes, numpy and torch (device buffers for
the operator state only) and NOTHING of paper_2405_10923_b200's Python code:
what it exercises is the C ABI declared in include/sketchqr_b200.h.

    import sketchqr, sketchqr_b200_binding as b200
    b200.install(sketchqr, "/path/to/libsketchqr_b200.so")   # patches in place
    F = sketchqr.rhqr_left(W, sketchqr.SRHTSketch(256, n - m, 8))   # runs on the GPU
    b200.uninstall(sketchqr)

Replaced (reference file:line -> export):
    SRHTSketch._apply / GaussianSketch._apply  sketching.py:149-155, :109-125 -> sqb_sketch_apply
    rhqr_left                                  rhqr.py:254-267              -> sqb_rhqr_left_host
    rec_rhqr                                   rhqr.py:368-395              -> sqb_rec_rhqr_host
    rhqr_arnoldi (hence rhqr_gmres)            krylov.py:82-150             -> sqb_rhqr_arnoldi
Policies whose sketch-space precision is not float64, and operators the
library has no descriptor for, fall through to the reference's own code.
"""
import ctypes as C

import numpy as np
import torch

SQB_OK, SQB_ERR_ARG, SQB_ERR_BREAKDOWN, SQB_ERR_SINGULAR, SQB_ERR_CUDA, SQB_ERR_NCCL, SQB_ERR_RANGE, SQB_ERR_NONFINITE = range(8)
DTYPE_CODE = {"double": 0, "single": 1, "half": 2, "bf16": 3}
NP_CODE = {np.dtype(np.float64): 0, np.dtype(np.float32): 1, np.dtype(np.float16): 2}
SCALING_CODE = {"sqrt2": 0, "unit": 1}


class _Sketch(C.Structure):  # include/sketchqr_b200.h: sqb_sketch
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("ell", C.c_int64), ("n", C.c_int64),
                ("n_pad", C.c_int64), ("scale", C.c_double), ("sign_bits", C.c_void_p), ("indices", C.c_void_p),
                ("G", C.c_void_p), ("ldg", C.c_int64)]


_MATVEC_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


class _Operator(C.Structure):  # include/sketchqr_b200.h: sqb_operator
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("n", C.c_int64), ("indptr", C.c_void_p),
                ("indices", C.c_void_p), ("data", C.c_void_p), ("A", C.c_void_p), ("lda", C.c_int64),
                ("cb", _MATVEC_CB), ("user", C.c_void_p), ("xbuf", C.c_void_p), ("ybuf", C.c_void_p)]


_state = {"lib": None, "ctx": None, "saved": {}}
_p, _i64, _int = C.c_void_p, C.c_int64, C.c_int


def _load(path):
    L = C.CDLL(path)
    L.sqb_ctx_create.argtypes = [_int, _p, C.POINTER(_p)]
    L.sqb_ctx_status.argtypes = [_p, C.POINTER(_int), C.POINTER(_int), C.POINTER(C.c_double)]
    L.sqb_ctx_last_error.argtypes = [_p]
    L.sqb_ctx_last_error.restype = C.c_char_p
    L.sqb_sketch_apply.argtypes = [_p, C.POINTER(_Sketch), _int, _p, _i64, _i64, _p, _i64]
    host = [_p, C.POINTER(_Sketch), _int, _int, _p, _i64, _i64, _i64, _int, _p, _i64, _p, _i64, _p, _i64, _p, _i64,
            _p, _p, _p]
    L.sqb_rhqr_left_host.argtypes = host
    L.sqb_rec_rhqr_host.argtypes = host
    L.sqb_rhqr_arnoldi.argtypes = [_p, C.POINTER(_Sketch), C.POINTER(_Operator), _int, _int, _int, C.c_double, _p, _p,
                                   _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _p, C.POINTER(_int)]
    ctx = _p()
    rc = L.sqb_ctx_create(torch.cuda.current_device(), None, C.byref(ctx))
    if rc != SQB_OK:
        raise RuntimeError(f"sqb_ctx_create failed ({rc})")
    return L, ctx


def _descriptor(om):
    """Device state + sqb_sketch of a reference operator (cached on the object)."""
    d = getattr(om, "_b200", None)
    if d is not None:
        return d
    kind = getattr(om, "kind", None)
    if kind == "srht":
        bits = np.packbits(om.signs < 0, bitorder="little")
        bits = np.concatenate([bits, np.zeros((-bits.size) % 4, np.uint8)])
        bits_d = torch.from_numpy(bits).cuda()
        idx_d = torch.from_numpy(np.ascontiguousarray(om.indices, dtype=np.int64)).cuda()
        sk = _Sketch(0, 0, om.ell, om.n, om.n_pad, om.scale, bits_d.data_ptr(), idx_d.data_ptr(), None, 0)
        keep = (bits_d, idx_d)
    elif kind == "gauss":
        # the reference's own rows (sketching.py:100-107), generated once and kept on the device
        G = om._cache.get(np.dtype(np.float64))
        if G is None:
            G = om._rows(0, om.ell)
        G_d = torch.from_numpy(np.ascontiguousarray(G)).cuda()
        sk = _Sketch(1, 0, om.ell, om.n, 0, 0.0, None, None, G_d.data_ptr(), om.n)
        keep = (G_d,)
    elif kind == "identity":
        sk = _Sketch(2, 0, om.ell, om.n, 0, 0.0, None, None, None, 0)
        keep = ()
    else:
        return None
    om._b200 = (sk, keep)
    return om._b200


def _raise(mod, what, tag="double"):
    L, ctx = _state["lib"], _state["ctx"]
    code, col, val = _int(), _int(), C.c_double()
    L.sqb_ctx_status(ctx, C.byref(code), C.byref(col), C.byref(val))
    code, col, val = code.value, col.value, val.value
    if code == SQB_OK:
        return
    lin = mod.linalg
    if code == SQB_ERR_BREAKDOWN:
        if what == "rec_rhqr":
            if val == -1.0:
                raise lin.BreakdownError(f"reconstruction factor has zero diagonal at column {col}")
            raise lin.BreakdownError(f"column {col} exactly dependent on its predecessors")
        if val == 0.0:
            raise lin.BreakdownError(f"sketched tail annihilated at column {col}")
        raise lin.BreakdownError(f"reflector scale degenerated at column {col} (rho={val:.3e})")
    if code == SQB_ERR_RANGE:
        raise mod.precision.PrecisionRangeError(f"value {val:g} overflows {tag} range")
    if code == SQB_ERR_NONFINITE:
        raise ValueError("array must not contain infs or NaNs")
    raise RuntimeError(f"{what}: device status {code} at column {col}")


def _check(rc, what):
    if rc != SQB_OK:
        msg = _state["lib"].sqb_ctx_last_error(_state["ctx"]).decode(errors="replace")
        if rc == SQB_ERR_ARG:
            raise ValueError(msg or what)
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def _factor(mod, entry, W, omega, scaling, policy):
    """rhqr_left / rec_rhqr through the host-operand exports; None = not handled."""
    policy = policy or mod.precision.DOUBLE_POLICY
    if policy.high != "double" or policy.low not in DTYPE_CODE:
        return None
    Wa = np.asarray(mod.linalg.as_array(W), dtype=np.float64)
    if Wa.ndim != 2:
        return None
    n, m = Wa.shape
    psi = mod.rhqr._embed(omega, n, m)  # the reference's own validation (ValueError texts)
    desc = _descriptor(omega)
    if desc is None:
        return None
    if not (Wa.flags.c_contiguous or Wa.flags.f_contiguous):
        Wa = np.ascontiguousarray(Wa)
    layout, ldw = (0, m) if Wa.flags.c_contiguous else (1, n)
    od = m + omega.ell
    U = torch.empty((m, n), dtype=torch.float64, pin_memory=True).numpy().T  # page-locked, column-major
    S, T, R, sc = np.empty((m, od)).T, np.empty((m, m)).T, np.empty((m, m)).T, np.empty(3 * m)
    p = lambda a: a.ctypes.data  # noqa: E731
    L, ctx = _state["lib"], _state["ctx"]
    rc = getattr(L, entry)(ctx, C.byref(desc[0]), SCALING_CODE[scaling], DTYPE_CODE[policy.low], p(Wa), n, m, ldw,
                           layout, p(U), n, p(S), od, p(T), m, p(R), m, p(sc), p(sc) + 8 * m, p(sc) + 16 * m)
    _check(rc, entry)
    _raise(mod, "rec_rhqr" if entry == "sqb_rec_rhqr_host" else "rhqr_left", policy.low)
    return mod.rhqr.RHQRFactors(U=U, S=S, T=T, R=R, psi=psi, scaling=scaling, sigmas=sc[:m].copy(),
                                rhos=sc[m:2 * m].copy(), betas=sc[2 * m:].copy())


def _arnoldi(mod, A, b, x0, m, omega, scaling, policy, store_q, happy_tol):
    """rhqr_arnoldi through sqb_rhqr_arnoldi (fp64 storage); None = not handled."""
    import scipy.sparse
    policy = policy or mod.precision.DOUBLE_POLICY
    if policy.high != "double" or policy.low != "double":
        return None
    b = np.asarray(mod.linalg.as_array(b), dtype=np.float64)
    n = b.shape[0]
    psi = mod.rhqr._embed(omega, n, m + 1)
    desc = _descriptor(omega)
    if desc is None:
        return None
    keep, err = [], []
    op = _Operator(n=n)
    if scipy.sparse.issparse(A):
        M = scipy.sparse.csr_matrix(A, dtype=np.float64)
        M.sort_indices()
        ip = torch.from_numpy(M.indptr.astype(np.int64)).cuda()
        ix = torch.from_numpy(M.indices.astype(np.int32)).cuda()
        dv = torch.from_numpy(np.ascontiguousarray(M.data)).cuda()
        keep += [ip, ix, dv]
        op.kind, op.indptr, op.indices, op.data = 0, ip.data_ptr(), ix.data_ptr(), dv.data_ptr()
    elif callable(A):
        xbuf = torch.empty(n, dtype=torch.float64, device="cuda")
        ybuf = torch.empty(n, dtype=torch.float64, device="cuda")

        def _cb(user, stream):  # the reference hands its matvec a numpy vector (krylov.py:28-35)
            try:
                y = np.asarray(A(xbuf.cpu().numpy()), dtype=np.float64)
                ybuf.copy_(torch.from_numpy(np.ascontiguousarray(y)).reshape(-1))
                return 0
            except BaseException as e:  # noqa: BLE001
                err.append(e)
                return 1

        cb = _MATVEC_CB(_cb)
        keep += [xbuf, ybuf, cb]
        op.kind, op.cb, op.xbuf, op.ybuf = 2, cb, xbuf.data_ptr(), ybuf.data_ptr()
    else:
        Ad = torch.from_numpy(np.ascontiguousarray(np.asarray(mod.linalg.as_array(A), dtype=np.float64))).cuda()
        keep.append(Ad)
        op.kind, op.A, op.lda = 1, Ad.data_ptr(), Ad.stride(0)
    if happy_tol is None:
        happy_tol = 32.0 * policy.u_high
    mt, od = m + 1, psi.out_dim
    ld = (n + 1) // 2 * 2
    f64 = dict(dtype=torch.float64, device="cuda")
    bd = torch.from_numpy(b).cuda()
    x0d = torch.zeros(n, **f64) if x0 is None else torch.from_numpy(np.asarray(x0, dtype=np.float64)).cuda()
    U, S, T = torch.zeros((mt, ld), **f64), torch.zeros((mt, od), **f64), torch.zeros((mt, mt), **f64)
    H, Q = torch.zeros((m, mt), **f64), (torch.zeros((m, ld), **f64) if store_q else None)
    beta, attained = torch.zeros(1, **f64), _int(-1)
    L, ctx = _state["lib"], _state["ctx"]
    rc = L.sqb_rhqr_arnoldi(ctx, C.byref(desc[0]), C.byref(op), m, SCALING_CODE[scaling], 0, float(happy_tol),
                            bd.data_ptr(), x0d.data_ptr(), U.data_ptr(), ld, S.data_ptr(), od, T.data_ptr(), mt,
                            H.data_ptr(), mt, Q.data_ptr() if store_q else None, ld if store_q else 1,
                            beta.data_ptr(), C.byref(attained))
    if err:
        raise err[0]
    _check(rc, "sqb_rhqr_arnoldi")
    _raise(mod, "rhqr_arnoldi")
    closed = None if attained.value < 0 else attained.value
    k = m if closed is None else closed
    r = mt if closed is None else closed
    h = lambda t: t.cpu().numpy().T  # noqa: E731  (column-major device buffers)
    return mod.krylov.KrylovBundle(U=h(U)[:n, :r], S=h(S)[:, :r], T=h(T)[:r, :r], H=h(H)[: k + 1, :k].copy(), psi=psi,
                                   beta=float(beta.item()), scaling=scaling,
                                   Q_cols=h(Q)[:n, :k].copy() if store_q else None, breakdown=closed)


def _apply(mod, om, X, dtype):
    """SketchOperator._apply (X: n x k float64, returns ell x k in `dtype`); None = not handled."""
    code = NP_CODE.get(np.dtype(dtype))
    desc = _descriptor(om)
    if code is None or desc is None:
        return None
    with np.errstate(over="ignore"):
        Xl = np.asfortranarray(np.asarray(X, dtype=np.float64).astype(dtype))
    n, k = Xl.shape
    ld = (n + 7) // 8 * 8  # 16-byte aligned columns in every format
    Xd = torch.zeros((k, ld), dtype={0: torch.float64, 1: torch.float32, 2: torch.float16}[code], device="cuda")
    Xd[:, :n] = torch.from_numpy(np.ascontiguousarray(Xl.T)).cuda()
    Y = torch.empty((k, om.ell), dtype=torch.float64, device="cuda")
    _check(_state["lib"].sqb_sketch_apply(_state["ctx"], C.byref(desc[0]), code, Xd.data_ptr(), ld, k, Y.data_ptr(),
                                          om.ell), "sqb_sketch_apply")
    _raise(mod, "sketch apply")
    return Y.cpu().numpy().T.astype(dtype)


def install(mod, lib_path):
    """Patch the reference package `mod` (the imported `sketchqr`) in place."""
    if _state["lib"] is None:
        _state["lib"], _state["ctx"] = _load(lib_path)
    saved = _state["saved"]
    if saved:
        return
    orig_left, orig_rec = mod.rhqr.rhqr_left, mod.rhqr.rec_rhqr
    orig_srht, orig_gauss = mod.sketching.SRHTSketch._apply, mod.sketching.GaussianSketch._apply

    def rhqr_left(W, omega, scaling=mod.linalg.SCALE_SQRT2, policy=None):
        mod.linalg.check_scaling(scaling)
        out = _factor(mod, "sqb_rhqr_left_host", W, omega, scaling, policy)
        return out if out is not None else orig_left(W, omega, scaling, policy)

    def rec_rhqr(W, omega, scaling=mod.linalg.SCALE_SQRT2, policy=None):
        mod.linalg.check_scaling(scaling)
        out = _factor(mod, "sqb_rec_rhqr_host", W, omega, scaling, policy)
        return out if out is not None else orig_rec(W, omega, scaling, policy)

    def srht_apply(self, X, dtype):
        out = _apply(mod, self, X, dtype)
        return out if out is not None else orig_srht(self, X, dtype)

    orig_arn = mod.krylov.rhqr_arnoldi

    def rhqr_arnoldi(A, b, x0, m, omega, scaling=mod.linalg.SCALE_SQRT2, policy=None, store_q=True, happy_tol=None):
        mod.linalg.check_scaling(scaling)
        out = _arnoldi(mod, A, b, x0, m, omega, scaling, policy, store_q, happy_tol)
        return out if out is not None else orig_arn(A, b, x0, m, omega, scaling, policy, store_q, happy_tol)

    rhqr_left.__doc__, rec_rhqr.__doc__, rhqr_arnoldi.__doc__ = orig_left.__doc__, orig_rec.__doc__, orig_arn.__doc__
    saved["funcs"] = []
    import sys
    for name, new, old in (("rhqr_left", rhqr_left, orig_left), ("rec_rhqr", rec_rhqr, orig_rec),
                           ("rhqr_arnoldi", rhqr_arnoldi, orig_arn)):
        for m2 in list(sys.modules.values()):  # every module that imported the name holds its own reference
            if m2 is not None and getattr(m2, "__name__", "").split(".")[0] == mod.__name__ and getattr(m2, name, None) is old:
                setattr(m2, name, new)
                saved["funcs"].append((m2, name, old))
    mod.sketching.SRHTSketch._apply = srht_apply
    saved["srht"] = orig_srht
    saved["gauss"] = orig_gauss


def uninstall(mod):
    saved = _state["saved"]
    for m2, name, old in saved.get("funcs", []):
        setattr(m2, name, old)
    if "srht" in saved:
        mod.sketching.SRHTSketch._apply = saved["srht"]
    saved.clear()
