"""ctypes binding of libsketchqr_b200.so (the C ABI in include/sketchqr_b200.h).

The product path has no CPU fallback: if the shared library or a CUDA device
is missing, `lib()` / `context()` raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsketchqr_b200.so")

SQB_OK, SQB_ERR_ARG, SQB_ERR_BREAKDOWN, SQB_ERR_SINGULAR, SQB_ERR_CUDA, SQB_ERR_NCCL, SQB_ERR_RANGE, \
    SQB_ERR_NONFINITE = range(8)
SQB_F64, SQB_F32, SQB_F16, SQB_BF16 = range(4)
SQB_SCALE_SQRT2, SQB_SCALE_UNIT = 0, 1
SQB_SKETCH_SRHT, SQB_SKETCH_DENSE, SQB_SKETCH_IDENTITY = 0, 1, 2

i64 = C.c_int64
vp = C.c_void_p
dp = C.c_void_p  # device pointers are passed as integers


class SketchDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("reserved", C.c_int32), ("ell", i64), ("n", i64), ("n_pad", i64),
        ("scale", C.c_double), ("sign_bits", vp), ("indices", vp), ("G", vp), ("ldg", i64),
    ]


SQB_OP_CSR, SQB_OP_DENSE, SQB_OP_CALLBACK = 0, 1, 2
MATVEC_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)


class OperatorDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("reserved", C.c_int32), ("n", i64), ("indptr", vp), ("indices", vp),
        ("data", vp), ("A", vp), ("lda", i64), ("cb", MATVEC_CB), ("user", vp), ("xbuf", vp), ("ybuf", vp),
    ]


# name -> (argtypes, restype); every export returns int unless stated
_SIGS = {
    "sqb_version": ([], C.c_int),
    "sqb_ctx_create": ([C.c_int, vp, C.POINTER(vp)], C.c_int),
    "sqb_ctx_destroy": ([vp], C.c_int),
    "sqb_ctx_set_stream": ([vp, vp], C.c_int),
    "sqb_ctx_last_error": ([vp], C.c_char_p),
    "sqb_ctx_status": ([vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_double)], C.c_int),
    "sqb_round_scalar": ([C.c_int, C.c_double], C.c_double),
    "sqb_ctx_launches": ([vp], i64),
    "sqb_ctx_profile": ([vp, C.c_int], C.c_int),
    "sqb_debug_step_stamps": ([vp, dp, C.c_int], C.c_int),
    "sqb_debug_col_stamps": ([vp, dp, C.c_int], C.c_int),
    "sqb_ctx_trace": ([vp, C.c_int], C.c_int),
    "sqb_ctx_trace_read": ([vp, C.c_char_p, i64], C.c_int),
    "sqb_ctx_profile_read": ([vp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(i64)], C.c_int),
    "sqb_sketch_apply": ([vp, C.POINTER(SketchDesc), C.c_int, dp, i64, i64, dp, i64], C.c_int),
    "sqb_embedded_apply": ([vp, C.POINTER(SketchDesc), i64, C.c_int, dp, i64, i64, dp, i64], C.c_int),
    "sqb_rhqr_left": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, dp, i64,
                       dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_rhqr_left_host": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, vp, i64, i64, i64, C.c_int,
                            vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, vp], C.c_int),
    "sqb_rec_rhqr_host": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, vp, i64, i64, i64, C.c_int,
                           vp, i64, vp, i64, vp, i64, vp, i64, vp, vp, vp], C.c_int),
    "sqb_ctx_trim": ([vp], C.c_int),
    "sqb_rhqr_block": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, i64, dp, i64,
                        dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_rhqr_right": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, dp, i64,
                        dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_t_factor": ([vp, dp, i64, i64, i64, dp, i64], C.c_int),
    "sqb_trim_rhqr_left": ([vp, C.POINTER(SketchDesc), dp, i64, dp, i64, C.c_int, C.c_int, dp, i64, i64, i64,
                            dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_ctx_set_halo": ([vp, C.c_int, vp], C.c_int),
    "sqb_trim_rhqr_right": ([vp, C.POINTER(SketchDesc), dp, i64, dp, i64, C.c_int, C.c_int, dp, i64, i64, i64,
                             dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_colscaled_apply": ([vp, C.POINTER(SketchDesc), dp, i64, C.c_int, dp, i64, i64, dp, i64], C.c_int),
    "sqb_trim_thin_q": ([vp, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64, dp, i64, i64, dp, i64], C.c_int),
    "sqb_rec_rhqr": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, dp, i64,
                      dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_apply_reflectors": ([vp, C.POINTER(SketchDesc), i64, C.c_int, dp, i64, i64, i64, dp, i64,
                              dp, i64, C.c_int, dp, i64, i64, dp, i64], C.c_int),
    "sqb_thin_q": ([vp, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64], C.c_int),
    "sqb_gram": ([vp, dp, i64, i64, i64, dp, i64], C.c_int),
    "sqb_sketch_q": ([vp, C.c_int, dp, i64, i64, dp, i64, dp, i64, i64, dp, i64], C.c_int),
    "sqb_residual_norms": ([vp, dp, i64, dp, i64, dp, i64, i64, i64, i64, dp], C.c_int),
    "sqb_rhqr_arnoldi": ([vp, C.POINTER(SketchDesc), C.POINTER(OperatorDesc), C.c_int, C.c_int, C.c_int,
                          C.c_double, dp, dp, dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp,
                          C.POINTER(C.c_int)], C.c_int),
    "sqb_hessenberg_lstsq": ([vp, dp, i64, i64, i64, C.c_double, dp, dp, dp, dp], C.c_int),
    "sqb_csr_spmv": ([vp, C.c_int, i64, dp, dp, dp, dp, dp, dp], C.c_int),
    "sqb_arnoldi_q": ([vp, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64, i64, dp, i64], C.c_int),
    "sqb_nccl_unique_id": ([C.c_char_p, C.c_int], C.c_int),
    "sqb_ctx_init_comm": ([vp, C.c_char_p, C.c_int, C.c_int], C.c_int),
    "sqb_p2p_mailbox": ([vp, C.c_int, i64, vp], C.c_int),
    "sqb_p2p_open": ([vp, C.c_int, vp], C.c_int),
    "sqb_p2p_virtual": ([vp, C.c_int, i64], C.c_int),
    "sqb_p2p_close": ([vp], C.c_int),
    "sqb_p2p_set_timeout_ms": ([vp, i64], C.c_int),
    "sqb_rhqr_left_dist": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64,
                            dp, i64, dp, i64, dp, dp, dp, dp], C.c_int),
    "sqb_rhqr_left_virtual": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, C.c_int, C.POINTER(vp),
                               C.POINTER(i64), C.POINTER(vp), C.POINTER(i64), i64, dp, i64, dp, i64, dp, i64,
                               dp, dp, dp, dp], C.c_int),
    "sqb_rec_rhqr_dist": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64,
                           dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_rec_rhqr_virtual": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, C.c_int, C.POINTER(vp),
                              C.POINTER(i64), C.POINTER(vp), C.POINTER(i64), i64, dp, i64, dp, i64, dp, i64,
                              dp, dp, dp, dp], C.c_int),
    "sqb_compact_update": ([vp, C.c_int, dp, i64, dp, i64, dp, i64, C.c_int, i64, dp, i64, i64, dp, dp], C.c_int),
    "sqb_rhqr_arnoldi_dist": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, C.c_int, C.c_double, i64, i64, i64,
                               dp, dp, dp, dp, dp, dp, i64, dp, i64, dp, i64, dp, i64, dp, i64, dp, dp,
                               C.POINTER(C.c_int)], C.c_int),
    "sqb_rhqr_arnoldi_virtual": ([vp, C.POINTER(SketchDesc), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  C.POINTER(i64), C.POINTER(i64), i64, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                  C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(i64), C.POINTER(vp), i64,
                                  C.POINTER(vp), i64, C.POINTER(vp), i64, C.POINTER(vp), C.POINTER(vp),
                                  C.POINTER(C.c_int)], C.c_int),
    "sqb_householder_qr": ([vp, C.c_int, dp, i64, i64, i64, dp, i64, dp, i64, dp, i64, dp, dp, dp], C.c_int),
    "sqb_upper_tri_solve": ([vp, dp, i64, i64, dp, i64, i64, dp, i64], C.c_int),
    "sqb_rh_vector": ([vp, C.c_int, C.c_int, dp, i64, dp, i64, i64, dp, dp, dp], C.c_int),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load the library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -m paper_2405_10923_b200.build` "
                        "(there is no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, (args, res) in _SIGS.items():
                    f = getattr(L, name)
                    f.argtypes = args
                    f.restype = res
                _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


class SketchQRError(RuntimeError):
    pass


class Context:
    """One library context per (device, stream)."""

    def __init__(self, device: int, stream: int):
        self.device = device
        self.stream = stream
        h = vp()
        rc = lib().sqb_ctx_create(device, vp(stream), C.byref(h))
        if rc != SQB_OK:
            raise SketchQRError(f"sqb_ctx_create failed with status {rc}")
        self.h = h

    def set_stream(self, stream: int):
        if stream != self.stream:
            # the C side orders the new stream after the old one (shared scratch)
            self.check(lib().sqb_ctx_set_stream(self.h, vp(stream)), "sqb_ctx_set_stream")
            self.stream = stream

    def check(self, rc, what):
        if rc != SQB_OK:
            msg = lib().sqb_ctx_last_error(self.h).decode(errors="replace")
            if rc == SQB_ERR_ARG:
                raise ValueError(msg or f"{what}: invalid argument")
            raise SketchQRError(f"{what} failed (status {rc}): {msg}")

    def status(self):
        code, col, val = C.c_int(), C.c_int(), C.c_double()
        self.check(lib().sqb_ctx_status(self.h, C.byref(code), C.byref(col), C.byref(val)), "status")
        return code.value, col.value, val.value

    def profile(self, enable: bool):
        lib().sqb_ctx_profile(self.h, 1 if enable else 0)

    def profile_read(self):
        ms, by, n = C.c_double(), C.c_double(), i64()
        self.check(lib().sqb_ctx_profile_read(self.h, C.byref(ms), C.byref(by), C.byref(n)), "profile_read")
        return ms.value, by.value, n.value

    def launches(self) -> int:
        return int(lib().sqb_ctx_launches(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and _lib is not None:
                _lib.sqb_ctx_destroy(self.h)
        except Exception:
            pass


_ctxs = {}
_ctx_lock = threading.Lock()


def context():
    """Context bound to torch's current device and stream.

    One context per (device, host thread): a context's scratch workspace,
    host-operand arena and status word are not safe to share between threads.
    Within a thread, switching torch streams orders the new stream after the
    old one (sqb_ctx_set_stream), so calls on different streams never race on
    the shared scratch."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2405_10923_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = torch.cuda.current_device()
    stream = torch.cuda.current_stream(dev).cuda_stream
    key = (dev, threading.get_ident())
    ctx = _ctxs.get(key)
    if ctx is None:
        with _ctx_lock:
            ctx = _ctxs.get(key)
            if ctx is None:
                ctx = _ctxs[key] = Context(dev, stream)
    ctx.set_stream(stream)
    return ctx


def round_scalar(dtype_code: int, x: float) -> float:
    return float(lib().sqb_round_scalar(dtype_code, float(x)))


def np_code(dt) -> int:
    dt = np.dtype(dt)
    if dt == np.float64:
        return SQB_F64
    if dt == np.float32:
        return SQB_F32
    if dt == np.float16:
        return SQB_F16
    if dt.name == "bfloat16":
        return SQB_BF16
    raise ValueError(f"unsupported arithmetic dtype {dt}")
