"""Device storage helpers: column-major buffers, host<->device conversion.

Layout: an (rows x cols) operand is stored column-major with a
leading dimension that is a multiple of 16 elements, and shifted so that row
`align_row` of every column starts on a 16-byte boundary (the sketch kernels
stream rows >= m with 128-bit loads).  It is exposed as a torch view of
shape (rows, cols) with strides (1, ld).
"""

from __future__ import annotations

import numpy as np
import torch

from .precision import DTYPES, round_to, tag_of_dtype

TORCH_DTYPES = {"double": torch.float64, "single": torch.float32, "half": torch.float16,
                "bf16": torch.bfloat16}
CODES = {"double": 0, "single": 1, "half": 2, "bf16": 3}
ESIZE = {"double": 8, "single": 4, "half": 2, "bf16": 2}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2405_10923_b200 needs a CUDA device (sm_100a); there is no CPU fallback")


def is_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def tag_of_torch(dt) -> str:
    for t, d in TORCH_DTYPES.items():
        if d == dt:
            return t
    raise ValueError(f"unsupported torch dtype {dt}")


def empty_colmajor(rows: int, cols: int, tag: str = "double", align_row: int = 0, device=None,
                   zero: bool = False) -> torch.Tensor:
    require_cuda()
    tdt = TORCH_DTYPES[tag]
    vn = 16 // ESIZE[tag]
    ld = max(16, -(-max(rows, 1) // 16) * 16)
    off = (-align_row) % vn
    n = ld * max(cols, 1) + off + vn
    flat = (torch.zeros if zero else torch.empty)(n, dtype=tdt, device=device or "cuda")
    return torch.as_strided(flat, (rows, cols), (1, ld), off)


def ld_of(t: torch.Tensor) -> int:
    if t.dim() == 1:
        return max(1, t.shape[0])
    if t.shape[1] <= 1:
        return max(t.stride(1), t.shape[0], 1)
    return t.stride(1)


def is_colmajor(t: torch.Tensor) -> bool:
    return t.dim() == 2 and (t.shape[0] <= 1 or t.stride(0) == 1) and (
        t.shape[1] <= 1 or t.stride(1) >= t.shape[0])


def host_to_lo(X, tag: str) -> np.ndarray:
    """Round a host array to the storage format (raises PrecisionRangeError on
    overflow, precision.py:45-50) and return it in that numpy dtype."""
    Xr = round_to(X, tag)
    return Xr.astype(DTYPES[tag])


def to_device(X, tag: str, align_row: int = 0) -> torch.Tensor:
    """Host array / device tensor -> column-major device tensor in `tag`."""
    require_cuda()
    if isinstance(X, torch.Tensor):
        X2 = X if X.dim() == 2 else X.reshape(-1, 1)
        if not X2.is_cuda:
            X2 = X2.cuda()
        if X2.dtype == TORCH_DTYPES[tag] and is_colmajor(X2) and (
                (X2.data_ptr() + align_row * ESIZE[tag]) % 16 == 0) and ld_of(X2) % (16 // ESIZE[tag]) == 0:
            return X2
        out = empty_colmajor(X2.shape[0], X2.shape[1], tag, align_row)
        if X2.dtype != TORCH_DTYPES[tag] and X2.dtype == torch.float64 and tag != "double":
            # round exactly like the host path: fp64 -> fp32 -> bf16 for bf16, direct otherwise
            X2 = X2.to(torch.float32) if tag in ("bf16", "single") else X2
        out.copy_(X2)
        return out
    A = host_to_lo(X, tag)
    if A.ndim == 1:
        A = A[:, None]
    if not (A.flags.c_contiguous or A.flags.f_contiguous):
        A = np.ascontiguousarray(A)
    # a Fortran-order host array is uploaded as is (the device copy keeps its
    # strides, so the column-major store below is a plain copy)
    if tag == "bf16":
        src = torch.from_numpy(A.view(np.int16)).view(torch.bfloat16)
    else:
        src = torch.from_numpy(A)
    out = empty_colmajor(A.shape[0], A.shape[1], tag, align_row)
    out.copy_(src.cuda(non_blocking=False))
    return out


def to_numpy(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> C-ordered float64 host ndarray (values representable in
    t's dtype).  The layout change and the widening run on the device; the
    copy lands in pinned host memory (full PCIe/C2C bandwidth)."""
    h = t.detach()
    if h.dtype != torch.float64:
        h = h.to(torch.float64)
    h = h.contiguous()  # row-major on the device (column-major views are transposed here)
    if h.numel() < (1 << 16):
        return h.cpu().numpy()
    out = torch.empty(h.shape, dtype=torch.float64, pin_memory=True)
    out.copy_(h, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def host_f64(X):
    """Host operand -> (float64 ndarray, layout, ld) for the host-buffer entry
    points: layout 0 = row-major (C-order, ld = row stride), 1 = column-major
    (Fortran order, ld = column stride).  A CPU tensor is viewed, not copied,
    so page-locked tensors keep their full-bandwidth DMA path."""
    if isinstance(X, torch.Tensor):
        X = X.detach()
        X = X.numpy() if X.dtype == torch.float64 else X.to(torch.float64).numpy()
    A = np.asarray(X, dtype=np.float64)
    if A.ndim == 1:
        A = A[:, None]
    if A.ndim != 2:
        raise ValueError(f"expected a matrix, got shape {A.shape}")
    n, m = A.shape
    if A.flags.c_contiguous and (A.strides[0] // 8) >= m:
        return A, 0, max(m, A.strides[0] // 8)
    if A.flags.f_contiguous:
        return A, 1, max(n, A.strides[1] // 8 if m > 1 else n)
    A = np.ascontiguousarray(A)
    return A, 0, m


def pinned_f64(rows: int, cols: int) -> np.ndarray:
    """Fresh float64 (rows x cols) Fortran-order ndarray in page-locked memory
    (torch's caching host allocator; the array keeps the block alive)."""
    t = torch.empty((max(cols, 1), max(rows, 1)), dtype=torch.float64, pin_memory=True)
    return t.numpy().T[:rows, :cols]


def np_dtype_tag(dt) -> str:
    return tag_of_dtype(dt)
