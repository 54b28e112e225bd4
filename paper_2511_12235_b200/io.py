"""CSM1 / CTT1 containers (reference io.hpp:31-48, io.cpp:153-270;
SURVEY.md §8(f) row 2) for device-resident data.

write_matrix streams a device CSR to a CSM1 file byte-identical to the
reference's writer (columns widened to u64 on the device, pinned double
buffering); read_matrix loads one straight into device memory with the
reference's checks. Tensors (CTT1) go through host buffers.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .geometry import CtsmError
from .projector import Context, SparseSystemMatrix, _stream

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def write_matrix(path: str, w: SparseSystemMatrix) -> None:
    """io.cpp:153-177."""
    ctx = Context.get(w.device)
    meta = w.meta.encode()
    _lib.check(_lib.lib().ctsm_write_csm1_device(
        ctx.handle, str(path).encode(), w.n_rows, w.n_cols, w.row_start.data_ptr(),
        w.col.data_ptr(), w.val.data_ptr(), meta, len(meta), _stream(ctx.device)))


def read_matrix(path: str, device: Optional[int] = None) -> SparseSystemMatrix:
    """io.cpp:179-227, into device memory."""
    n_rows, n_cols, nnz, meta_len = (ctypes.c_uint64() for _ in range(4))
    _lib.check(_lib.lib().ctsm_csm1_header(str(path).encode(), ctypes.byref(n_rows),
                                           ctypes.byref(n_cols), ctypes.byref(nnz),
                                           ctypes.byref(meta_len)))
    ctx = Context.get(device)
    dev = f"cuda:{ctx.device}"
    rs = torch.empty(n_rows.value + 1, dtype=torch.int64, device=dev)
    col = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    val = torch.empty(nnz.value, dtype=torch.float64, device=dev)
    meta = ctypes.create_string_buffer(max(1, meta_len.value))
    _lib.check(_lib.lib().ctsm_read_csm1_device(ctx.handle, str(path).encode(), rs.data_ptr(),
                                                col.data_ptr(), val.data_ptr(),
                                                ctypes.cast(meta, ctypes.c_void_p),
                                                _stream(ctx.device)))
    return SparseSystemMatrix(n_rows=n_rows.value, n_cols=n_cols.value, row_start=rs, col=col,
                              val=val, meta=meta.raw[:meta_len.value].decode(),
                              device=ctx.device)


def write_tensor(path: str, dims, data) -> None:
    """io.cpp:229-247 (CTT1)."""
    d = np.ascontiguousarray(dims, np.uint64)
    if torch is not None and isinstance(data, torch.Tensor):
        data = data.detach().cpu().numpy()
    x = np.ascontiguousarray(data, np.float64)
    if d.size < 1 or d.size > 8:
        raise CtsmError("InvalidSpec", "tensor rank must be between 1 and 8")
    if int(np.prod(d, dtype=np.uint64)) != x.size:
        raise CtsmError("DimensionMismatch", "tensor dims do not match payload size")
    _lib.check(_lib.lib().ctsm_write_ctt1(str(path).encode(), d.ctypes.data_as(ctypes.c_void_p),
                                          int(d.size), x.ctypes.data_as(ctypes.c_void_p)))


def read_tensor(path: str) -> Tuple[np.ndarray, list]:
    """io.cpp:249-270 -> (data, dims)."""
    dims = np.zeros(8, np.uint64)
    rank = ctypes.c_int(0)
    _lib.check(_lib.lib().ctsm_ctt1_header(str(path).encode(), dims.ctypes.data_as(ctypes.c_void_p),
                                           ctypes.byref(rank)))
    d = [int(v) for v in dims[:rank.value]]
    out = np.empty(int(np.prod(d)) if d else 0, np.float64)
    _lib.check(_lib.lib().ctsm_read_ctt1(str(path).encode(), out.ctypes.data_as(ctypes.c_void_p),
                                         out.size))
    return out, d
