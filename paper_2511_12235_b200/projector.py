"""The reference's projector API (projector.hpp:12-79) on B200.

Every function keeps the reference's name, argument meaning and error
behaviour (raises ``CtsmError`` with the reference ErrorCode name):

===============================  ==============================================
reference (projector.hpp)        here
===============================  ==============================================
build_system_matrix   (41-44)    build_system_matrix -> SparseSystemMatrix
forward_project       (47-48)    forward_project      (K3, CSR SpMV)
back_project          (51-52)    back_project         (K4, transpose SpMV)
forward_project_matrix_free      forward_project_matrix_free (K5)
                      (56-59)
(absent)                         back_project_matrix_free    (K6)
spectral_norm_power   (63-64)    spectral_norm_power  (on K3/K4)
scale_values          (66)       scale_values
angle_column_sums     (69-70)    angle_column_sums    (K6 on one angle)
(absent)                         sirt                 (K7/K8, BASELINE config 4)
===============================  ==============================================

Operands may be numpy arrays (host; results come back as numpy, like the
reference's value semantics) or CUDA torch tensors (device-resident; results
stay on the device). All compute runs in libctsm_b200.so; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .geometry import CtsmError, ScanGeometry

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

DEFAULT_BUDGET = 5 << 30  # projector.hpp:43-44


class MatrixMode:
    consistent = "consistent"
    line = "line"
    multiline = "multiline"


def parse_matrix_mode(text: str):
    """projector.cpp:16-31 -> (mode, k)."""
    if text == "consistent":
        return MatrixMode.consistent, 1
    if text == "line":
        return MatrixMode.line, 1
    if text.startswith("multiline:"):
        try:
            k = int(text[10:])
        except ValueError:
            raise CtsmError("InvalidConfig", f"bad multiline ray count in '{text}'")
        if k <= 0:
            raise CtsmError("InvalidConfig", "multiline ray count must be > 0")
        return MatrixMode.multiline, k
    raise CtsmError("InvalidConfig", f"unknown matrix mode '{text}'")


def matrix_mode_name(mode: str, k: int = 1) -> str:
    return f"multiline:{k}" if mode == MatrixMode.multiline else mode


_MODE_CODES = {MatrixMode.consistent: 0, MatrixMode.line: 1, MatrixMode.multiline: 2}


def _mode_code(mode: str, k: int) -> int:
    """MatrixMode ordinal (projector.hpp:12-16) for the C-ABI; line and
    multiline(k) run the device ray tracer (baseline.cpp:13-128)."""
    if mode not in _MODE_CODES:
        raise CtsmError("InvalidSpec", f"unknown matrix mode '{mode}'")
    if mode == MatrixMode.multiline and k <= 0:
        raise CtsmError("InvalidSpec", "multiline ray count must be > 0")
    return _MODE_CODES[mode]


# ---- device context -----------------------------------------------------
class Context:
    """Owns a ctsm_ctx (device status word, scratch buffers) for one GPU."""

    _by_device: dict[int, "Context"] = {}

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().ctsm_create(device, ctypes.byref(h)))
        self.handle = h

    @classmethod
    def get(cls, device: Optional[int] = None) -> "Context":
        if device is None:
            device = torch.cuda.current_device() if torch is not None else 0
        if device not in cls._by_device:
            cls._by_device[device] = Context(device)
        return cls._by_device[device]

    def close(self) -> None:
        if self.handle:
            _lib.lib().ctsm_destroy(self.handle)
            self.handle = None


def _stream(device: int):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev_ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def _dtype_code(t) -> int:
    if t.dtype == torch.float64:
        return _lib.CTSM_F64
    if t.dtype == torch.float32:
        return _lib.CTSM_F32
    raise CtsmError("InvalidSpec", f"unsupported dtype {t.dtype} (float64/float32)")


def _to_device(a, device: int, dtype=None):
    """numpy / tensor -> contiguous CUDA tensor (host arrays are copied)."""
    if torch is not None and isinstance(a, torch.Tensor):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device.type != "cuda":
            t = t.to(f"cuda:{device}")
        return t.contiguous(), True
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if dtype is not None:
        t = t.to(dtype)
    elif t.dtype not in (torch.float64, torch.float32):
        t = t.to(torch.float64)
    return t.to(f"cuda:{device}"), False


def quarter_symmetric(g: ScanGeometry) -> bool:
    """True if the scan is invariant under a quarter turn (square grid with an
    even side, a == b, n_angles % 4 == 0, one full turn): the matrix-free
    kernels then evaluate each weight once for four (voxel, angle) pairs."""
    return bool(_lib.lib().ctsm_quarter_symmetric(ctypes.byref(g.to_c())))


def symmetry_order(g: ScanGeometry) -> int:
    """8 (dihedral: quarter turns and the reflection phi -> -phi, y -> -y;
    scans starting at angle 0 with n_angles % 8 == 0), 4 (quarter turns) or 1: the
    number of (pixel, angle) pairs each weight evaluation of the matrix-free
    kernels serves."""
    return int(_lib.lib().ctsm_symmetry_order(ctypes.byref(g.to_c())))


def _angle_shard(g: ScanGeometry, angles):
    """(begin, end, step) or ("orbits", base_begin, base_step)."""
    if isinstance(angles, tuple) and len(angles) == 3 and angles[0] == "orbits":
        return angles
    if angles is None:
        return 0, g.n_angles, 1
    if isinstance(angles, range):
        step = angles.step
        if step <= 0 or len(angles) == 0:
            raise CtsmError("InvalidSpec", "empty or descending angle range")
        return angles.start, min(g.n_angles, angles.start + step * len(angles)), step
    a0, a1, st = angles
    return int(a0), int(a1), int(st)


# ---- CSR system matrix (K1/K2/K3/K4) --------------------------------------
@dataclass
class SparseSystemMatrix:
    """projector.hpp:26-35. Arrays are CUDA tensors (row_start int64 holding
    u64 values, col int32 holding u32 columns, val float64)."""

    n_rows: int
    n_cols: int
    row_start: "torch.Tensor"
    col: "torch.Tensor"
    val: "torch.Tensor"
    meta: str = ""
    device: int = 0
    row_offset: int = 0  # first global row of this shard (angle sharding)

    def nnz(self) -> int:
        return int(self.col.numel())

    def to_host(self):
        return (self.row_start.cpu().numpy().view(np.uint64), self.col.cpu().numpy().view(np.uint32),
                self.val.cpu().numpy())


def _meta(g: ScanGeometry, mode: str, k: int) -> str:
    # projector.cpp:191-199 (operator<< of doubles uses 6 significant digits)
    def f(v):
        return f"{v:g}"
    return (f"mode={matrix_mode_name(mode, k)}\n"
            f"s={f(g.s)}\nd={f(g.d)}\ndy={f(g.d_y)}\ndz={f(g.d_z)}\nndy={g.n_det_y}\nndz={g.n_det_z}"
            f"\nnp={g.n_angles}\nangle_start={f(g.angle_start)}\nangle_end={f(g.angle_end)}"
            f"\na={f(g.a)}\nb={f(g.b)}\nc={f(g.c)}\nnx={g.n_x}\nny={g.n_y}\nnz={g.n_z}\n")


def build_system_matrix(g: ScanGeometry, mode: str = MatrixMode.consistent, k: int = 1,
                        threads: int = 1, memory_budget_bytes: int = DEFAULT_BUDGET,
                        device: Optional[int] = None, angle_range: Optional[tuple] = None,
                        two_pass: bool = False) -> SparseSystemMatrix:
    """projector.cpp:144-201 on the GPU (K1 2D / K2 3D; line / multiline(k)
    by the device ray tracer, K9). ``threads`` is accepted for API
    compatibility and ignored. ``angle_range=(a0, a1)`` builds one contiguous
    angle shard (rows a0*rpa .. a1*rpa). The consistent matrix is built by
    ``ctsm_csr_build`` (each weight evaluated once); ``two_pass=True`` uses
    the count / fill protocol instead (two evaluations, exact-size arrays)."""
    mc = _mode_code(mode, k)
    g.validate()
    if g.n_voxels > 0xFFFFFFFF:
        raise CtsmError("TooLarge", "grid exceeds 2^32 voxel columns")
    ctx = Context.get(device)
    a0, a1 = (0, g.n_angles) if angle_range is None else angle_range
    n_rows = (a1 - a0) * g.rows_per_angle
    dev = ctx.device
    cg = g.to_c()
    row_start = torch.empty(n_rows + 1, dtype=torch.int64, device=f"cuda:{dev}")
    nnz = ctypes.c_uint64(0)
    st = _stream(dev)
    L = _lib.lib()
    if mc == 0 and not two_pass:
        # single evaluation (ctsm_csr_build): arrays sized from the angle-0
        # estimate; the views keep the (slightly larger) storage alive
        nnz0 = ctypes.c_uint64(0)
        _lib.check(L.ctsm_csr_angle_nnz(ctx.handle, ctypes.byref(cg), 0, ctypes.byref(nnz0), st))
        cap = int(nnz0.value * (a1 - a0) * 1.2) + 65536
        if 12 * nnz0.value * g.n_angles + 8 * (g.n_measurements + 1) > memory_budget_bytes:
            cap = 0  # the call raises OutOfMemory (projector.cpp:155-169)
        for _ in range(2):
            col = torch.empty(cap, dtype=torch.int32, device=f"cuda:{dev}")
            val = torch.empty(cap, dtype=torch.float64, device=f"cuda:{dev}")
            _lib.check(L.ctsm_csr_build(ctx.handle, ctypes.byref(cg), a0, a1, memory_budget_bytes,
                                        _dev_ptr(row_start), _dev_ptr(col), _dev_ptr(val), cap,
                                        ctypes.byref(nnz), st))
            if nnz.value <= cap:
                break
            cap = nnz.value
        return SparseSystemMatrix(n_rows=n_rows, n_cols=g.n_voxels, row_start=row_start,
                                  col=col[:nnz.value], val=val[:nnz.value],
                                  meta=_meta(g, mode, k), device=dev,
                                  row_offset=a0 * g.rows_per_angle)
    _lib.check(L.ctsm_csr_count_mode(ctx.handle, ctypes.byref(cg), mc, k, a0, a1,
                                     memory_budget_bytes, _dev_ptr(row_start),
                                     ctypes.byref(nnz), st))
    col = torch.empty(nnz.value, dtype=torch.int32, device=f"cuda:{dev}")
    val = torch.empty(nnz.value, dtype=torch.float64, device=f"cuda:{dev}")
    _lib.check(L.ctsm_csr_fill_mode(ctx.handle, ctypes.byref(cg), mc, k, a0, a1,
                                    _dev_ptr(row_start), _dev_ptr(col), _dev_ptr(val), st))
    return SparseSystemMatrix(n_rows=n_rows, n_cols=g.n_voxels, row_start=row_start, col=col,
                              val=val, meta=_meta(g, mode, k), device=dev,
                              row_offset=a0 * g.rows_per_angle)


def weights_batch(g: ScanGeometry, ix, iy, iz, phi, cap: int = 256, device: Optional[int] = None):
    """pixel_area_factors (weights2d.hpp:31-32) / voxel_volume_factors
    (weights3d.hpp:90-91) for a batch of (voxel, phi) queries in one device
    launch. Returns (count[n], m_y[n, cap], m_z[n, cap], w[n, cap]) numpy
    arrays; query q's weights are the first count[q] entries of its rows, in
    the reference's order."""
    g.validate()
    ix = np.ascontiguousarray(ix, np.int32)
    n = ix.size
    iy = np.ascontiguousarray(iy, np.int32)
    iz = np.zeros(n, np.int32) if iz is None else np.ascontiguousarray(iz, np.int32)
    phi = np.ascontiguousarray(phi, np.float64)
    if not (iy.size == n and iz.size == n and phi.size == n):
        raise CtsmError("DimensionMismatch", "one (ix, iy, iz, phi) per query is required")
    ctx = Context.get(device)
    cg = g.to_c()
    count = np.zeros(n, np.int32)
    my = np.zeros((n, cap), np.int32)
    mz = np.zeros((n, cap), np.int32)
    w = np.zeros((n, cap), np.float64)
    _lib.check(_lib.lib().ctsm_weights_batch(ctx.handle, ctypes.byref(cg), n, ix.ctypes.data,
                                             iy.ctypes.data, iz.ctypes.data, phi.ctypes.data, cap,
                                             count.ctypes.data, my.ctypes.data, mz.ctypes.data,
                                             w.ctypes.data))
    return count, my, mz, w


def pixel_area_factors(n, phi: float, g: ScanGeometry):
    """weights2d.hpp:31-32: [(m_y, w), ...] of pixel n = (ix, iy) at angle phi."""
    count, my, _, w = weights_batch(g, [n[0]], [n[1]], None, [phi])
    return [(int(my[0, i]), float(w[0, i])) for i in range(count[0])]


def voxel_volume_factors(n, phi: float, g: ScanGeometry):
    """weights3d.hpp:90-91: [(m_y, m_z, w), ...] of voxel n = (ix, iy, iz)."""
    if g.is_2d():
        raise CtsmError("InvalidSpec", "voxel_volume_factors needs a 3D scan")
    count, my, mz, w = weights_batch(g, [n[0]], [n[1]], [n[2]], [phi])
    return [(int(my[0, i]), int(mz[0, i]), float(w[0, i])) for i in range(count[0])]


def angle_block_entries(g: ScanGeometry, mode: str, k: int, angle_index: int,
                        device: Optional[int] = None):
    """detail::angle_block_entries (projector.hpp:72-78): (raster, col, w)
    CUDA tensors of one angle block in the reference's emission order."""
    mc = _mode_code(mode, k)
    g.validate()
    ctx = Context.get(device)
    dev = ctx.device
    cg = g.to_c()
    st = _stream(dev)
    L = _lib.lib()
    cap = ctypes.c_uint64(0)
    if mc == 0:
        _lib.check(L.ctsm_csr_angle_nnz(ctx.handle, ctypes.byref(cg), angle_index,
                                        ctypes.byref(cap), st))
    n = ctypes.c_uint64(0)
    capv = cap.value
    for _ in range(2):
        raster = torch.empty(capv, dtype=torch.int32, device=f"cuda:{dev}")
        col = torch.empty(capv, dtype=torch.int32, device=f"cuda:{dev}")
        w = torch.empty(capv, dtype=torch.float64, device=f"cuda:{dev}")
        _lib.check(L.ctsm_angle_block_entries(ctx.handle, ctypes.byref(cg), mc, k, angle_index,
                                              capv, _dev_ptr(raster), _dev_ptr(col), _dev_ptr(w),
                                              ctypes.byref(n), st))
        if n.value <= capv:
            break
        capv = n.value
    return raster[:n.value], col[:n.value], w[:n.value]


def forward_project(w: SparseSystemMatrix, x):
    """projector.cpp:203-217 (K3)."""
    n = int(x.numel()) if (torch is not None and isinstance(x, torch.Tensor)) else int(np.size(x))
    if n != w.n_cols:
        raise CtsmError("DimensionMismatch", "image size does not match matrix columns")
    ctx = Context.get(w.device)
    xt, was_t = _to_device(x, w.device, torch.float64)
    y = torch.empty(w.n_rows, dtype=torch.float64, device=xt.device)
    _lib.check(_lib.lib().ctsm_spmv(ctx.handle, w.n_rows, w.n_cols, _dev_ptr(w.row_start),
                                    _dev_ptr(w.col), _dev_ptr(w.val), _dev_ptr(xt), _dev_ptr(y),
                                    _stream(w.device)))
    return y if was_t else y.cpu().numpy()


def _colsum_max(w: SparseSystemMatrix) -> float:
    """max_c sum_r |A_rc| (the fixed-point bound of K4), computed once per
    matrix and kept while its arrays are unchanged: the key holds the tensors'
    storage pointers and torch version counters (bumped by every in-place
    torch op); scale_values drops it."""
    key = (w.col.data_ptr(), w.col._version, w.val.data_ptr(), w.val._version,
           w.row_start.data_ptr(), w.row_start._version)
    cached = getattr(w, "_colsum_cache", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    ctx = Context.get(w.device)
    out = ctypes.c_double()
    _lib.check(_lib.lib().ctsm_csr_colsum_max(ctx.handle, w.n_rows, w.n_cols, _dev_ptr(w.row_start),
                                              _dev_ptr(w.col), _dev_ptr(w.val), ctypes.byref(out),
                                              _stream(w.device)))
    w._colsum_cache = (key, out.value)
    return out.value


def _csr_key(w: SparseSystemMatrix):
    return (w.col.data_ptr(), w.col._version, w.val.data_ptr(), w.val._version,
            w.row_start.data_ptr(), w.row_start._version)


def build_transpose(w: SparseSystemMatrix) -> None:
    """Keeps a CSC transpose of the matrix beside the CSR (``ctsm_csc_build``):
    ``back_project`` then gathers (every entry read once) instead of issuing
    one 64-bit reduction per entry, with bit-identical results. Costs the
    CSR's col / val bytes again (C2: 55 GB); dropped when the arrays change."""
    if w.n_rows >= 1 << 32:
        raise CtsmError("TooLarge", "CSC row indices are 32-bit")
    ctx = Context.get(w.device)
    dev = w.val.device
    col_start = torch.empty(w.n_cols + 1, dtype=torch.int64, device=dev)
    row = torch.empty(w.nnz(), dtype=torch.int32, device=dev)
    valt = torch.empty(w.nnz(), dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().ctsm_csc_build(ctx.handle, w.n_rows, w.n_cols, _dev_ptr(w.row_start),
                                         _dev_ptr(w.col), _dev_ptr(w.val), _dev_ptr(col_start),
                                         _dev_ptr(row), _dev_ptr(valt), _stream(w.device)))
    w._csc = (_csr_key(w), col_start, row, valt)


def drop_transpose(w: SparseSystemMatrix) -> None:
    w._csc = None


def back_project(w: SparseSystemMatrix, y):
    """projector.cpp:219-233 (K4): the fixed-point scatter over the CSR, or,
    after ``build_transpose(w)``, the gather over its CSC transpose (same
    bits)."""
    n = int(y.numel()) if (torch is not None and isinstance(y, torch.Tensor)) else int(np.size(y))
    if n != w.n_rows:
        raise CtsmError("DimensionMismatch", "sinogram size does not match matrix rows")
    ctx = Context.get(w.device)
    yt, was_t = _to_device(y, w.device, torch.float64)
    x = torch.empty(w.n_cols, dtype=torch.float64, device=yt.device)
    csc = getattr(w, "_csc", None)
    if csc is not None and csc[0] != _csr_key(w):
        csc = w._csc = None  # the arrays changed under the transpose
    if csc is not None:
        _lib.check(_lib.lib().ctsm_spmv_t_csc(ctx.handle, w.n_rows, w.n_cols, _dev_ptr(csc[1]),
                                              _dev_ptr(csc[2]), _dev_ptr(csc[3]), _colsum_max(w),
                                              _dev_ptr(yt), _dev_ptr(x), _stream(w.device)))
    else:
        _lib.check(_lib.lib().ctsm_spmv_t_bound(ctx.handle, w.n_rows, w.n_cols,
                                                _dev_ptr(w.row_start), _dev_ptr(w.col),
                                                _dev_ptr(w.val), _colsum_max(w), _dev_ptr(yt),
                                                _dev_ptr(x), _stream(w.device)))
    return x if was_t else x.cpu().numpy()


def scale_values(w: SparseSystemMatrix, factor: float) -> None:
    """projector.cpp:282-286 (device kernel)."""
    if not math.isfinite(factor):
        raise CtsmError("NonFinite", "scale factor must be finite")
    ctx = Context.get(w.device)
    w._colsum_cache = None  # values change through the C-ABI, not a torch op
    w._csc = None
    _lib.check(_lib.lib().ctsm_scale_values(ctx.handle, w.nnz(), _dev_ptr(w.val), float(factor),
                                            _stream(ctx.device)))


def csr_operator(w: SparseSystemMatrix):
    """ctsm_operator of a device CSR matrix (solvers)."""
    op = _lib.COperator()
    op.kind = _lib.CTSM_OP_CSR
    op.n_rows, op.n_cols = w.n_rows, w.n_cols
    op.row_start, op.col, op.val = w.row_start.data_ptr(), w.col.data_ptr(), w.val.data_ptr()
    op.scale = 1.0
    csc = getattr(w, "_csc", None)
    if csc is not None and csc[0] == _csr_key(w):  # build_transpose: W^T as a gather
        op.col_start, op.trow, op.tval = csc[1].data_ptr(), csc[2].data_ptr(), csc[3].data_ptr()
    return op, None


def mf_operator(g: ScanGeometry, scale: float = 1.0):
    """ctsm_operator of the fp64 matrix-free projector of a scan, times scale."""
    g.validate()
    cg = g.to_c()
    op = _lib.COperator()
    op.kind = _lib.CTSM_OP_MATRIX_FREE
    op.geom = ctypes.pointer(cg)
    op.scale = float(scale)
    return op, cg  # keep cg alive with op


def _spectral_norm(op, n_cols: int, device: int, iters: int, seed: int) -> float:
    from .phantoms import normal_samples

    ctx = Context.get(device)
    v = torch.from_numpy(normal_samples(n_cols, seed)).to(f"cuda:{ctx.device}")
    out = ctypes.c_double(0.0)
    _lib.check(_lib.lib().ctsm_spectral_norm_power(ctx.handle, ctypes.byref(op), int(iters),
                                                   _dev_ptr(v), ctypes.byref(out),
                                                   _stream(ctx.device)))
    return float(out.value)


def spectral_norm_power(w: SparseSystemMatrix, iters: int = 100, seed: int = 7) -> float:
    """projector.cpp:262-280 on the device (K3/K4 + deterministic reductions);
    the start vector is normal_samples(n_cols, seed) (phantoms.cpp:78-87)."""
    if w.nnz() == 0:
        raise CtsmError("ZeroMatrix", "matrix has no entries")
    op, _keep = csr_operator(w)
    return _spectral_norm(op, w.n_cols, w.device, iters, seed)


def spectral_norm_power_matrix_free(g: ScanGeometry, iters: int = 100, seed: int = 7,
                                    device: Optional[int] = None) -> float:
    """spectral_norm_power on the matrix-free projector (K5/K6): the paper's
    normalisation step for scans whose matrix is too large to store."""
    op, _keep = mf_operator(g)
    return _spectral_norm(op, g.n_voxels, device if device is not None else 0, iters, seed)


# ---- matrix-free projectors (K5/K6) ---------------------------------------
def forward_project_matrix_free(g: ScanGeometry, mode: str = MatrixMode.consistent, k: int = 1,
                                x=None, threads: int = 1, *, angles=None, out=None,
                                device: Optional[int] = None, context: Optional["Context"] = None):
    """projector.cpp:235-260 (K5). ``angles`` = (begin, end, step) restricts the
    projection to an angle shard (rows of other angles are left untouched in
    ``out``, zero in a fresh output); ("orbits", b0, bstep) selects the base
    angles b0 + k bstep < n/4 of a quarter-turn symmetric scan together with
    their quarter-turn images. dtype follows x (float64 / float32). Line /
    multiline(k) modes trace the detector rays on the device (K9)."""
    mc = _mode_code(mode, k)
    g.validate()
    n = int(x.numel()) if (torch is not None and isinstance(x, torch.Tensor)) else int(np.size(x))
    if n != g.n_voxels:
        raise CtsmError("DimensionMismatch", "image size does not match the grid")
    # context: an explicit Context (own scratch and status word) lets two
    # host threads or two streams run projections concurrently
    ctx = context if context is not None else Context.get(
        device if device is not None else
        (x.device.index if (torch is not None and isinstance(x, torch.Tensor) and x.is_cuda) else None))
    xt, was_t = _to_device(x, ctx.device)
    sh = _angle_shard(g, angles)
    y = out if out is not None else torch.zeros(g.n_measurements, dtype=xt.dtype, device=xt.device)
    cg = g.to_c()
    if sh[0] == "orbits":
        if mc != 0:
            raise CtsmError("InvalidSpec", "orbit shards exist for the consistent mode only")
        _lib.check(_lib.lib().ctsm_fwd_mf_orbits(ctx.handle, ctypes.byref(cg), _dtype_code(xt),
                                                 sh[1], sh[2], _dev_ptr(xt), _dev_ptr(y),
                                                 _stream(ctx.device)))
    else:
        a0, a1, st = sh
        _lib.check(_lib.lib().ctsm_fwd_mf_mode(ctx.handle, ctypes.byref(cg), mc, k,
                                               _dtype_code(xt), a0, a1, st, _dev_ptr(xt),
                                               _dev_ptr(y), _stream(ctx.device)))
    return y if (was_t or out is not None) else y.cpu().numpy()


def back_project_matrix_free(g: ScanGeometry, mode: str = MatrixMode.consistent, k: int = 1,
                             y=None, threads: int = 1, *, angles=None, out=None,
                             device: Optional[int] = None, context: Optional["Context"] = None):
    """Matrix-free A^T y (K6; the reference only has CSR back_project,
    projector.cpp:219-233). With ``angles`` the result is the partial volume
    of that angle shard (summed across ranks by the multi-GPU driver)."""
    mc = _mode_code(mode, k)
    g.validate()
    n = int(y.numel()) if (torch is not None and isinstance(y, torch.Tensor)) else int(np.size(y))
    if n != g.n_measurements:
        raise CtsmError("DimensionMismatch", "sinogram size does not match the scan")
    ctx = context if context is not None else Context.get(
        device if device is not None else
        (y.device.index if (torch is not None and isinstance(y, torch.Tensor) and y.is_cuda) else None))
    yt, was_t = _to_device(y, ctx.device)
    sh = _angle_shard(g, angles)
    x = out if out is not None else torch.empty(g.n_voxels, dtype=yt.dtype, device=yt.device)
    cg = g.to_c()
    if sh[0] == "orbits":
        if mc != 0:
            raise CtsmError("InvalidSpec", "orbit shards exist for the consistent mode only")
        _lib.check(_lib.lib().ctsm_bwd_mf_orbits(ctx.handle, ctypes.byref(cg), _dtype_code(yt),
                                                 sh[1], sh[2], _dev_ptr(yt), _dev_ptr(x),
                                                 _stream(ctx.device)))
    else:
        a0, a1, st = sh
        _lib.check(_lib.lib().ctsm_bwd_mf_mode(ctx.handle, ctypes.byref(cg), mc, k,
                                               _dtype_code(yt), a0, a1, st, _dev_ptr(yt),
                                               _dev_ptr(x), _stream(ctx.device)))
    return x if (was_t or out is not None) else x.cpu().numpy()


def last_kernel_path(context: Optional["Context"] = None, device: Optional[int] = None) -> int:
    """CTSM_PATH_* bits of the last matrix-free call on a context
    (include/ctsm_b200.h): 1 general, 4 quarter-turn, 8 dihedral, +16 z mirror,
    +32 fp32 vector-reduction forward."""
    ctx = context if context is not None else Context.get(device)
    return int(_lib.lib().ctsm_last_kernel_path(ctx.handle))


def angle_column_sums(g: ScanGeometry, mode: str = MatrixMode.consistent, k: int = 1,
                      angle_index: int = 0, device: Optional[int] = None):
    """projector.cpp:288-295: per-voxel sums of one angle block (A^T 1 on one angle)."""
    _mode_code(mode, k)
    ctx = Context.get(device)
    ones = torch.ones(g.n_measurements, dtype=torch.float64, device=f"cuda:{ctx.device}")
    return back_project_matrix_free(g, mode, k, ones, angles=(angle_index, angle_index + 1, 1),
                                    device=ctx.device).cpu().numpy()


def sirt(g: ScanGeometry, y, x0=None, iters: int = 10, device: Optional[int] = None):
    """SIRT (BASELINE.json configs[4]): x <- x + C A^T (R (y - A x)),
    R = 1/(A 1), C = 1/(A^T 1) (zero sums -> 0). Single device."""
    g.validate()
    ctx = Context.get(device)
    yt, was_t = _to_device(y, ctx.device)
    if x0 is None:
        x = torch.zeros(g.n_voxels, dtype=yt.dtype, device=yt.device)
    else:
        x, _ = _to_device(x0, ctx.device, yt.dtype)
        x = x.clone()
    cg = g.to_c()
    _lib.check(_lib.lib().ctsm_sirt(ctx.handle, ctypes.byref(cg), _dtype_code(yt), _dev_ptr(yt),
                                    _dev_ptr(x), iters, _stream(ctx.device)))
    return x if was_t else x.cpu().numpy()
