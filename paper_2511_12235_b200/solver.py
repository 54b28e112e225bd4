"""Reconstruction solver on the device.

Mirrors the reference's solver API (include/ctsm/solver.hpp:10-35,
src/solver.cpp:17-75): Nesterov-accelerated gradient for
0.5 ||W u - p||^2 + 0.5 lambda ||u||^2 with the fixed step 1 / (1 + lambda),
W scaled to unit spectral norm beforehand (scale_values /
spectral_norm_power). The iteration runs in the C-ABI (ctsm_nag_tikhonov) on
the K3/K4 CSR appliers or the K5/K6 matrix-free projectors; vectors stay on
the device, reductions are fixed-order (deterministic).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .geometry import CtsmError, ScanGeometry
from .projector import (Context, SparseSystemMatrix, _dev_ptr, _stream, _to_device, csr_operator,
                        mf_operator)

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


@dataclass
class SolveOptions:
    """solver.hpp:10-14."""
    lam: float = 1e-4   # Tikhonov weight ("lambda")
    max_iter: int = 1000
    tol: float = 1e-9   # stop when the squared gradient norm drops below this


@dataclass
class SolveTraceRow:
    """solver.hpp:16-20."""
    iter: int
    objective: float      # 0.5 ||W u - p||^2 + 0.5 lambda ||u||^2
    grad_norm_sq: float   # ||W^T (W u - p) + lambda u||^2


@dataclass
class SolveResult:
    """solver.hpp:22-27; u is a CUDA float64 tensor."""
    u: "torch.Tensor"
    iterations: int = 0
    converged: bool = False
    trace: List[SolveTraceRow] = field(default_factory=list)


def _solve(op, n_rows: int, n_cols: int, device: int, p, opt: SolveOptions,
           keep_trace: bool) -> SolveResult:
    ctx = Context.get(device)
    pt, _ = _to_device(p, ctx.device, torch.float64)
    if pt.numel() != n_rows:
        raise CtsmError("DimensionMismatch", "data size does not match matrix rows")
    u = torch.empty(n_cols, dtype=torch.float64, device=pt.device)
    trace = np.zeros(3 * max(opt.max_iter, 1)) if keep_trace else None
    its, conv = ctypes.c_int(0), ctypes.c_int(0)
    tptr = trace.ctypes.data_as(ctypes.c_void_p) if keep_trace else None
    _lib.check(_lib.lib().ctsm_nag_tikhonov(ctx.handle, ctypes.byref(op), _dev_ptr(pt),
                                            float(opt.lam), int(opt.max_iter), float(opt.tol),
                                            _dev_ptr(u), tptr, ctypes.byref(its),
                                            ctypes.byref(conv), _stream(ctx.device)))
    rows = []
    if keep_trace:
        for i in range(its.value):
            rows.append(SolveTraceRow(int(trace[3 * i]), float(trace[3 * i + 1]),
                                      float(trace[3 * i + 2])))
    return SolveResult(u=u, iterations=its.value, converged=bool(conv.value), trace=rows)


def nag_tikhonov(w: SparseSystemMatrix, p, opt: Optional[SolveOptions] = None,
                 keep_trace: bool = False) -> SolveResult:
    """solver.cpp:17-75 on a device CSR matrix."""
    opt = opt or SolveOptions()
    op, _keep = csr_operator(w)
    return _solve(op, w.n_rows, w.n_cols, w.device, p, opt, keep_trace)


def nag_tikhonov_matrix_free(g: ScanGeometry, p, opt: Optional[SolveOptions] = None,
                             keep_trace: bool = False, scale: float = 1.0,
                             device: Optional[int] = None) -> SolveResult:
    """The same iteration on W = scale * A with A the fp64 matrix-free
    projector (scale = 1 / spectral_norm_power_matrix_free(g) normalises W)."""
    opt = opt or SolveOptions()
    op, _keep = mf_operator(g, scale)
    return _solve(op, g.n_measurements, g.n_voxels, device if device is not None else 0, p, opt,
                  keep_trace)
