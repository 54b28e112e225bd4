"""The reference's independent numerical oracles (oracle.hpp:24-45) on the
device: Monte-Carlo volume fractions and Gauss-Legendre ray-bundle integrals
for batches of (voxel box, detector cell) cases. They
share no code with the closed-form weights and scale the 3D oracle suite
(validate.cpp:167-293) to many cases per launch."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .geometry import ScanGeometry
from .projector import Context


@dataclass
class McEstimate:  # oracle.hpp:24-27
    value: float = 0.0
    std_err: float = 0.0


def voxel_box(g: ScanGeometry, ix: int, iy: int, iz: int) -> np.ndarray:
    """{x0, x1, y0, y1, zb, zt} of voxel (ix, iy, iz) (geometry.hpp:53-55)."""
    return np.array([(ix - g.n_x / 2.0) * g.a, (ix + 1 - g.n_x / 2.0) * g.a,
                     (iy - g.n_y / 2.0) * g.b, (iy + 1 - g.n_y / 2.0) * g.b,
                     (iz - g.n_z / 2.0) * g.c, (iz + 1 - g.n_z / 2.0) * g.c], np.float64)


def _cases(boxes, phi, m_y, m_z):
    boxes = np.ascontiguousarray(boxes, np.float64).reshape(-1, 6)
    n = boxes.shape[0]
    phi = np.ascontiguousarray(np.broadcast_to(np.asarray(phi, np.float64), (n,)))
    m_y = np.ascontiguousarray(np.broadcast_to(np.asarray(m_y, np.int32), (n,)))
    m_z = np.ascontiguousarray(np.broadcast_to(np.asarray(m_z, np.int32), (n,)))
    return n, boxes, phi, m_y, m_z


def mc_volume_3d_batch(boxes, phi, s: float, d: float, d_y: float, d_z: float, m_y, m_z,
                       n_samples: int, seed: int, device: Optional[int] = None):
    """(value[n], std_err[n], hits[n]) of mc_volume_3d (oracle.cpp:70-98) for n cases."""
    n, boxes, phi, m_y, m_z = _cases(boxes, phi, m_y, m_z)
    ctx = Context.get(device)
    value = np.zeros(n, np.float64)
    se = np.zeros(n, np.float64)
    hits = np.zeros(n, np.uint64)
    _lib.check(_lib.lib().ctsm_mc_volume_3d(ctx.handle, n, boxes.ctypes.data, phi.ctypes.data, s, d,
                                            d_y, d_z, m_y.ctypes.data, m_z.ctypes.data, n_samples,
                                            seed, value.ctypes.data, se.ctypes.data,
                                            hits.ctypes.data))
    return value, se, hits


def mc_volume_3d(x0, x1, y0, y1, zb, zt, phi, s, d, d_y, d_z, m_y, m_z, n_samples, seed) -> McEstimate:
    """oracle.hpp:32-35 (one case)."""
    v, se, _ = mc_volume_3d_batch([[x0, x1, y0, y1, zb, zt]], phi, s, d, d_y, d_z, m_y, m_z,
                                  n_samples, seed)
    return McEstimate(float(v[0]), float(se[0]))


def multiline_volume_3d_batch(boxes, phi, s: float, d: float, d_y: float, d_z: float, m_y, m_z,
                              k: int = 200, device: Optional[int] = None) -> np.ndarray:
    """multiline_volume_3d (oracle.cpp:124-196) for n cases."""
    n, boxes, phi, m_y, m_z = _cases(boxes, phi, m_y, m_z)
    ctx = Context.get(device)
    out = np.zeros(n, np.float64)
    _lib.check(_lib.lib().ctsm_multiline_volume_3d(ctx.handle, n, boxes.ctypes.data, phi.ctypes.data,
                                                   s, d, d_y, d_z, m_y.ctypes.data, m_z.ctypes.data,
                                                   k, out.ctypes.data))
    return out


def multiline_volume_3d(x0, x1, y0, y1, zb, zt, phi, s, d, d_y, d_z, m_y, m_z, k: int = 200) -> float:
    """oracle.hpp:40-43 (one case)."""
    return float(multiline_volume_3d_batch([[x0, x1, y0, y1, zb, zt]], phi, s, d, d_y, d_z, m_y,
                                           m_z, k)[0])


def gauss_legendre(k: int):
    """oracle.hpp:45: nodes and weights on [-1, 1] (host; oracle.cpp:100-122)."""
    x = np.zeros(k, np.float64)
    w = np.zeros(k, np.float64)
    _lib.lib().ctsm_gauss_legendre(k, x.ctypes.data, w.ctypes.data)
    return x, w
