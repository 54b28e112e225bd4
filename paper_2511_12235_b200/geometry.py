"""ScanGeometry and the BASELINE configurations (host side).

``ScanGeometry`` mirrors the reference's ``ctsm::ScanGeometry``
(/root/reference/proj/include/ctsm/geometry.hpp:29-64): same fields, defaults,
angle formula (geometry.hpp:50-52), face positions (53-55), column/row raster
maps (76-84) and ``validate()`` rules (geometry.cpp:27-54). The C-ABI mirror is
``ctsm_geometry`` in include/ctsm_b200.h.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace

K_PI = 3.14159265358979323846


class CtsmError(RuntimeError):
    """Raised for every failure; ``code`` is the reference ErrorCode name
    (common.hpp:11-25)."""

    NAMES = [
        "DegenerateGeometry", "RayParallelToFace", "SingularPhi", "CentralRow",
        "ZRestrictionViolation", "DimensionMismatch", "NonFinite", "ZeroMatrix", "TooLarge",
        "InvalidSpec", "OutOfMemory", "InvalidConfig", "IoFailure",
    ]

    def __init__(self, code: str, message: str):
        self.code = code
        super().__init__(f"{code}: {message}")

    @classmethod
    def from_status(cls, status: int, message: str) -> "CtsmError":
        idx = status - 1
        name = cls.NAMES[idx] if 0 <= idx < len(cls.NAMES) else f"Status{status}"
        return cls(name, message)


class CGeometry(ctypes.Structure):
    """``ctsm_geometry`` (include/ctsm_b200.h)."""

    _fields_ = [
        ("s", ctypes.c_double), ("d", ctypes.c_double), ("d_y", ctypes.c_double),
        ("d_z", ctypes.c_double), ("n_det_y", ctypes.c_int32), ("n_det_z", ctypes.c_int32),
        ("n_angles", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("angle_start", ctypes.c_double), ("angle_end", ctypes.c_double),
        ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
        ("n_x", ctypes.c_int32), ("n_y", ctypes.c_int32), ("n_z", ctypes.c_int32),
        ("pad1", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class ScanGeometry:
    s: float = 0.0
    d: float = 0.0
    d_y: float = 1.0
    d_z: float = 1.0
    n_det_y: int = 0
    n_det_z: int = 1
    n_angles: int = 0
    angle_start: float = 0.0
    angle_end: float = 2.0 * K_PI
    a: float = 1.0
    b: float = 1.0
    c: float = 1.0
    n_x: int = 0
    n_y: int = 0
    n_z: int = 1

    # geometry.hpp:46-63
    def is_2d(self) -> bool:
        return self.n_z == 1 and self.n_det_z == 1

    def sdd(self) -> float:
        return self.s + self.d

    def angle(self, i: int) -> float:
        return self.angle_start + (self.angle_end - self.angle_start) * i / self.n_angles

    @property
    def n_voxels(self) -> int:
        return self.n_x * self.n_y * self.n_z

    @property
    def rows_per_angle(self) -> int:
        return self.n_det_y * self.n_det_z

    @property
    def n_measurements(self) -> int:
        return self.n_angles * self.n_det_y * self.n_det_z

    def voxel_column(self, ix: int, iy: int, iz: int = 0) -> int:
        return (iz * self.n_y + iy) * self.n_x + ix

    def measurement_row(self, ip: int, m_y: int, m_z: int = 0) -> int:
        raster = (m_z + self.n_det_z // 2) * self.n_det_y + (m_y + self.n_det_y // 2)
        return ip * self.n_det_y * self.n_det_z + raster

    def validate(self) -> None:
        """geometry.cpp:27-54."""
        if not (self.s > 0.0):
            raise CtsmError("InvalidSpec", "source distance s must be > 0")
        if not (self.d >= 0.0):
            raise CtsmError("InvalidSpec", "detector distance d must be >= 0")
        if not (self.d_y > 0.0) or not (self.d_z > 0.0):
            raise CtsmError("InvalidSpec", "detector pitches must be > 0")
        if self.n_det_y <= 0 or self.n_det_z <= 0 or self.n_angles <= 0:
            raise CtsmError("InvalidSpec", "detector and angle counts must be > 0")
        if self.n_det_y % 2 != 0:
            raise CtsmError("InvalidSpec", "n_det_y must be even (centered detector)")
        if self.n_det_z != 1 and self.n_det_z % 2 != 0:
            raise CtsmError("InvalidSpec", "n_det_z must be 1 (2D) or even (centered detector)")
        if not (self.a > 0.0) or not (self.b > 0.0) or not (self.c > 0.0):
            raise CtsmError("InvalidSpec", "voxel sizes must be > 0")
        if self.n_x <= 0 or self.n_y <= 0 or self.n_z <= 0:
            raise CtsmError("InvalidSpec", "grid dimensions must be > 0")
        if self.n_det_z == 1 and self.n_z > 1:
            raise CtsmError("InvalidSpec", "volume grid requires n_det_z > 1")
        if not (self.angle_end > self.angle_start):
            raise CtsmError("InvalidSpec", "angle_end must exceed angle_start")
        for v in (self.s, self.d, self.d_y, self.d_z, self.a, self.b, self.c,
                  self.angle_start, self.angle_end):
            if not math.isfinite(v):
                raise CtsmError("NonFinite", "geometry parameters must be finite")
        rx, ry = self.n_x * self.a / 2.0, self.n_y * self.b / 2.0
        if self.s <= math.hypot(rx, ry):
            raise CtsmError("DegenerateGeometry", "source circle intersects the grid")

    def to_c(self) -> CGeometry:
        g = CGeometry()
        for name, _ in CGeometry._fields_:
            if not name.startswith("pad"):
                setattr(g, name, getattr(self, name))
        return g

    def with_(self, **kw) -> "ScanGeometry":
        return replace(self, **kw)


# ---- BASELINE.json configs (SURVEY.md §8(d) geometry mapping) -------------
# "source-to-isocentre 500" -> s = 500; "source-to-detector 1000" -> d = 500
# (d is origin-to-detector, sdd = s + d, geometry.hpp:30-31); angles over
# [0, 2pi) -> the defaults; 3D detector "W x H" -> n_det_y = W, n_det_z = H.
CONFIGS = {
    "c0": ScanGeometry(s=500.0, d=500.0, d_y=1.2, n_det_y=256, n_angles=360,
                       a=1.0, b=1.0, n_x=128, n_y=128),
    "c1": ScanGeometry(s=500.0, d=500.0, d_y=0.6, n_det_y=1024, n_angles=720,
                       a=0.5, b=0.5, n_x=512, n_y=512),
    "c2": ScanGeometry(s=500.0, d=500.0, d_y=1.6, d_z=1.6, n_det_y=256, n_det_z=256,
                       n_angles=360, a=1.0, b=1.0, c=1.0, n_x=128, n_y=128, n_z=128),
    "c3": ScanGeometry(s=500.0, d=500.0, d_y=0.8, d_z=0.8, n_det_y=512, n_det_z=384,
                       n_angles=720, a=0.5, b=0.5, c=0.5, n_x=256, n_y=256, n_z=256),
    "c4": ScanGeometry(s=500.0, d=500.0, d_y=0.4, d_z=0.4, n_det_y=1024, n_det_z=768,
                       n_angles=1440, a=0.25, b=0.25, c=0.25, n_x=512, n_y=512, n_z=512),
}

# Small geometries used by the reference's own unit tests.
TEST_GEOMETRIES = {
    # test_projector.cpp:15-32
    "proj2d": ScanGeometry(s=250, d=250, d_y=1.5, n_det_y=44, n_angles=6, a=1.5, b=1.5,
                           n_x=12, n_y=12),
    "proj3d": ScanGeometry(s=250, d=250, d_y=1.5, d_z=1.5, n_det_y=44, n_det_z=12, n_angles=6,
                           a=1.5, b=1.5, c=1.5, n_x=12, n_y=12, n_z=12),
    # test_weights2d.cpp:15-26
    "wide2d": ScanGeometry(s=250, d=250, d_y=2.0, n_det_y=200, n_angles=8, a=2.5, b=2.5,
                           n_x=12, n_y=12),
    # test_weights3d.cpp:17-30
    "cone3d": ScanGeometry(s=300, d=150, d_y=2.5, d_z=1.5, n_det_y=200, n_det_z=160, n_angles=8,
                           a=5.0, b=5.0, c=5.0, n_x=6, n_y=6, n_z=6),
}
