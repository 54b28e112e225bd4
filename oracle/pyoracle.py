"""ctypes front-end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module. The product (paper_2511_12235_b200) never does.

Four interchangeable libraries export the same ``ref_*`` C-ABI
(oracle/ref_shim.cpp == oracle/ctsm_oracle.h):

=========  =================================================================
variant    library
=========  =================================================================
ref_glibc  oracle/_ref/libctsm_ref_glibc.so  unmodified reference + glibc libm
ref_cr     oracle/_ref/libctsm_ref_cr.so     unmodified reference + crmath libm
port_glibc oracle/_build/libctsm_oracle_glibc.so  C restatement + glibc libm
port_cr    oracle/_build/libctsm_oracle_cr.so     C restatement + crmath libm
=========  =================================================================

``ref_*`` exist only where /root/reference was present at build time (they are
prebuilt here and travel to the GPU box with the snapshot).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

LIBS = {
    "ref_glibc": os.path.join(HERE, "_ref", "libctsm_ref_glibc.so"),
    "ref_cr": os.path.join(HERE, "_ref", "libctsm_ref_cr.so"),
    "port_glibc": os.path.join(HERE, "_build", "libctsm_oracle_glibc.so"),
    "port_cr": os.path.join(HERE, "_build", "libctsm_oracle_cr.so"),
}

ERROR_NAMES = [
    "DegenerateGeometry", "RayParallelToFace", "SingularPhi", "CentralRow",
    "ZRestrictionViolation", "DimensionMismatch", "NonFinite", "ZeroMatrix", "TooLarge",
    "InvalidSpec", "OutOfMemory", "InvalidConfig", "IoFailure",
]


# MatrixMode ordinals (projector.hpp:12-16)
MODES = {"consistent": 0, "line": 1, "multiline": 2}


class OGeom(ctypes.Structure):
    """Mirror of ScanGeometry (geometry.hpp:29-44) == ctsm_geometry."""

    _fields_ = [
        ("s", ctypes.c_double), ("d", ctypes.c_double), ("d_y", ctypes.c_double),
        ("d_z", ctypes.c_double), ("n_det_y", ctypes.c_int32), ("n_det_z", ctypes.c_int32),
        ("n_angles", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("angle_start", ctypes.c_double), ("angle_end", ctypes.c_double),
        ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
        ("n_x", ctypes.c_int32), ("n_y", ctypes.c_int32), ("n_z", ctypes.c_int32),
        ("pad1", ctypes.c_int32),
    ]


def to_ogeom(g) -> OGeom:
    o = OGeom()
    for name, _ in OGeom._fields_:
        if name.startswith("pad"):
            continue
        setattr(o, name, getattr(g, name))
    return o


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = ERROR_NAMES[code] if 0 <= code < len(ERROR_NAMES) else f"code{code}"
        super().__init__(msg)


_P = ctypes.c_void_p
_cache: dict[str, "Oracle"] = {}


def available(variant: str) -> bool:
    return os.path.exists(LIBS[variant])


def load(variant: str = "port_cr") -> "Oracle":
    if variant not in _cache:
        _cache[variant] = Oracle(variant)
    return _cache[variant]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


@dataclass
class Csr:
    row_start: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col.size)


class Oracle:
    def __init__(self, variant: str):
        path = LIBS[variant]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run `make -C oracle`)")
        self.variant = variant
        L = self.lib = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_validate.argtypes = [_P]
        L.ref_angle.argtypes = [_P, ctypes.c_int]
        L.ref_angle.restype = ctypes.c_double
        L.ref_pixel_area_factors.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_double, _P, _P, ctypes.c_long]
        L.ref_pixel_area_factors.restype = ctypes.c_long
        L.ref_voxel_volume_factors.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, _P, _P, _P, ctypes.c_long]
        L.ref_voxel_volume_factors.restype = ctypes.c_long
        L.ref_angle_block_entries.argtypes = [_P, ctypes.c_int, _P, _P, _P, ctypes.c_long]
        L.ref_angle_block_entries.restype = ctypes.c_long
        L.ref_build_system_matrix.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int)]
        L.ref_build_system_matrix.restype = _P
        L.ref_csr_nnz.argtypes = [_P]
        L.ref_csr_nnz.restype = ctypes.c_uint64
        L.ref_csr_rows.argtypes = [_P]
        L.ref_csr_rows.restype = ctypes.c_uint64
        L.ref_csr_copy.argtypes = [_P, _P, _P, _P]
        L.ref_csr_free.argtypes = [_P]
        for f in ("ref_forward_project", "ref_back_project"):
            getattr(L, f).argtypes = [_P, _P, _P]
        L.ref_forward_project_matrix_free.argtypes = [_P, _P, _P, ctypes.c_int]
        L.ref_back_project_matrix_free.argtypes = [_P, _P, _P, ctypes.c_int]
        L.ref_forward_mf_angles.argtypes = [_P, _P, ctypes.c_int, _P, _P, ctypes.c_int]
        L.ref_back_mf_angles.argtypes = [_P, _P, ctypes.c_int, _P, _P, ctypes.c_int]
        L.ref_sirt.argtypes = [_P, _P, _P, ctypes.c_int, ctypes.c_int]
        self.has_par = hasattr(L, "ref_forward_mf_angles_par")
        if self.has_par:
            L.ref_forward_mf_angles_par.argtypes = [_P, _P, ctypes.c_int, _P, _P, ctypes.c_int]
            L.ref_back_mf_angles_par.argtypes = [_P, _P, ctypes.c_int, _P, _P, ctypes.c_int]
        # slab-parallel angle blocks: the restatement, and the reference's own
        # voxel_volume_factors / pixel_area_factors per slab (ref_shim.cpp)
        self.has_numeric = hasattr(L, "ref_mc_volume_3d")
        if self.has_numeric:
            L.ref_mc_volume_3d.argtypes = [_P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _P]
            L.ref_mc_volume_3d.restype = ctypes.c_uint64
            L.ref_gauss_legendre.argtypes = [ctypes.c_int, _P, _P]
            L.ref_gauss_legendre.restype = None
            L.ref_multiline_volume_3d.argtypes = [_P, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                  ctypes.c_int, ctypes.c_int, ctypes.c_int]
            L.ref_multiline_volume_3d.restype = ctypes.c_double
        self.has_entries_par = hasattr(L, "ref_angle_block_entries_par")
        if self.has_entries_par:
            L.ref_angle_block_entries_par.argtypes = [_P, ctypes.c_int, _P, _P, _P, ctypes.c_long,
                                                      ctypes.c_int]
            L.ref_angle_block_entries_par.restype = ctypes.c_long
        self.has_slabs = hasattr(L, "ref_forward_mf_angles_slabs")
        if self.has_slabs:
            L.ref_forward_mf_angles_slabs.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_int, _P, _P, ctypes.c_int]
            L.ref_back_mf_angles_slabs.argtypes = [_P, _P, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, _P, _P, ctypes.c_int]
        # bounded samples for bench.py's reference arm (ref_* variants only)
        self.has_pair_sample = hasattr(L, "ref_mf_pair_sample")
        if self.has_pair_sample:
            L.ref_mf_pair_sample.argtypes = [_P, _P, ctypes.c_int, _P, ctypes.c_int, _P, _P, _P, _P,
                                             ctypes.c_int]
            L.ref_csr_angle_sample.argtypes = [_P, _P, ctypes.c_int, _P, ctypes.c_int]
        L.ref_angle_column_sums.argtypes = [_P, ctypes.c_int, _P]
        L.ref_line_weights.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, _P, _P, ctypes.c_long]
        L.ref_line_weights.restype = ctypes.c_long
        L.ref_build_system_matrix_mode.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_uint64, ctypes.POINTER(ctypes.c_int)]
        L.ref_build_system_matrix_mode.restype = _P
        L.ref_angle_block_entries_mode.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   _P, _P, _P, ctypes.c_long]
        L.ref_angle_block_entries_mode.restype = ctypes.c_long
        L.ref_forward_mf_mode.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_int]
        L.ref_back_mf_mode.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_int]
        # reference-only entry points (solver / io / phantoms), absent in the ports
        self.has_solver = hasattr(L, "ref_nag_tikhonov")
        if self.has_solver:
            L.ref_spectral_norm_power.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, _P]
            L.ref_scale_values.argtypes = [_P, ctypes.c_double]
            L.ref_nag_tikhonov.argtypes = [_P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                           _P, _P, _P, _P]
            L.ref_write_matrix.argtypes = [_P, ctypes.c_char_p]
            L.ref_read_matrix.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)]
            L.ref_read_matrix.restype = _P
            L.ref_csr_cols.argtypes = [_P]
            L.ref_csr_cols.restype = ctypes.c_uint64
            L.ref_csr_meta.argtypes = [_P, _P, ctypes.c_uint64]
            L.ref_csr_meta.restype = ctypes.c_uint64
            L.ref_write_tensor.argtypes = [ctypes.c_char_p, _P, ctypes.c_int, _P]
            L.ref_normal_samples.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _P]

    # -- helpers -----------------------------------------------------------
    def _check(self, st: int):
        if st < 0:
            code = -st - 1
            raise OracleError(code, self.lib.ref_last_error().decode())

    @staticmethod
    def _g(g):
        og = to_ogeom(g)
        return og, ctypes.byref(og)

    # -- API ---------------------------------------------------------------
    def validate(self, g):
        og, p = self._g(g)
        self._check(self.lib.ref_validate(p))

    def angle(self, g, i: int) -> float:
        og, p = self._g(g)
        return self.lib.ref_angle(p, i)

    def pixel_area_factors(self, g, ix: int, iy: int, phi: float):
        og, p = self._g(g)
        my = np.zeros(256, np.int32)
        w = np.zeros(256, np.float64)
        n = self.lib.ref_pixel_area_factors(p, ix, iy, phi, _ptr(my), _ptr(w), 256)
        self._check(n)
        return my[:n].copy(), w[:n].copy()

    def voxel_volume_factors(self, g, ix: int, iy: int, iz: int, phi: float):
        og, p = self._g(g)
        my = np.zeros(256, np.int32)
        mz = np.zeros(256, np.int32)
        w = np.zeros(256, np.float64)
        n = self.lib.ref_voxel_volume_factors(p, ix, iy, iz, phi, _ptr(my), _ptr(mz), _ptr(w), 256)
        self._check(n)
        return my[:n].copy(), mz[:n].copy(), w[:n].copy()

    # -- independent numerical oracles (oracle.cpp:70-196; restatement only) --
    @staticmethod
    def voxel_box(g, ix: int, iy: int, iz: int) -> np.ndarray:
        return np.array([(ix - g.n_x / 2.0) * g.a, (ix + 1 - g.n_x / 2.0) * g.a,
                         (iy - g.n_y / 2.0) * g.b, (iy + 1 - g.n_y / 2.0) * g.b,
                         (iz - g.n_z / 2.0) * g.c, (iz + 1 - g.n_z / 2.0) * g.c], np.float64)

    def mc_volume_3d(self, g, box, phi: float, m_y: int, m_z: int, n_samples: int, seed: int):
        """(value, std_err, hits) of oracle.cpp:70-98."""
        box = np.ascontiguousarray(box, np.float64)
        out = np.zeros(2, np.float64)
        hits = self.lib.ref_mc_volume_3d(_ptr(box), phi, g.s, g.d, g.d_y, g.d_z, m_y, m_z,
                                         n_samples, seed, _ptr(out))
        return float(out[0]), float(out[1]), int(hits)

    def gauss_legendre(self, k: int):
        x = np.zeros(k, np.float64)
        w = np.zeros(k, np.float64)
        self.lib.ref_gauss_legendre(k, _ptr(x), _ptr(w))
        return x, w

    def multiline_volume_3d(self, g, box, phi: float, m_y: int, m_z: int, k: int = 200) -> float:
        box = np.ascontiguousarray(box, np.float64)
        return float(self.lib.ref_multiline_volume_3d(_ptr(box), phi, g.s, g.d, g.d_y, g.d_z, m_y,
                                                      m_z, k))

    def angle_block_entries(self, g, ip: int, threads: int = 1, mode: str = "consistent",
                            k: int = 1):
        """(row_raster u32, col u32, w f64) in emission order (projector.cpp:44-84).
        threads > 1 (restatement only) computes slabs in parallel; the result is
        identical."""
        og, p = self._g(g)
        if mode != "consistent":
            f = self.lib.ref_angle_block_entries_mode
            n = f(p, MODES[mode], k, ip, None, None, None, 0)
            self._check(n)
            row = np.empty(n, np.uint32)
            col = np.empty(n, np.uint32)
            w = np.empty(n, np.float64)
            self._check(f(p, MODES[mode], k, ip, _ptr(row), _ptr(col), _ptr(w), n))
            return row, col, w
        if threads > 1 and self.has_entries_par:
            f = self.lib.ref_angle_block_entries_par
            n = int(1.3 * 12 * g.n_x * g.n_y * g.n_z) + 1024
            for _ in range(2):
                row = np.empty(n, np.uint32)
                col = np.empty(n, np.uint32)
                w = np.empty(n, np.float64)
                m = f(p, ip, _ptr(row), _ptr(col), _ptr(w), n, threads)
                self._check(m)
                if m <= n:
                    return row[:m].copy(), col[:m].copy(), w[:m].copy()
                n = m
        n = self.lib.ref_angle_block_entries(p, ip, None, None, None, 0)
        self._check(n)
        row = np.empty(n, np.uint32)
        col = np.empty(n, np.uint32)
        w = np.empty(n, np.float64)
        n2 = self.lib.ref_angle_block_entries(p, ip, _ptr(row), _ptr(col), _ptr(w), n)
        self._check(n2)
        return row, col, w

    def build_system_matrix(self, g, threads: int = 1, budget: int = 5 << 30,
                            mode: str = "consistent", k: int = 1) -> Csr:
        og, p = self._g(g)
        st = ctypes.c_int(0)
        h = self.lib.ref_build_system_matrix_mode(p, MODES[mode], k, threads, budget,
                                                  ctypes.byref(st))
        self._check(st.value)
        try:
            nnz = self.lib.ref_csr_nnz(h)
            rows = self.lib.ref_csr_rows(h)
            rs = np.empty(rows + 1, np.uint64)
            col = np.empty(nnz, np.uint32)
            val = np.empty(nnz, np.float64)
            self.lib.ref_csr_copy(h, _ptr(rs), _ptr(col), _ptr(val))
        finally:
            self.lib.ref_csr_free(h)
        return Csr(rs, col, val)

    def forward_project_matrix_free(self, g, x: np.ndarray, threads: int = 1,
                                    mode: str = "consistent", k: int = 1) -> np.ndarray:
        og, p = self._g(g)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(g.n_angles * g.n_det_y * g.n_det_z, np.float64)
        if mode == "consistent":
            self._check(self.lib.ref_forward_project_matrix_free(p, _ptr(x), _ptr(y), threads))
        else:
            self._check(self.lib.ref_forward_mf_mode(p, MODES[mode], k, _ptr(x), _ptr(y), threads))
        return y

    def back_project_matrix_free(self, g, y: np.ndarray, threads: int = 1,
                                 mode: str = "consistent", k: int = 1) -> np.ndarray:
        og, p = self._g(g)
        y = np.ascontiguousarray(y, np.float64)
        x = np.zeros(g.n_x * g.n_y * g.n_z, np.float64)
        if mode == "consistent":
            self._check(self.lib.ref_back_project_matrix_free(p, _ptr(y), _ptr(x), threads))
        else:
            self._check(self.lib.ref_back_mf_mode(p, MODES[mode], k, _ptr(y), _ptr(x), threads))
        return x

    def line_weights(self, g, m_y: int, m_z: int, ip: int, mode: str = "line", k: int = 1):
        """line_weights / multiline_weights (baseline.cpp:98-128): (col, len)."""
        og, p = self._g(g)
        n = 4096
        for _ in range(2):
            col = np.empty(n, np.uint32)
            ln = np.empty(n, np.float64)
            m = self.lib.ref_line_weights(p, MODES[mode], k, m_y, m_z, ip, _ptr(col), _ptr(ln), n)
            self._check(m)
            if m <= n:
                return col[:m].copy(), ln[:m].copy()
            n = m
        raise AssertionError("unreachable")

    def forward_mf_angles(self, g, angles, x: np.ndarray, threads: int = 1,
                          split: bool = False) -> np.ndarray:
        """A x rows of the listed angles. split=True (restatement only) also
        splits each angle into slabs to use all threads (same values up to
        summation order)."""
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.size * g.n_det_y * g.n_det_z, np.float64)
        f = self.lib.ref_forward_mf_angles_par if (split and self.has_par) else self.lib.ref_forward_mf_angles
        self._check(f(p, _ptr(a), a.size, _ptr(x), _ptr(y), threads))
        return y

    def back_mf_angles(self, g, angles, y: np.ndarray, threads: int = 1,
                       split: bool = False) -> np.ndarray:
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        y = np.ascontiguousarray(y, np.float64)
        x = np.zeros(g.n_x * g.n_y * g.n_z, np.float64)
        f = self.lib.ref_back_mf_angles_par if (split and self.has_par) else self.lib.ref_back_mf_angles
        self._check(f(p, _ptr(a), a.size, _ptr(y), _ptr(x), threads))
        return x

    def forward_mf_angles_slabs(self, g, angles, zlo: int, zhi: int, x: np.ndarray,
                                threads: int = 1) -> np.ndarray:
        """A x rows of the listed angles from the voxels of z slabs [zlo, zhi)
        only (restatement only): BASELINE-scale parity of chosen slabs."""
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(a.size * g.n_det_y * g.n_det_z, np.float64)
        self._check(self.lib.ref_forward_mf_angles_slabs(p, _ptr(a), a.size, zlo, zhi, _ptr(x),
                                                         _ptr(y), threads))
        return y

    def back_mf_angles_slabs(self, g, angles, zlo: int, zhi: int, y_rows: np.ndarray,
                             threads: int = 1) -> np.ndarray:
        """A^T y of the listed angles on the voxels of z slabs [zlo, zhi)
        (others 0); y_rows = the rows of the listed angles, in list order."""
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        yr = np.ascontiguousarray(y_rows, np.float64)
        assert yr.size == a.size * g.n_det_y * g.n_det_z
        x = np.zeros(g.n_x * g.n_y * g.n_z, np.float64)
        self._check(self.lib.ref_back_mf_angles_slabs(p, _ptr(a), a.size, zlo, zhi, _ptr(yr),
                                                      _ptr(x), threads))
        return x

    def mf_pair_sample(self, g, angles, slabs, x: np.ndarray, y: np.ndarray, threads: int = 1):
        """One bounded A x + A^T y sample: the listed angles x the listed slabs
        (z planes in 3D, pixel rows in 2D), weights evaluated once per product
        as the reference does -> (updates applied, checksum). ref_* variants
        use the reference's own weight functions (ref_shim.cpp); the ports fall
        back to the slab restatements."""
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        sl = np.ascontiguousarray(slabs, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        if self.has_pair_sample:
            cs = ctypes.c_double(0.0)
            nu = ctypes.c_uint64(0)
            self._check(self.lib.ref_mf_pair_sample(p, _ptr(a), a.size, _ptr(sl), sl.size, _ptr(x),
                                                    _ptr(y), ctypes.byref(cs), ctypes.byref(nu),
                                                    threads))
            return int(nu.value), float(cs.value)
        if g.n_z == 1:
            raise NotImplementedError("2D slab samples need the ref_* oracle")
        rpa = g.n_det_y * g.n_det_z
        yrows = np.concatenate([y[int(k) * rpa:(int(k) + 1) * rpa] for k in a])
        cs, nu = 0.0, 0
        for z in sl:
            yy = self.forward_mf_angles_slabs(g, a, int(z), int(z) + 1, x, threads)
            xx = self.back_mf_angles_slabs(g, a, int(z), int(z) + 1, yrows, threads)
            cs += float(yy.sum() + xx.sum())
        return nu, cs

    def csr_angle_sample(self, g, angles, threads: int = 1) -> int:
        """build_angle_block (projector.cpp:92-104) of the listed angles, one
        angle per worker -> entries built (ref_* variants only)."""
        og, p = self._g(g)
        a = np.ascontiguousarray(angles, np.int32)
        nnz = ctypes.c_uint64(0)
        self._check(self.lib.ref_csr_angle_sample(p, _ptr(a), a.size, ctypes.byref(nnz), threads))
        return int(nnz.value)

    def sirt(self, g, y: np.ndarray, x0: np.ndarray, iters: int, threads: int = 1) -> np.ndarray:
        og, p = self._g(g)
        y = np.ascontiguousarray(y, np.float64)
        x = np.array(x0, np.float64, copy=True)
        self._check(self.lib.ref_sirt(p, _ptr(y), _ptr(x), iters, threads))
        return x

    # -- reference solver / io (ref_* variants only) -------------------------
    def _with_matrix(self, g, fn, budget: int = 5 << 30, threads: int = 1):
        og, p = self._g(g)
        st = ctypes.c_int(0)
        h = self.lib.ref_build_system_matrix(p, threads, budget, ctypes.byref(st))
        self._check(st.value)
        try:
            return fn(h)
        finally:
            self.lib.ref_csr_free(h)

    def spectral_norm_power(self, g, iters: int = 100, seed: int = 7, scale: float = 1.0,
                            threads: int = 1) -> float:
        """build_system_matrix + (scale_values) + spectral_norm_power."""
        def run(h):
            if scale != 1.0:
                self._check(self.lib.ref_scale_values(h, scale))
            out = ctypes.c_double(0.0)
            self._check(self.lib.ref_spectral_norm_power(h, iters, seed, ctypes.byref(out)))
            return out.value
        return self._with_matrix(g, run, threads=threads)

    def nag_tikhonov(self, g, p, lam: float, max_iter: int, tol: float, scale: float = 1.0,
                     keep_trace: bool = False, threads: int = 1):
        """build_system_matrix + scale_values(scale) + nag_tikhonov ->
        (u, iterations, converged, trace[n, 3] or None)."""
        p = np.ascontiguousarray(p, np.float64)

        def run(h):
            if scale != 1.0:
                self._check(self.lib.ref_scale_values(h, scale))
            u = np.zeros(self.lib.ref_csr_cols(h), np.float64)
            its, conv = ctypes.c_int(0), ctypes.c_int(0)
            tr = np.zeros(3 * max(max_iter, 1)) if keep_trace else None
            self._check(self.lib.ref_nag_tikhonov(h, _ptr(p), lam, max_iter, tol, _ptr(u),
                                                  ctypes.byref(its), ctypes.byref(conv),
                                                  _ptr(tr) if keep_trace else None))
            trace = tr[:3 * its.value].reshape(-1, 3) if keep_trace else None
            return u, its.value, bool(conv.value), trace
        return self._with_matrix(g, run, threads=threads)

    def back_project_csr(self, g, y, threads: int = 1) -> np.ndarray:
        """build_system_matrix + back_project (projector.cpp:219-233)."""
        y = np.ascontiguousarray(y, np.float64)
        x = np.zeros(g.n_x * g.n_y * g.n_z, np.float64)
        self._with_matrix(g, lambda h: self._check(self.lib.ref_back_project(h, _ptr(y), _ptr(x))),
                          threads=threads)
        return x

    def write_matrix(self, g, path: str, threads: int = 1) -> None:
        """build_system_matrix + write_matrix (CSM1, io.cpp:153-177)."""
        self._with_matrix(g, lambda h: self._check(self.lib.ref_write_matrix(h, path.encode())),
                          threads=threads)

    def read_matrix(self, path: str):
        """read_matrix (io.cpp:179-227) -> (Csr, n_cols, meta)."""
        st = ctypes.c_int(0)
        h = self.lib.ref_read_matrix(path.encode(), ctypes.byref(st))
        self._check(st.value)
        try:
            nnz = self.lib.ref_csr_nnz(h)
            rows = self.lib.ref_csr_rows(h)
            rs = np.empty(rows + 1, np.uint64)
            col = np.empty(nnz, np.uint32)
            val = np.empty(nnz, np.float64)
            self.lib.ref_csr_copy(h, _ptr(rs), _ptr(col), _ptr(val))
            n = self.lib.ref_csr_meta(h, None, 0)
            buf = ctypes.create_string_buffer(int(n))
            self.lib.ref_csr_meta(h, ctypes.cast(buf, _P), n)
            return Csr(rs, col, val), int(self.lib.ref_csr_cols(h)), buf.raw.decode()
        finally:
            self.lib.ref_csr_free(h)

    def write_tensor(self, path: str, dims, data) -> None:
        d = np.ascontiguousarray(dims, np.uint64)
        x = np.ascontiguousarray(data, np.float64)
        self._check(self.lib.ref_write_tensor(path.encode(), _ptr(d), int(d.size), _ptr(x)))

    def normal_samples(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.ref_normal_samples(n, seed, _ptr(out))
        return out

    def angle_column_sums(self, g, ip: int) -> np.ndarray:
        og, p = self._g(g)
        s = np.zeros(g.n_x * g.n_y * g.n_z, np.float64)
        self._check(self.lib.ref_angle_column_sums(p, ip, _ptr(s)))
        return s


def csr_forward(c: Csr, x: np.ndarray) -> np.ndarray:
    """Row-ordered CSR A x in numpy (same association as projector.cpp:203-217
    only up to summation order; use for tolerance checks)."""
    rows = np.repeat(np.arange(c.row_start.size - 1), np.diff(c.row_start).astype(np.int64))
    y = np.zeros(c.row_start.size - 1)
    np.add.at(y, rows, c.val * x[c.col])
    return y


def csr_back(c: Csr, y: np.ndarray, n_cols: int) -> np.ndarray:
    """Transpose scatter in row order, skipping y_r == 0 (projector.cpp:219-233):
    np.add.at applies the adds in input order, i.e. the reference's order."""
    rows = np.repeat(np.arange(c.row_start.size - 1), np.diff(c.row_start).astype(np.int64))
    keep = y[rows] != 0.0
    x = np.zeros(n_cols)
    np.add.at(x, c.col[keep], c.val[keep] * y[rows[keep]])
    return x


def _seq_sum(a: np.ndarray) -> float:
    """Left-to-right sum (the reference's accumulation loops)."""
    return float(np.cumsum(a)[-1]) if a.size else 0.0


def nag_tikhonov_np(c: Csr, n_cols: int, p: np.ndarray, lam: float, max_iter: int, tol: float,
                    keep_trace: bool = False):
    """numpy restatement of solver.cpp:17-75 (same expressions, sequential
    sums) -> (u, iterations, converged, trace[n, 3] or None)."""
    L = 1.0 + lam
    q = csr_back(c, p, n_cols)
    u = np.zeros(n_cols)
    u_prev = np.zeros(n_cols)
    h = np.zeros(n_cols)
    h_prev = np.zeros(n_cols)
    t = 1.0
    its, conv, trace = 0, False, []
    for it in range(max_iter):
        t_next = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        m = (t - 1.0) / t_next
        y = (1.0 + m) * u - m * u_prev
        grad = (1.0 + m) * (h + lam * u) - m * (h_prev + lam * u_prev) - q
        u_prev = u
        h_prev = h
        u = y - grad / L
        t = t_next
        v = csr_forward(c, u)
        h = csr_back(c, v, n_cols)
        gi = h + lam * u - q
        grad_sq = _seq_sum(gi * gi)
        its = it + 1
        if keep_trace:
            r = v - p
            trace.append((it + 1, 0.5 * _seq_sum(r * r) + 0.5 * lam * _seq_sum(u * u), grad_sq))
        if not np.isfinite(grad_sq):
            raise OracleError(6, "solver iterate diverged")
        if grad_sq < tol:
            conv = True
            break
    return u, its, conv, (np.array(trace) if keep_trace else None)


def spectral_norm_power_np(c: Csr, n_cols: int, v0: np.ndarray, iters: int) -> float:
    """numpy restatement of projector.cpp:262-280 from the start vector v0
    (normal_samples(n_cols, seed))."""
    v = v0 / np.sqrt(_seq_sum(v0 * v0))
    lam = 0.0
    for _ in range(iters):
        u = csr_back(c, csr_forward(c, v), n_cols)
        lam = np.sqrt(_seq_sum(u * u))
        if lam == 0.0:
            raise OracleError(7, "power iteration collapsed")
        v = u / lam
    return float(np.sqrt(lam))
