"""Seeded synthetic inputs (BASELINE.json configs).

RNG conventions follow the reference: mt19937_64 with u01 = (rng() >> 11) *
2^-53 (validate.cpp:20-24) and Box-Muller normals, cosine branch, two engine
outputs per sample (phantoms.cpp:78-87). Phantoms are additive ellipses /
ellipsoids sampled at pixel / voxel centres, the reference's Shepp-Logan
convention (phantoms.cpp:60-75). Bulk i.i.d. arrays (sinograms, noise) with
more than ~10^7 entries use numpy's PCG64 seeded with the same seed (an
mt19937_64 stream that long is too slow to draw in Python); the arrays are
generated once on the host and fed identically to the CPU oracle and the GPU.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

_NN = 312
_MM = 156
_MATA = np.uint64(0xB5026F5AA96619E9)
_UM = np.uint64(0xFFFFFFFF80000000)
_LM = np.uint64(0x7FFFFFFF)


class MT19937_64:
    """std::mt19937_64 (vectorised twist); bit-identical output sequence."""

    def __init__(self, seed: int):
        mt = [0] * _NN
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, _NN):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt = np.array(mt, dtype=np.uint64)
        self.idx = _NN

    def _twist(self):
        mt = self.mt
        one = np.uint64(1)
        with np.errstate(over="ignore"):
            y = (mt[: _NN - _MM] & _UM) | (mt[1: _NN - _MM + 1] & _LM)
            mt[: _NN - _MM] = mt[_MM:] ^ (y >> one) ^ ((y & one) * _MATA)
            y = (mt[_NN - _MM: _NN - 1] & _UM) | (mt[_NN - _MM + 1:] & _LM)
            mt[_NN - _MM: _NN - 1] = mt[: _MM - 1] ^ (y >> one) ^ ((y & one) * _MATA)
            y = (mt[_NN - 1] & _UM) | (mt[0] & _LM)
            mt[_NN - 1] = mt[_MM - 1] ^ (y >> one) ^ ((y & one) * _MATA)
        self.idx = 0

    @staticmethod
    def _temper(x):
        x = x ^ ((x >> np.uint64(29)) & np.uint64(0x5555555555555555))
        x = x ^ ((x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
        x = x ^ ((x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
        x = x ^ (x >> np.uint64(43))
        return x

    def draw(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        k = 0
        while k < n:
            if self.idx >= _NN:
                self._twist()
            take = min(n - k, _NN - self.idx)
            out[k:k + take] = self._temper(self.mt[self.idx:self.idx + take].copy())
            self.idx += take
            k += take
        return out

    def u01(self, n: int) -> np.ndarray:
        return (self.draw(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def normal_samples(n: int, seed: int) -> np.ndarray:
    """phantoms.cpp:78-87, computed by the library's host code
    (ctsm_normal_samples: std::mt19937_64 + the C library's log/cos, so the
    samples equal the reference's bit for bit)."""
    from . import _lib
    out = np.empty(n, np.float64)
    _lib.lib().ctsm_normal_samples(n, seed, out.ctypes.data_as(ctypes.c_void_p))
    return out


def uniform_sinogram(n: int, seed: int) -> np.ndarray:
    """i.i.d. U[0, 1) values (A^T y inputs)."""
    if n <= 10_000_000:
        return MT19937_64(seed).u01(n)
    return np.random.Generator(np.random.PCG64(seed)).random(n)


def ellipse_phantom_2d(g, n_ellipses: int, disc_radius: float, seed: int) -> np.ndarray:
    """Sum of ellipses: centres uniform in a disc, semi-axes U[5, 40] mm,
    rotation U[0, pi), attenuation U[0.005, 0.02] /mm; pixel-centre sampling;
    x fastest."""
    rng = MT19937_64(seed)
    xc = (np.arange(g.n_x) + 0.5 - g.n_x / 2.0) * g.a
    yc = (np.arange(g.n_y) + 0.5 - g.n_y / 2.0) * g.b
    X, Y = np.meshgrid(xc, yc)  # [n_y, n_x]
    img = np.zeros((g.n_y, g.n_x))
    for _ in range(n_ellipses):
        u = rng.u01(6)
        r = disc_radius * math.sqrt(u[0])
        th = 2.0 * math.pi * u[1]
        cx, cy = r * math.cos(th), r * math.sin(th)
        ax, ay = 5.0 + 35.0 * u[2], 5.0 + 35.0 * u[3]
        rot = math.pi * u[4]
        mu = 0.005 + 0.015 * u[5]
        dx, dy = X - cx, Y - cy
        xr = dx * math.cos(rot) + dy * math.sin(rot)
        yr = -dx * math.sin(rot) + dy * math.cos(rot)
        img += mu * ((xr / ax) ** 2 + (yr / ay) ** 2 <= 1.0)
    return img.reshape(-1)


def ellipsoid_phantom_3d(g, n_ellipsoids: int, ball_radius: float, seed: int,
                         dtype=np.float64) -> np.ndarray:
    """Sum of ellipsoids: centres uniform in a ball, semi-axes U[4, 30] mm,
    uniform random rotation (unit quaternion from 4 normals), attenuation
    U[0.005, 0.02] /mm; voxel-centre sampling; layout [n_z][n_y][n_x]."""
    rng = MT19937_64(seed)
    xc = ((np.arange(g.n_x) + 0.5 - g.n_x / 2.0) * g.a).astype(np.float32)
    yc = ((np.arange(g.n_y) + 0.5 - g.n_y / 2.0) * g.b).astype(np.float32)
    zc = ((np.arange(g.n_z) + 0.5 - g.n_z / 2.0) * g.c).astype(np.float32)
    vol = np.zeros((g.n_z, g.n_y, g.n_x), dtype=dtype)

    def normals(k):
        raw = rng.draw(2 * k).reshape(k, 2) >> np.uint64(11)
        u1 = (raw[:, 0].astype(np.float64) + 1.0) * 2.0 ** -53
        u2 = raw[:, 1].astype(np.float64) * 2.0 ** -53
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)

    for _ in range(n_ellipsoids):
        u = rng.u01(5)
        r = ball_radius * u[0] ** (1.0 / 3.0)
        dvec = normals(3)
        dvec /= np.linalg.norm(dvec)
        c = r * dvec
        axes = 4.0 + 26.0 * u[1:4]
        mu = 0.005 + 0.015 * u[4]
        q = normals(4)
        q /= np.linalg.norm(q)
        w, x, y, z = q
        Rm = np.array([
            [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
            [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
            [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
        ])
        # bounding box in index space to limit work
        ext = np.abs(Rm) @ axes
        lo = c - ext
        hi = c + ext
        ix = np.nonzero((xc >= lo[0]) & (xc <= hi[0]))[0]
        iy = np.nonzero((yc >= lo[1]) & (yc <= hi[1]))[0]
        iz = np.nonzero((zc >= lo[2]) & (zc <= hi[2]))[0]
        if ix.size == 0 or iy.size == 0 or iz.size == 0:
            continue
        Z, Y, X = np.meshgrid(zc[iz] - c[2], yc[iy] - c[1], xc[ix] - c[0], indexing="ij")
        P = np.stack([X, Y, Z], axis=-1) @ Rm.astype(np.float32)  # body coordinates
        inside = ((P[..., 0] / axes[0]) ** 2 + (P[..., 1] / axes[1]) ** 2 +
                  (P[..., 2] / axes[2]) ** 2) <= 1.0
        vol[iz[0]:iz[-1] + 1, iy[0]:iy[-1] + 1, ix[0]:ix[-1] + 1] += (mu * inside).astype(dtype)
    return vol.reshape(-1)


# Workload recipes of BASELINE.json configs (seed = phantom, seed+1 = sinogram,
# seed+2 = noise; default seed 12345 as io.hpp:20).
DEFAULT_SEED = 12345
PHANTOM_SPEC = {
    "c0": ("2d", 10, 50.0),
    "c1": ("2d", 40, 100.0),
    "c2": ("3d", 20, 40.0),
    "c3": ("3d", 50, 40.0),
    "c4": ("3d", 100, 40.0),
}


def phantom_for(name: str, g, seed: int = DEFAULT_SEED, dtype=np.float64) -> np.ndarray:
    kind, n, radius = PHANTOM_SPEC[name]
    if kind == "2d":
        return ellipse_phantom_2d(g, n, radius, seed).astype(dtype)
    return ellipsoid_phantom_3d(g, n, radius, seed, dtype=dtype)
