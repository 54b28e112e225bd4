"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (needs oracle/_ref, i.e. /root/reference compiled by
oracle/Makefile):   python tests/golden/make_golden.py [--rays]
(--rays regenerates only the line / multiline fixtures rays_*.npz, c0_rays_*.npz)

Each fixture is produced twice: with the reference linked against glibc's libm
(`*_glibc.npz`, the reference exactly as shipped) and against the correctly
rounded crmath.h (`*_cr.npz`, deterministic on every machine -- the bit-exact
pin for the oracle restatement and the GPU kernels). The reference ships no
golden vectors of its own; these are its outputs on seeded
inputs and on the geometries of its own unit tests.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import pyoracle  # noqa: E402
from paper_2511_12235_b200.geometry import CONFIGS, TEST_GEOMETRIES  # noqa: E402

THREADS = os.cpu_count() or 1


def csr_fixture(orc, g, seed):
    m = orc.build_system_matrix(g, threads=THREADS)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(g.n_voxels)
    y = rng.uniform(0, 1, g.n_measurements)
    return dict(row_start=m.row_start, col=m.col, val=m.val, x=x, y=y,
                fwd=orc.forward_project_matrix_free(g, x, THREADS),
                bwd=orc.back_project_matrix_free(g, y, THREADS))


def weight_samples(orc, g, n, seed, angles=None, zslab=None):
    """voxel/pixel weights at seeded (voxel, angle) samples."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        ix, iy = int(rng.integers(g.n_x)), int(rng.integers(g.n_y))
        iz = 0 if g.is_2d() else (int(rng.integers(g.n_z)) if zslab is None else int(zslab[i % len(zslab)]))
        ip = int(rng.integers(g.n_angles)) if angles is None else int(angles[i % len(angles)])
        phi = orc.angle(g, ip)
        if g.is_2d():
            my, w = orc.pixel_area_factors(g, ix, iy, phi)
            mz = np.zeros_like(my)
        else:
            my, mz, w = orc.voxel_volume_factors(g, ix, iy, iz, phi)
        for a, b, c in zip(my, mz, w):
            rows.append((ix, iy, iz, ip, a, b, c))
    arr = np.array(rows, dtype=np.float64) if rows else np.zeros((0, 7))
    return dict(vox=arr[:, :4].astype(np.int32), my=arr[:, 4].astype(np.int32),
                mz=arr[:, 5].astype(np.int32), w=arr[:, 6])


RAY_CASES = [("proj2d", "line", 1), ("proj2d", "multiline", 3), ("proj3d", "line", 1),
             ("proj3d", "multiline", 2)]


def ray_fixture(orc, g, mode, k, seed):
    """line / multiline(k) matrices (baseline.cpp:13-128) of a test geometry."""
    m = orc.build_system_matrix(g, threads=THREADS, mode=mode, k=k)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(g.n_voxels)
    y = rng.uniform(0, 1, g.n_measurements)
    return dict(row_start=m.row_start, col=m.col, val=m.val, x=x, y=y,
                fwd=orc.forward_project_matrix_free(g, x, THREADS, mode, k),
                bwd=orc.back_project_matrix_free(g, y, THREADS, mode, k))


def main_rays():
    for variant in ("ref_glibc", "ref_cr"):
        orc = pyoracle.load(variant)
        tag = variant.split("_")[1]
        for name, mode, k in RAY_CASES:
            np.savez_compressed(os.path.join(HERE, f"rays_{name}_{mode}{k}_{tag}.npz"),
                                **ray_fixture(orc, TEST_GEOMETRIES[name], mode, k, 13))
        # C0 (BASELINE configs[0]) line / multiline:4 angle blocks
        g = CONFIGS["c0"]
        blocks = {}
        for mode, k, ip in (("line", 1, 17), ("multiline", 4, 45), ("line", 1, 90)):
            r, c, w = orc.angle_block_entries(g, ip, mode=mode, k=k)
            key = f"{mode}{k}_{ip}"
            blocks[f"row_{key}"], blocks[f"col_{key}"], blocks[f"w_{key}"] = r, c, w
        np.savez_compressed(os.path.join(HERE, f"c0_rays_{tag}.npz"), **blocks)


def main():
    for variant in ("ref_glibc", "ref_cr"):
        orc = pyoracle.load(variant)
        tag = variant.split("_")[1]
        for name in ("proj2d", "wide2d", "proj3d", "cone3d"):
            np.savez_compressed(os.path.join(HERE, f"csr_{name}_{tag}.npz"),
                                **csr_fixture(orc, TEST_GEOMETRIES[name], 11))
        # C0 angle blocks (incl. the flat angle 0 and 45 deg)
        g = CONFIGS["c0"]
        blocks = {}
        for ip in (0, 17, 45):
            r, c, w = orc.angle_block_entries(g, ip)
            blocks[f"row_{ip}"], blocks[f"col_{ip}"], blocks[f"w_{ip}"] = r, c, w
        np.savez_compressed(os.path.join(HERE, f"c0_blocks_{tag}.npz"), **blocks)
        # sampled weights at BASELINE geometries; 3D samples include the top
        # z-slab (the cancellation-noise band) and flat-source angles
        np.savez_compressed(os.path.join(HERE, f"w_c1_{tag}.npz"),
                            **weight_samples(orc, CONFIGS["c1"], 400, 21))
        np.savez_compressed(os.path.join(HERE, f"w_c2_{tag}.npz"),
                            **weight_samples(orc, CONFIGS["c2"], 400, 22, angles=[0, 37, 90, 181, 270]))
        np.savez_compressed(os.path.join(HERE, f"w_c2top_{tag}.npz"),
                            **weight_samples(orc, CONFIGS["c2"], 200, 23, angles=[37], zslab=[124, 125, 126, 127]))
        np.savez_compressed(os.path.join(HERE, f"w_c3_{tag}.npz"),
                            **weight_samples(orc, CONFIGS["c3"], 200, 24, angles=[0, 111, 180, 500]))
        np.savez_compressed(os.path.join(HERE, f"w_c4_{tag}.npz"),
                            **weight_samples(orc, CONFIGS["c4"], 200, 25, angles=[0, 37, 360, 1001]))
        print("wrote fixtures for", variant)


if __name__ == "__main__":
    if "--rays" in sys.argv:
        main_rays()
    else:
        main()
        main_rays()
