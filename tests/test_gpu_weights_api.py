"""GPU parity of the reference's weight API (SURVEY.md §8(b) "signatures to
keep": pixel_area_factors weights2d.hpp:31-32, voxel_volume_factors
weights3d.hpp:90-91, detail::angle_block_entries projector.hpp:72-78) and of
the multi-GPU context, through the C-ABI, against the CPU oracle."""
import ctypes
import os

import numpy as np
import pytest

from paper_2511_12235_b200 import (CONFIGS, TEST_GEOMETRIES, _lib, angle_block_entries,
                                   back_project_matrix_free, forward_project_matrix_free,
                                   pixel_area_factors, sirt, voxel_volume_factors, weights_batch)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NTHREADS = max(1, os.cpu_count() or 1)


def _queries(g, n, seed, on_grid):
    rng = np.random.default_rng(seed)
    ix = rng.integers(0, g.n_x, n)
    iy = rng.integers(0, g.n_y, n)
    iz = rng.integers(0, g.n_z, n)
    if on_grid:
        phi = np.array([g.angle(int(i)) for i in rng.integers(0, g.n_angles, n)])
    else:  # the reference's functions take any phi, not an angle index
        phi = rng.uniform(-1.0, 7.0, n)
    return ix, iy, iz, phi


@pytest.mark.parametrize("name,on_grid", [("proj2d", True), ("wide2d", False), ("c0", True),
                                          ("c1", False)])
def test_pixel_area_factors_bitexact(name, on_grid, oracle_cr):
    g = TEST_GEOMETRIES.get(name) or CONFIGS[name]
    ix, iy, _, phi = _queries(g, 400, 11, on_grid)
    count, my, _, w = weights_batch(g, ix, iy, None, phi)
    for q in range(ix.size):
        rmy, rw = oracle_cr.pixel_area_factors(g, int(ix[q]), int(iy[q]), float(phi[q]))
        n = int(count[q])
        assert n == rmy.size
        assert np.array_equal(my[q, :n], rmy)
        assert np.array_equal(w[q, :n].view(np.uint64), rw.view(np.uint64))
    # the single-query form (the reference's signature)
    one = pixel_area_factors((int(ix[0]), int(iy[0])), float(phi[0]), g)
    rmy, rw = oracle_cr.pixel_area_factors(g, int(ix[0]), int(iy[0]), float(phi[0]))
    assert [m for m, _ in one] == list(rmy) and [v for _, v in one] == list(rw)


@pytest.mark.parametrize("name,on_grid", [("proj3d", True), ("cone3d", False), ("c2", True),
                                          ("c3", False), ("c4", True)])
def test_voxel_volume_factors_bitexact(name, on_grid, oracle_cr):
    g = TEST_GEOMETRIES.get(name) or CONFIGS[name]
    ix, iy, iz, phi = _queries(g, 300, 12, on_grid)
    if on_grid:  # include the flat-source branch (phi = 0, pi/2) and the top slab
        phi[:4] = [g.angle(0), g.angle(g.n_angles // 4), g.angle(g.n_angles // 2), g.angle(1)]
        iz[:8] = [g.n_z - 1, 0, g.n_z // 2, g.n_z // 2 - 1, g.n_z - 1, 0, g.n_z // 2, 1]
    count, my, mz, w = weights_batch(g, ix, iy, iz, phi)
    for q in range(ix.size):
        rmy, rmz, rw = oracle_cr.voxel_volume_factors(g, int(ix[q]), int(iy[q]), int(iz[q]),
                                                      float(phi[q]))
        n = int(count[q])
        assert n == rmy.size, (q, n, rmy.size)
        assert np.array_equal(my[q, :n], rmy) and np.array_equal(mz[q, :n], rmz)
        assert np.array_equal(w[q, :n].view(np.uint64), rw.view(np.uint64))
    one = voxel_volume_factors((int(ix[0]), int(iy[0]), int(iz[0])), float(phi[0]), g)
    assert len(one) == int(count[0])


@pytest.mark.parametrize("name,ip", [("proj2d", 3), ("proj3d", 2), ("cone3d", 0), ("c0", 37),
                                     ("c2", 37)])
def test_angle_block_entries_emission_order(name, ip, oracle_cr):
    """Same entries in the same order as the reference's emission (voxels z ->
    y -> x, each voxel's weights by (m_y, m_z)), bit for bit."""
    g = TEST_GEOMETRIES.get(name) or CONFIGS[name]
    raster, col, w = angle_block_entries(g, "consistent", 1, ip)
    rr, rc, rw = oracle_cr.angle_block_entries(g, ip, threads=NTHREADS)
    assert raster.numel() == rr.size
    assert np.array_equal(raster.cpu().numpy().view(np.uint32), rr)
    assert np.array_equal(col.cpu().numpy().view(np.uint32), rc)
    assert np.array_equal(w.cpu().numpy().view(np.uint64), rw.view(np.uint64))


@pytest.mark.parametrize("mode,k", [("line", 1), ("multiline", 2)])
def test_angle_block_entries_ray_modes(mode, k, oracle_cr):
    g = TEST_GEOMETRIES["proj3d"]
    raster, col, w = angle_block_entries(g, mode, k, 1)
    rr, rc, rw = oracle_cr.angle_block_entries(g, 1, mode=mode, k=k)
    got = sorted(zip(raster.cpu().numpy().view(np.uint32).tolist(),
                     col.cpu().numpy().view(np.uint32).tolist(),
                     w.cpu().numpy().view(np.uint64).tolist()))
    ref = sorted(zip(rr.tolist(), rc.tolist(), rw.view(np.uint64).tolist()))
    assert got == ref


# ---- multi-GPU context (one device here: the one-rank NCCL communicator) ----
def _multi(devices):
    h = ctypes.c_void_p()
    arr = (ctypes.c_int * len(devices))(*devices)
    _lib.check(_lib.lib().ctsm_multi_create(arr, len(devices), ctypes.byref(h)))
    return h


@pytest.mark.parametrize("name,dtype", [("proj2d", np.float64), ("cone3d", np.float64),
                                        ("cone3d", np.float32)])
def test_multi_context_one_device_with_nccl(name, dtype, monkeypatch):
    """ctsm_multi_* on a one-device list with CTSM_MULTI_FORCE_NCCL=1: the
    library creates the communicator and runs ncclAllReduce on the GPU; the
    results equal the single-context calls."""
    monkeypatch.setenv("CTSM_MULTI_FORCE_NCCL", "1")
    g = TEST_GEOMETRIES[name]
    L = _lib.lib()
    m = _multi([0])
    try:
        assert L.ctsm_multi_size(m) == 1
        assert L.ctsm_multi_nccl_version(m) >= 21000
        code = 0 if dtype == np.float64 else 1
        rng = np.random.default_rng(5)
        x = rng.uniform(0, 1, g.n_voxels).astype(dtype)
        y = rng.uniform(0, 1, g.n_measurements).astype(dtype)
        cg = g.to_c()
        yo = np.zeros(g.n_measurements, dtype)
        xo = np.zeros(g.n_voxels, dtype)
        _lib.check(L.ctsm_multi_forward_project_matrix_free_host(m, ctypes.byref(cg), code,
                                                                 x.ctypes.data, yo.ctypes.data))
        _lib.check(L.ctsm_multi_back_project_matrix_free_host(m, ctypes.byref(cg), code,
                                                              y.ctypes.data, xo.ctypes.data))
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        ys = forward_project_matrix_free(g, "consistent", 1, torch.tensor(x, device="cuda", dtype=tdt))
        xs = back_project_matrix_free(g, "consistent", 1, torch.tensor(y, device="cuda", dtype=tdt))
        tol = 1e-12 if dtype == np.float64 else 1e-5
        assert np.max(np.abs(yo - ys.cpu().numpy())) <= tol * max(1.0, float(ys.abs().max()))
        assert np.max(np.abs(xo - xs.cpu().numpy())) <= tol * max(1.0, float(xs.abs().max()))
        xi = np.zeros(g.n_voxels, dtype)
        _lib.check(L.ctsm_multi_sirt_host(m, ctypes.byref(cg), code, y.ctypes.data, xi.ctypes.data, 3))
        xr = sirt(g, torch.tensor(y, device="cuda", dtype=tdt),
                  torch.zeros(g.n_voxels, device="cuda", dtype=tdt), 3)
        assert np.max(np.abs(xi - xr.cpu().numpy())) <= (1e-10 if dtype == np.float64 else 1e-4) * \
            max(1.0, float(xr.abs().max()))
    finally:
        L.ctsm_multi_destroy(m)


def test_multi_context_rejects_bad_device_lists():
    L = _lib.lib()
    h = ctypes.c_void_p()
    arr = (ctypes.c_int * 2)(0, 0)
    assert L.ctsm_multi_create(arr, 2, ctypes.byref(h)) == 10  # InvalidSpec: listed twice
    assert L.ctsm_multi_create(arr, 0, ctypes.byref(h)) == 10
    arr = (ctypes.c_int * 1)(99)
    assert L.ctsm_multi_create(arr, 1, ctypes.byref(h)) == 10  # no such device


# ---- device MC / Gauss-Legendre oracles -------------
def test_device_numeric_oracles(oracle_cr):
    """mc_volume_3d on the device reproduces the CPU oracle's hit counts (same
    16 mt19937_64 sub-streams, same arithmetic); multiline_volume_3d agrees to
    rounding; both agree with the closed-form weights by the reference's
    criteria (test_weights3d.cpp:198-212)."""
    from paper_2511_12235_b200.oracles import (mc_volume_3d, mc_volume_3d_batch,
                                               multiline_volume_3d_batch, voxel_box)
    g = TEST_GEOMETRIES["cone3d"]
    rng = np.random.default_rng(8)
    boxes, phis, mys, mzs, ws = [], [], [], [], []
    for _ in range(24):
        ix, iy, iz = (int(v) for v in rng.integers(0, 6, 3))
        phi = float(rng.uniform(0, 6.28))
        my, mz, w = oracle_cr.voxel_volume_factors(g, ix, iy, iz, phi)
        i = int(np.argmax(w))
        boxes.append(voxel_box(g, ix, iy, iz))
        phis.append(phi)
        mys.append(int(my[i]))
        mzs.append(int(mz[i]))
        ws.append(float(w[i]))
    n_samples, seed = 100003, 99
    v, se, hits = mc_volume_3d_batch(boxes, phis, g.s, g.d, g.d_y, g.d_z, mys, mzs, n_samples, seed)
    gl = multiline_volume_3d_batch(boxes, phis, g.s, g.d, g.d_y, g.d_z, mys, mzs, 100)
    for c in range(len(ws)):
        rv, rse, rh = oracle_cr.mc_volume_3d(g, boxes[c], phis[c], mys[c], mzs[c], n_samples, seed)
        assert int(hits[c]) == rh and v[c] == rv and se[c] == rse
        assert abs(ws[c] - v[c]) < 4 * se[c] + 1e-6
        rgl = oracle_cr.multiline_volume_3d(g, boxes[c], phis[c], mys[c], mzs[c], 100)
        assert abs(gl[c] - rgl) <= 1e-12 * max(1.0, abs(rgl))
        assert abs(gl[c] - ws[c]) < 2e-5  # k = 100 quadrature of a kinked integrand
    one = mc_volume_3d(*boxes[0], phis[0], g.s, g.d, g.d_y, g.d_z, mys[0], mzs[0], n_samples, seed)
    assert one.value == v[0] and one.std_err == se[0]
