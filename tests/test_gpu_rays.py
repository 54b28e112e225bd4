"""GPU parity of the line / multiline(k) modes (baseline.cpp:13-128, the
paper's comparison method) through the C-ABI.

Bars: the CSR (row_start, col, every val bit) is identical to the crmath
oracle -- the same trace_ray arithmetic with the same libm; against the glibc
reference the sparsity is identical on these cases and lengths agree within
1e-10. Matrix-free A x / A^T y: 1e-10 (fp64) / 1e-5 (fp32) relative,
max|diff| <= tol * max(1, max|ref|).
"""
import os

import numpy as np
import pytest

from paper_2511_12235_b200 import (CONFIGS, TEST_GEOMETRIES, CtsmError, back_project,
                                   back_project_matrix_free, build_system_matrix, forward_project,
                                   forward_project_matrix_free)
from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NTHREADS = max(1, os.cpu_count() or 1)
TOL64 = 1e-10
TOL32 = 1e-5
MODES = [("line", 1), ("multiline", 1), ("multiline", 3)]


def rel_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref))) / max(1.0, float(np.max(np.abs(ref))))


def block_csr(g, row, col, w):
    """angle-block entries (emission order) -> CSR with the reference's stable
    per-row column order (projector.cpp:92-104)."""
    rpa = g.rows_per_angle
    order = np.lexsort((np.arange(row.size), col, row))
    counts = np.bincount(row, minlength=rpa)
    rs = np.zeros(rpa + 1, np.uint64)
    rs[1:] = np.cumsum(counts)
    return rs, col[order], w[order]


def same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64),
                          np.asarray(b, np.float64).view(np.uint64))


@pytest.mark.parametrize("name", ["proj2d", "wide2d", "proj3d", "cone3d"])
@pytest.mark.parametrize("mode,k", MODES)
def test_ray_csr_bitexact_small(name, mode, k, oracle_cr):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g, mode, k)
    rs, col, val = w.to_host()
    ref = oracle_cr.build_system_matrix(g, threads=NTHREADS, mode=mode, k=k)
    assert np.array_equal(rs, ref.row_start)
    assert np.array_equal(col, ref.col)
    assert same_bits(val, ref.val)
    assert w.meta.startswith("mode=" + ("line" if mode == "line" else f"multiline:{k}"))


@pytest.mark.parametrize("mode,k", [("line", 1), ("multiline", 4)])
def test_ray_csr_c0_full(mode, k, oracle_cr, oracle_glibc):
    """BASELINE configs[0] geometry, whole matrix."""
    g = CONFIGS["c0"]
    w = build_system_matrix(g, mode, k)
    rs, col, val = w.to_host()
    ref = oracle_cr.build_system_matrix(g, threads=NTHREADS, mode=mode, k=k)
    assert np.array_equal(rs, ref.row_start) and np.array_equal(col, ref.col)
    assert same_bits(val, ref.val)
    refg = oracle_glibc.build_system_matrix(g, threads=NTHREADS, mode=mode, k=k)
    assert np.array_equal(rs, refg.row_start) and np.array_equal(col, refg.col)
    assert np.max(np.abs(val - refg.val)) <= TOL64
    # A x through the device CSR vs the device matrix-free ray projector
    x = torch.from_numpy(phantom_for("c0", g)).cuda()
    y0 = forward_project(w, x).cpu().numpy()
    y1 = forward_project_matrix_free(g, mode, k, x).cpu().numpy()
    assert rel_err(y1, y0) <= 1e-12


@pytest.mark.parametrize("mode,k,ip", [("line", 1, 0), ("line", 1, 37), ("multiline", 2, 90),
                                       ("multiline", 3, 181)])
def test_ray_csr_c2_angle_blocks(mode, k, ip, oracle_cr):
    """BASELINE configs[2] (3D 128^3, 256x256 detector) angle blocks."""
    g = CONFIGS["c2"]
    w = build_system_matrix(g, mode, k, angle_range=(ip, ip + 1), memory_budget_bytes=1 << 40)
    rs, col, val = w.to_host()
    ref = block_csr(g, *oracle_cr.angle_block_entries(g, ip, mode=mode, k=k))
    assert np.array_equal(rs, ref[0])
    assert np.array_equal(col, ref[1])
    assert same_bits(val, ref[2])


@pytest.mark.parametrize("name", ["proj2d", "wide2d", "proj3d", "cone3d"])
@pytest.mark.parametrize("mode,k", MODES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_ray_matrix_free_small(name, mode, k, dtype, oracle_cr):
    g = TEST_GEOMETRIES[name]
    rng = np.random.default_rng(9)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    tol = TOL64 if dtype == "f64" else TOL32
    xt = torch.tensor(rng.uniform(0, 1, g.n_voxels), dtype=tdt, device="cuda")
    yt = torch.tensor(rng.uniform(0, 1, g.n_measurements), dtype=tdt, device="cuda")
    xr, yr = xt.double().cpu().numpy(), yt.double().cpu().numpy()
    yg = forward_project_matrix_free(g, mode, k, xt).double().cpu().numpy()
    assert rel_err(yg, oracle_cr.forward_project_matrix_free(g, xr, NTHREADS, mode, k)) <= tol
    xg = back_project_matrix_free(g, mode, k, yt).double().cpu().numpy()
    assert rel_err(xg, oracle_cr.back_project_matrix_free(g, yr, NTHREADS, mode, k)) <= tol


def test_ray_adjoint_and_csr_transpose():
    """<A x, y> == <x, A^T y> for the matrix-free pair; the matrix-free A^T y
    equals the CSR back_project."""
    g = TEST_GEOMETRIES["cone3d"]
    gen = torch.Generator().manual_seed(5)
    x = torch.rand(g.n_voxels, generator=gen, dtype=torch.float64).cuda()
    y = torch.rand(g.n_measurements, generator=gen, dtype=torch.float64).cuda()
    for mode, k in (("line", 1), ("multiline", 2)):
        ax = forward_project_matrix_free(g, mode, k, x)
        aty = back_project_matrix_free(g, mode, k, y)
        lhs, rhs = float(torch.dot(ax, y)), float(torch.dot(x, aty))
        assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
        w = build_system_matrix(g, mode, k)
        assert rel_err(back_project(w, y).cpu().numpy(), aty.cpu().numpy()) <= 1e-12


def test_ray_c1_sampled_angles(oracle_glibc):
    """BASELINE configs[1] geometry: line / multiline:2 A x and A^T y on angle
    shards against the reference's own ray tracer (glibc)."""
    g = CONFIGS["c1"]
    x = torch.from_numpy(phantom_for("c1", g)).cuda()
    y = torch.from_numpy(uniform_sinogram(g.n_measurements, 12346)).cuda()
    for mode, k in (("line", 1), ("multiline", 2)):
        sel = (5, 720, 179)
        yg = forward_project_matrix_free(g, mode, k, x, angles=sel).cpu().numpy()
        xg = back_project_matrix_free(g, mode, k, y, angles=sel).cpu().numpy()
        rpa = g.rows_per_angle
        yref = np.zeros(g.n_measurements)
        xref = np.zeros(g.n_voxels)
        ynp = y.cpu().numpy()
        xnp = x.cpu().numpy()
        for a in range(*sel):
            r, c, w = oracle_glibc.angle_block_entries(g, a, mode=mode, k=k)
            np.add.at(yref, a * rpa + r.astype(np.int64), w * xnp[c])
            np.add.at(xref, c, w * ynp[a * rpa + r.astype(np.int64)])
        assert rel_err(yg, yref) <= TOL64
        assert rel_err(xg, xref) <= TOL64


def test_ray_deterministic_and_errors():
    g = CONFIGS["c1"]
    y = torch.from_numpy(uniform_sinogram(g.n_measurements, 7)).cuda()
    a = back_project_matrix_free(g, "multiline", 2, y, angles=(0, 720, 13))
    b = back_project_matrix_free(g, "multiline", 2, y, angles=(0, 720, 13))
    assert torch.equal(a, b)
    gs = TEST_GEOMETRIES["proj2d"]
    with pytest.raises(CtsmError) as e:
        build_system_matrix(gs, "multiline", 0)
    assert e.value.code == "InvalidSpec"
    with pytest.raises(CtsmError) as e:
        build_system_matrix(TEST_GEOMETRIES["proj3d"], "line", 1, memory_budget_bytes=1024)
    assert e.value.code == "OutOfMemory"
