"""GPU parity tests: CUDA path (through the C-ABI) vs the CPU oracle.

Bars (BASELINE.json north_star):
  * CSR sparsity bit-exact; with the crmath oracle (same libm on both sides)
    the whole CSR (row_start, col, val) is bit-identical;
  * weights / projections within 1e-10 (fp64) and 1e-5 (fp32) relative,
    max|diff| <= tol * max(1, max|ref|) (test_projector.cpp:117 convention).
"""
import os

import numpy as np
import pytest

import pyoracle
from paper_2511_12235_b200 import (CONFIGS, TEST_GEOMETRIES, CtsmError, back_project,
                                   back_project_matrix_free, build_system_matrix,
                                   forward_project, forward_project_matrix_free, sirt)
from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NTHREADS = max(1, os.cpu_count() or 1)
TOL64 = 1e-10
TOL32 = 1e-5


def rel_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref))) / max(1.0, float(np.max(np.abs(ref))))


def entries_to_csr(g, row, col, w):
    """angle-block entries (emission order) -> CSR of that angle block."""
    rpa = g.rows_per_angle
    order = np.argsort(row, kind="stable")
    counts = np.bincount(row, minlength=rpa)
    rs = np.zeros(rpa + 1, np.uint64)
    rs[1:] = np.cumsum(counts)
    return rs, col[order], w[order]


def assert_csr_bitexact(got, ref):
    rs, col, val = got
    assert np.array_equal(rs, ref.row_start), "row_start differs"
    assert np.array_equal(col, ref.col), "columns differ"
    assert np.array_equal(val.view(np.uint64), ref.val.view(np.uint64)), \
        f"values differ (max |diff| {np.max(np.abs(val - ref.val)):.3g})"


# ---- K1/K2: CSR emission ------------------------------------------------------
@pytest.mark.parametrize("name", ["proj2d", "wide2d", "proj3d", "cone3d"])
def test_csr_bitexact_small(name, oracle_cr):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    ref = oracle_cr.build_system_matrix(g, threads=NTHREADS)
    assert_csr_bitexact(w.to_host(), ref)
    # strictly ascending columns per row (test_projector.cpp:55-68)
    rs, col, _ = w.to_host()
    d = np.diff(col.astype(np.int64))
    starts = rs[1:-1].astype(np.int64)
    mask = np.ones(d.size, bool)
    mask[starts[(starts > 0) & (starts <= d.size)] - 1] = False
    assert np.all(d[mask] > 0)


def test_csr_c0_full_bitexact(oracle_cr, oracle_glibc):
    g = CONFIGS["c0"]
    w = build_system_matrix(g)
    got = w.to_host()
    assert w.nnz() == 18_291_648
    ref = oracle_cr.build_system_matrix(g, threads=NTHREADS)
    assert_csr_bitexact(got, ref)
    # against the glibc-libm reference: identical sparsity, weights within 1e-10
    refg = oracle_glibc.build_system_matrix(g, threads=NTHREADS)
    assert np.array_equal(got[0], refg.row_start)
    assert np.array_equal(got[1], refg.col)
    assert np.max(np.abs(got[2] - refg.val)) <= TOL64


@pytest.mark.parametrize("ip", [0, 37, 90, 181])
def test_csr_c2_angle_blocks_bitexact(ip, oracle_cr):
    g = CONFIGS["c2"]
    w = build_system_matrix(g, angle_range=(ip, ip + 1), memory_budget_bytes=1 << 40)
    ref = entries_to_csr(g, *oracle_cr.angle_block_entries(g, ip, threads=NTHREADS))
    rs, col, val = w.to_host()
    assert np.array_equal(rs, ref[0])
    assert np.array_equal(col, ref[1])
    assert np.array_equal(val.view(np.uint64), ref[2].view(np.uint64))


@pytest.mark.parametrize("name", ["proj2d", "cone3d"])
def test_csr_two_pass_equals_single_evaluation(name):
    """count / fill (two evaluations, exact-size arrays) and ctsm_csr_build
    (one evaluation) give the same bits."""
    g = TEST_GEOMETRIES[name]
    a = build_system_matrix(g).to_host()
    b = build_system_matrix(g, two_pass=True).to_host()
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64) if x.dtype == np.float64 else x,
                              y.view(np.uint64) if y.dtype == np.float64 else y)


def test_csr_long_rows_block_sort(oracle_cr):
    """C1's grid (512^2 pixels) with a 3x coarser detector: rows hold ~2,400
    entries, beyond the warp radix sort's 1,024, so they take the block-wide
    sort. Three angle blocks (axis-aligned, oblique, diagonal), bit-identical
    to the oracle."""
    g = CONFIGS["c1"].with_(d_y=1.8, n_det_y=344)
    for ip in (0, 37, 90):
        w = build_system_matrix(g, angle_range=(ip, ip + 1), memory_budget_bytes=1 << 40)
        ref = entries_to_csr(g, *oracle_cr.angle_block_entries(g, ip, threads=NTHREADS))
        rs, col, val = w.to_host()
        assert int(np.max(np.diff(rs.astype(np.int64)))) > 1024
        assert np.array_equal(rs, ref[0])
        assert np.array_equal(col, ref[1])
        assert np.array_equal(val.view(np.uint64), ref[2].view(np.uint64))
        w2 = build_system_matrix(g, angle_range=(ip, ip + 1), memory_budget_bytes=1 << 40,
                                 two_pass=True)
        assert torch.equal(w2.col, w.col) and torch.equal(w2.val.view(torch.int64),
                                                          w.val.view(torch.int64))


def test_csr_build_capacity_protocol(oracle_cr):
    """ctsm_csr_build with too small arrays reports the needed entry count
    and leaves the caller to retry; several angle chunks (C2, 9 angles: the
    chunk holds 7) are stitched at the right offsets."""
    import ctypes
    import torch
    from paper_2511_12235_b200 import _lib
    from paper_2511_12235_b200.projector import Context, _dev_ptr, _stream
    g = CONFIGS["c2"]
    ctx = Context.get(None)
    cg = g.to_c()
    a0, a1 = 88, 97
    n_rows = (a1 - a0) * g.rows_per_angle
    rs = torch.empty(n_rows + 1, dtype=torch.int64, device="cuda")
    nnz = ctypes.c_uint64(0)
    small = torch.empty(1000, dtype=torch.int32, device="cuda")
    smallv = torch.empty(1000, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    _lib.check(L.ctsm_csr_build(ctx.handle, ctypes.byref(cg), a0, a1, 1 << 40, _dev_ptr(rs),
                                _dev_ptr(small), _dev_ptr(smallv), 1000, ctypes.byref(nnz),
                                _stream(ctx.device)))
    need = nnz.value
    assert need > 1000
    w = build_system_matrix(g, angle_range=(a0, a1), memory_budget_bytes=1 << 40)
    assert w.nnz() == need
    assert int(rs[-1].item()) == need and torch.equal(rs, w.row_start)
    rs_h, col, val = w.to_host()
    rpa = g.rows_per_angle
    for ip in (88, 94, 96):  # first chunk, last angle of it, second chunk
        ref = entries_to_csr(g, *oracle_cr.angle_block_entries(g, ip, threads=NTHREADS))
        lo, hi = int(rs_h[(ip - a0) * rpa]), int(rs_h[(ip - a0 + 1) * rpa])
        assert np.array_equal(rs_h[(ip - a0) * rpa:(ip - a0 + 1) * rpa + 1] - np.uint64(lo), ref[0])
        assert np.array_equal(col[lo:hi], ref[1])
        assert np.array_equal(val[lo:hi].view(np.uint64), ref[2].view(np.uint64))
    w2 = build_system_matrix(g, angle_range=(a0, a1), memory_budget_bytes=1 << 40, two_pass=True)
    assert torch.equal(w2.row_start, w.row_start) and torch.equal(w2.col, w.col)
    assert torch.equal(w2.val.view(torch.int64), w.val.view(torch.int64))


def test_division_by_reciprocal_is_ieee_exact():
    """csr3d.cuh div_by (reciprocal + one fma correction) against the IEEE
    division on 2^28 pseudo-random operand pairs: no differing bit."""
    import ctypes
    from paper_2511_12235_b200 import _lib
    from paper_2511_12235_b200.projector import Context
    bad = ctypes.c_uint64(1)
    _lib.check(_lib.lib().ctsm_selftest_division(Context.get(None).handle, 1 << 28, 20261021,
                                                 ctypes.byref(bad)))
    assert bad.value == 0


def test_wide_shadows_csr_exact_and_matrix_free_limit(oracle_cr):
    """A detector 4x finer than cone3d's: a voxel's shadow spans ~18 cells.
    The exact CSR path (24 breakpoints) still matches the oracle bit for bit;
    the 3D matrix-free kernels (12 pieces per column) refuse by name instead
    of failing inside a kernel."""
    g0 = TEST_GEOMETRIES["cone3d"]
    g = g0.with_(d_y=g0.d_y / 4, n_det_y=g0.n_det_y * 4)
    w = build_system_matrix(g, memory_budget_bytes=1 << 34)
    ref = oracle_cr.build_system_matrix(g, threads=NTHREADS, budget=1 << 34)
    assert_csr_bitexact(w.to_host(), ref)
    with pytest.raises(CtsmError) as e:
        forward_project_matrix_free(g, "consistent", 1,
                                    torch.zeros(g.n_voxels, dtype=torch.float64, device="cuda"))
    assert e.value.code == "TooLarge" and "shadow" in str(e.value)


def test_csr_budget_and_size_limits():
    g = TEST_GEOMETRIES["proj3d"]
    with pytest.raises(CtsmError) as e:
        build_system_matrix(g, memory_budget_bytes=1024)
    assert e.value.code == "OutOfMemory"
    huge = g.with_(n_x=2048, n_y=2048, n_z=2048, a=0.01, b=0.01, c=0.01)
    with pytest.raises(CtsmError) as e:
        build_system_matrix(huge)
    assert e.value.code == "TooLarge"


# ---- K3/K4: CSR appliers --------------------------------------------------------
@pytest.mark.parametrize("name", ["proj2d", "proj3d"])
def test_spmv_and_transpose(name, oracle_cr):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(g.n_voxels)
    y = rng.standard_normal(g.n_measurements)
    ref = oracle_cr.build_system_matrix(g)
    assert rel_err(forward_project(w, x), pyoracle.csr_forward(ref, x)) <= 1e-13
    xb = back_project(w, y)
    xr = np.zeros(g.n_voxels)
    rows = np.repeat(np.arange(g.n_measurements), np.diff(ref.row_start).astype(np.int64))
    np.add.at(xr, ref.col, ref.val * y[rows])
    assert rel_err(xb, xr) <= 1e-13
    # adjoint identity (test_projector.cpp:81-91)
    lhs = float(np.dot(forward_project(w, x), y))
    rhs = float(np.dot(x, xb))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    with pytest.raises(CtsmError) as e:
        forward_project(w, np.zeros(g.n_voxels + 1))
    assert e.value.code == "DimensionMismatch"
    # K4 as a gather over the CSC transpose: the same fixed-point integers in
    # another order, so the same bits
    from paper_2511_12235_b200 import build_transpose, drop_transpose, scale_values
    build_transpose(w)
    xc = back_project(w, y)
    assert np.array_equal(np.asarray(xb).view(np.uint64), np.asarray(xc).view(np.uint64))
    key, col_start, row, valt = w._csc
    cs = col_start.cpu().numpy().view(np.uint64)
    assert cs[0] == 0 and cs[-1] == w.nnz()
    assert np.array_equal(np.diff(cs.astype(np.int64)), np.bincount(ref.col, minlength=g.n_voxels))
    # a column's entries are its (row, value) pairs, in any order
    rr, vv = row.cpu().numpy().view(np.uint32), valt.cpu().numpy()
    c = int(np.argmax(np.diff(cs.astype(np.int64))))
    got = sorted(zip(rr[cs[c]:cs[c + 1]].tolist(), vv[cs[c]:cs[c + 1]].tolist()))
    sel = np.nonzero(ref.col == c)[0]
    assert got == sorted(zip(rows[sel].tolist(), ref.val[sel].tolist()))
    scale_values(w, 2.0)  # drops the transpose with the column-sum bound
    assert w._csc is None
    assert rel_err(back_project(w, y), 2.0 * xr) <= 1e-13
    drop_transpose(w)


def test_csc_back_project_c0_bitexact():
    """C0 in full: back_project through the CSC transpose equals the scatter
    bit for bit (18.3 M entries, random sinogram with zeros)."""
    from paper_2511_12235_b200 import build_transpose
    g = CONFIGS["c0"]
    w = build_system_matrix(g)
    gen = torch.Generator().manual_seed(5)
    y = torch.rand(g.n_measurements, generator=gen, dtype=torch.float64)
    y[::7] = 0.0
    y = y.cuda()
    xs = back_project(w, y)
    build_transpose(w)
    xc = back_project(w, y)
    assert torch.equal(xs, xc)


# ---- K5/K6: matrix-free ---------------------------------------------------------
@pytest.mark.parametrize("case", ["odd_nz", "two_zblocks", "quarter_odd_nz"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_symmetric_3d_shapes_vs_oracle(case, dtype, oracle_cr, monkeypatch):
    """Symmetric 3D kernels against the oracle on the column shapes the
    BASELINE configs do not reach: odd n_z (no z mirror: every voxel
    evaluated, all accumulator slots on one side), a column longer than one
    z-block (two passes over the plans), and the quarter-turn (order 4) form
    of the member-outer back-projection."""
    from paper_2511_12235_b200.projector import symmetry_order
    base = TEST_GEOMETRIES["cone3d"].with_(n_angles=16)
    if case == "odd_nz":
        g = base.with_(n_z=5)
    elif case == "two_zblocks":  # 300 voxels: mirror half 150 > 128 per z-block
        g = base.with_(n_z=300, c=0.1)
    else:
        g = base.with_(n_z=7)
        monkeypatch.setenv("CTSM_NO_DIHEDRAL", "1")
    assert symmetry_order(g) == (4 if case == "quarter_odd_nz" else 8)
    rng = np.random.default_rng(11)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    tol = TOL64 if dtype == "f64" else TOL32
    xt = torch.tensor(rng.uniform(0, 1, g.n_voxels), dtype=tdt, device="cuda")
    yt = torch.tensor(rng.uniform(0, 1, g.n_measurements), dtype=tdt, device="cuda")
    yg = forward_project_matrix_free(g, "consistent", 1, xt).double().cpu().numpy()
    xg = back_project_matrix_free(g, "consistent", 1, yt).double().cpu().numpy()
    yref = oracle_cr.forward_project_matrix_free(g, xt.double().cpu().numpy(), NTHREADS)
    xref = oracle_cr.back_project_matrix_free(g, yt.double().cpu().numpy(), NTHREADS)
    assert rel_err(yg, yref) <= tol
    assert rel_err(xg, xref) <= tol
    # repeated calls are bit-equal in fp64 (fixed point / fixed order)
    if dtype == "f64":
        yg2 = forward_project_matrix_free(g, "consistent", 1, xt).double().cpu().numpy()
        xg2 = back_project_matrix_free(g, "consistent", 1, yt).double().cpu().numpy()
        assert np.array_equal(yg, yg2) and np.array_equal(xg, xg2)


@pytest.mark.parametrize("name", ["proj2d", "wide2d", "proj3d", "cone3d"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_matrix_free_small(name, dtype, oracle_cr):
    g = TEST_GEOMETRIES[name]
    rng = np.random.default_rng(7)
    x = rng.uniform(0, 1, g.n_voxels)
    y = rng.uniform(0, 1, g.n_measurements)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    tol = TOL64 if dtype == "f64" else TOL32
    xt = torch.tensor(x, dtype=tdt, device="cuda")
    yt = torch.tensor(y, dtype=tdt, device="cuda")
    xr = xt.double().cpu().numpy()  # oracle sees the same (rounded) inputs
    yr = yt.double().cpu().numpy()
    yg = forward_project_matrix_free(g, "consistent", 1, xt).double().cpu().numpy()
    assert rel_err(yg, oracle_cr.forward_project_matrix_free(g, xr, NTHREADS)) <= tol
    xg = back_project_matrix_free(g, "consistent", 1, yt).double().cpu().numpy()
    assert rel_err(xg, oracle_cr.back_project_matrix_free(g, yr, NTHREADS)) <= tol


def test_matrix_free_matches_csr_small():
    g = TEST_GEOMETRIES["proj3d"]
    w = build_system_matrix(g)
    x = torch.rand(g.n_voxels, dtype=torch.float64, device="cuda")
    y0 = forward_project(w, x)
    y1 = forward_project_matrix_free(g, "consistent", 1, x)
    # test_projector.cpp:104-119 asks 1e-12 where both paths share arithmetic;
    # the matrix-free kernels use the transcendental-free t-formulation, so the
    # bar is the fp64 parity tolerance.
    assert rel_err(y1.cpu().numpy(), y0.cpu().numpy()) <= TOL64


def test_matrix_free_deterministic():
    g = CONFIGS["c1"]
    x = torch.from_numpy(phantom_for("c1", g)).cuda()
    a = forward_project_matrix_free(g, "consistent", 1, x, angles=(0, 720, 7))
    b = forward_project_matrix_free(g, "consistent", 1, x, angles=(0, 720, 7))
    assert torch.equal(a, b)


@pytest.mark.parametrize("seed", list(range(10)))
def test_symmetric_3d_random_clipped_geometries(seed, oracle_cr):
    """Seeded random small cone-beam scans whose volume overshoots the detector
    in rows and columns (clamped row ranges, voxels with no row at all, the
    central row edge L = 0, odd and even n_z, columns of more than one
    z-block): symmetric kernels against the oracle in fp64, fwd and bwd."""
    from paper_2511_12235_b200.projector import symmetry_order
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([4, 6, 8]))
    a = float(rng.uniform(0.6, 2.0))
    g = TEST_GEOMETRIES["cone3d"].with_(
        n_x=n, n_y=n, a=a, b=a, n_z=int(rng.integers(3, 40)), c=float(rng.uniform(0.3, 2.5)),
        s=float(rng.uniform(60.0, 200.0)), d=float(rng.uniform(30.0, 150.0)),
        d_y=float(rng.uniform(0.8, 3.0)), d_z=float(rng.uniform(0.5, 3.0)),
        n_det_y=int(2 * rng.integers(3, 12)), n_det_z=int(2 * rng.integers(2, 14)),
        n_angles=int(rng.choice([8, 16, 24])))
    g.validate()
    assert symmetry_order(g) == 8
    xt = torch.tensor(rng.uniform(0, 1, g.n_voxels), dtype=torch.float64, device="cuda")
    yt = torch.tensor(rng.uniform(0, 1, g.n_measurements), dtype=torch.float64, device="cuda")
    try:
        yg = forward_project_matrix_free(g, "consistent", 1, xt).cpu().numpy()
    except CtsmError as e:  # a shadow wider than the matrix-free kernels hold
        assert e.code == "TooLarge"
        pytest.skip("shadow beyond the matrix-free capacity")
    xg = back_project_matrix_free(g, "consistent", 1, yt).cpu().numpy()
    assert rel_err(yg, oracle_cr.forward_project_matrix_free(g, xt.cpu().numpy(), NTHREADS)) <= TOL64
    assert rel_err(xg, oracle_cr.back_project_matrix_free(g, yt.cpu().numpy(), NTHREADS)) <= TOL64
    # fp32 through the vector-reduction forward and the fp32 accumulators
    yf = forward_project_matrix_free(g, "consistent", 1, xt.float()).double().cpu().numpy()
    xf = back_project_matrix_free(g, "consistent", 1, yt.float()).double().cpu().numpy()
    assert rel_err(yf, yg) <= TOL32 and rel_err(xf, xg) <= TOL32


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_symmetric_back_projection_deterministic(dtype):
    """The 3D symmetric back-projection (orbit shared by a warp pair, two
    partial volumes, member sums folded with plain loads and stores) repeats
    bit for bit in fp64 and in fp32 -- a race on the fold would show here --
    and so does the fp64 forward (fixed point)."""
    g = CONFIGS["c3"].with_(n_x=64, n_y=64, n_z=32, n_det_z=96, n_angles=64)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    gen = torch.Generator().manual_seed(9)
    y = torch.rand(g.n_measurements, generator=gen, dtype=tdt).cuda()
    x = torch.rand(g.n_voxels, generator=gen, dtype=tdt).cuda()
    a = back_project_matrix_free(g, "consistent", 1, y)
    for _ in range(3):
        assert torch.equal(a, back_project_matrix_free(g, "consistent", 1, y))
    if dtype == "f64":
        f = forward_project_matrix_free(g, "consistent", 1, x)
        assert torch.equal(f, forward_project_matrix_free(g, "consistent", 1, x))


# Matrix-free parity at BASELINE sizes is tolerance-checked, so the faster
# glibc-libm oracle is used (crmath costs ~10x on the CPU); angle blocks are
# split into slabs to use all host cores.
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c1_sampled_angles(dtype, oracle_glibc):
    g = CONFIGS["c1"]
    tdt = torch.float64 if dtype == "f64" else torch.float32
    tol = TOL64 if dtype == "f64" else TOL32
    x = torch.from_numpy(phantom_for("c1", g)).to(tdt).cuda()
    y = torch.from_numpy(uniform_sinogram(g.n_measurements, 12346)).to(tdt).cuda()
    angles = np.array([0, 45, 90, 133, 180, 271, 360, 719], np.int32)
    rpa = g.rows_per_angle
    yg = forward_project_matrix_free(g, "consistent", 1, x).double().cpu().numpy()
    ysel = np.concatenate([yg[a * rpa:(a + 1) * rpa] for a in angles])
    yref = oracle_glibc.forward_mf_angles(g, angles, x.double().cpu().numpy(), NTHREADS, split=True)
    assert rel_err(ysel, yref) <= tol
    # A^T y over a strided angle shard
    xg = back_project_matrix_free(g, "consistent", 1, y, angles=(3, 720, 90)).double().cpu().numpy()
    sel = np.arange(3, 720, 90, dtype=np.int32)
    xref = oracle_glibc.back_mf_angles(g, sel, y.double().cpu().numpy(), NTHREADS, split=True)
    assert rel_err(xg, xref) <= tol


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_3d_sampled_angles(cfg, oracle_glibc):
    g = CONFIGS[cfg]
    dt = torch.float64 if cfg == "c2" else torch.float32
    tol = TOL64 if cfg == "c2" else TOL32
    x = torch.from_numpy(phantom_for(cfg, g, dtype=np.float32)).to(dt).cuda()
    angles = np.array([0, 37, 90] if cfg == "c2" else [0, 111], np.int32)
    rpa = g.rows_per_angle
    xr = x.double().cpu().numpy()
    for a in angles:
        yg = forward_project_matrix_free(g, "consistent", 1, x, angles=(int(a), int(a) + 1, 1))
        yg = yg[a * rpa:(a + 1) * rpa].double().cpu().numpy()
        yref = oracle_glibc.forward_mf_angles(g, np.array([a], np.int32), xr, NTHREADS, split=True)
        assert rel_err(yg, yref) <= tol


def test_sirt_small(oracle_cr):
    g = TEST_GEOMETRIES["proj3d"]
    rng = np.random.default_rng(3)
    xt = rng.uniform(0, 1, g.n_voxels)
    y = oracle_cr.forward_project_matrix_free(g, xt, NTHREADS)
    x0 = np.zeros(g.n_voxels)
    xg = sirt(g, y, x0, iters=5)
    xref = oracle_cr.sirt(g, y, x0, 5, NTHREADS)
    assert rel_err(xg, xref) <= 1e-9


# ---- quarter-turn symmetric path ------------------------------------------------
@pytest.mark.parametrize("name", ["c1", "cone3d", "c2"])
def test_symmetric_path_matches_general(name, monkeypatch):
    """The quarter-turn symmetric kernels (4x weight reuse) reproduce the
    general kernels to rounding; orbit shards tile the scan."""
    from paper_2511_12235_b200.projector import quarter_symmetric
    g = CONFIGS[name] if name in CONFIGS else TEST_GEOMETRIES[name]
    assert quarter_symmetric(g)
    gen = torch.Generator().manual_seed(3)
    x = torch.rand(g.n_voxels, generator=gen, dtype=torch.float64).cuda()
    y = torch.rand(g.n_measurements, generator=gen, dtype=torch.float64).cuda()
    if name == "c2":  # keep the general 3D run short: a shard closed under +n/4
        shard = (0, g.n_angles, 30)
    else:
        shard = (0, g.n_angles, 1)
    ys = forward_project_matrix_free(g, "consistent", 1, x, angles=shard)
    xs = back_project_matrix_free(g, "consistent", 1, y, angles=shard)
    monkeypatch.setenv("CTSM_NO_SYMMETRY", "1")
    yg = forward_project_matrix_free(g, "consistent", 1, x, angles=shard)
    xg = back_project_matrix_free(g, "consistent", 1, y, angles=shard)
    assert rel_err(ys.cpu().numpy(), yg.cpu().numpy()) <= 1e-12
    assert rel_err(xs.cpu().numpy(), xg.cpu().numpy()) <= 1e-12
    monkeypatch.delenv("CTSM_NO_SYMMETRY")
    # orbit shards of 3 "ranks" add up to the full projections
    yo = torch.zeros_like(ys)
    xo = torch.zeros_like(xs)
    for r in range(3):
        forward_project_matrix_free(g, "consistent", 1, x, angles=("orbits", r, 3), out=yo)
        xo += back_project_matrix_free(g, "consistent", 1, y, angles=("orbits", r, 3))
    if shard[2] == 1:
        assert rel_err(yo.cpu().numpy(), ys.cpu().numpy()) <= 1e-12
        assert rel_err(xo.cpu().numpy(), xs.cpu().numpy()) <= 1e-12


# ---- dihedral (8-fold) symmetric 2D path ----------------------------------------
@pytest.mark.parametrize("name", ["c1", "wide24", "odd_det", "fine_det", "cone16", "c2"])
def test_dihedral_path_matches_quarter_and_general(name, monkeypatch):
    """The dihedral kernels (8x weight reuse: quarter turns + reflection)
    reproduce the quarter-turn and the general kernels to rounding; orbit
    shards over the dihedral base set tile the scan."""
    from paper_2511_12235_b200.projector import symmetry_order
    if name == "c1":
        g = CONFIGS["c1"]
    elif name == "wide24":
        g = TEST_GEOMETRIES["wide2d"].with_(n_angles=24)
    elif name == "cone16":  # 3D, 16 angles: base angles 0, 1, 2 (1 has all 8 images)
        g = TEST_GEOMETRIES["cone3d"].with_(n_angles=16)
    elif name == "c2":
        g = CONFIGS["c2"]
    elif name == "odd_det":  # fewer detector cells than the shadow: clipped cells
        g = TEST_GEOMETRIES["wide2d"].with_(n_angles=16, n_det_y=60)
    else:  # tile shadows wider than the forward kernel's shared-memory window
        g = TEST_GEOMETRIES["wide2d"].with_(n_angles=16, d_y=0.25, n_det_y=1000)
    assert symmetry_order(g) == 8
    gen = torch.Generator().manual_seed(4)
    x = torch.rand(g.n_voxels, generator=gen, dtype=torch.float64).cuda()
    y = torch.rand(g.n_measurements, generator=gen, dtype=torch.float64).cuda()
    res = {}
    for mode in ("d8", "quarter", "general"):
        monkeypatch.delenv("CTSM_NO_DIHEDRAL", raising=False)
        monkeypatch.delenv("CTSM_NO_SYMMETRY", raising=False)
        if mode == "quarter":
            monkeypatch.setenv("CTSM_NO_DIHEDRAL", "1")
            assert symmetry_order(g) == 4
        elif mode == "general":
            monkeypatch.setenv("CTSM_NO_SYMMETRY", "1")
        res[mode] = (forward_project_matrix_free(g, "consistent", 1, x).cpu().numpy(),
                     back_project_matrix_free(g, "consistent", 1, y).cpu().numpy())
    monkeypatch.delenv("CTSM_NO_SYMMETRY", raising=False)
    for other in ("quarter", "general"):
        assert rel_err(res["d8"][0], res[other][0]) <= 1e-12
        assert rel_err(res["d8"][1], res[other][1]) <= 1e-12
    # f32 through the dihedral kernels
    yf = forward_project_matrix_free(g, "consistent", 1, x.float()).cpu().numpy()
    assert rel_err(yf, res["general"][0]) <= 1e-5
    # orbit shards of 3 "ranks" add up to the full projections
    yo = torch.zeros(g.n_measurements, dtype=torch.float64, device="cuda")
    xo = torch.zeros(g.n_voxels, dtype=torch.float64, device="cuda")
    for r in range(3):
        forward_project_matrix_free(g, "consistent", 1, x, angles=("orbits", r, 3), out=yo)
        xo += back_project_matrix_free(g, "consistent", 1, y, angles=("orbits", r, 3))
    assert rel_err(yo.cpu().numpy(), res["d8"][0]) <= 1e-12
    assert rel_err(xo.cpu().numpy(), res["d8"][1]) <= 1e-12


@pytest.mark.parametrize("name", ["cone16", "c3_slab"])
def test_f32_3d_vector_reduction_forward(name, monkeypatch):
    """fp32 dihedral 3D forward (vector float reductions into interleaved
    rows, then un-interleaved): matches the fixed-point fp32 path and the fp64
    general kernels within the fp32 bar, and orbit shards tile the scan."""
    if name == "cone16":
        g = TEST_GEOMETRIES["cone3d"].with_(n_angles=16)
    else:  # C3 detector / grid pitch on a thin slab of angles' orbits
        g = CONFIGS["c3"].with_(n_x=64, n_y=64, n_z=32, n_det_z=96, n_angles=64)
    gen = torch.Generator().manual_seed(5)
    x = torch.rand(g.n_voxels, generator=gen, dtype=torch.float64).cuda()
    yf = forward_project_matrix_free(g, "consistent", 1, x.float())
    monkeypatch.setenv("CTSM_FWD3_FIXED", "1")
    yx = forward_project_matrix_free(g, "consistent", 1, x.float())
    monkeypatch.delenv("CTSM_FWD3_FIXED")
    y64 = forward_project_matrix_free(g, "consistent", 1, x)
    assert rel_err(yf.cpu().numpy(), yx.cpu().numpy()) <= 1e-5
    assert rel_err(yf.cpu().numpy(), y64.cpu().numpy()) <= 1e-5
    yo = torch.zeros_like(yf)
    for r in range(3):
        forward_project_matrix_free(g, "consistent", 1, x.float(), angles=("orbits", r, 3), out=yo)
    assert rel_err(yo.cpu().numpy(), yf.cpu().numpy()) <= 1e-6
