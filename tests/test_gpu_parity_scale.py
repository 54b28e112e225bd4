"""BASELINE-scale parity through the PRODUCTION kernels (GPU vs CPU oracle).

The full-scan projections of C3/C4 run the dihedral + z-mirror kernels
(`fwd3d_sym_kernel` / `fwd3d_mf_d8_f32`, `bwd3d_sym_kernel`; asserted through
ctsm_last_kernel_path), never the per-angle general kernels. Rows of sampled
angles -- 0, n/4, n/2, 3n/4 (the flat-source branch and its quarter-turn
images) plus 4 strided angles -- are compared with the C restatement
(`port_glibc`, pinned bit-exactly to the unmodified reference in
tests/test_oracle_pin.py) on the same fp32-rounded inputs:

  max|got - ref| <= tol * max(1, max|ref|)      (test_projector.cpp:117)

with tol = 1e-5 for fp32 (BASELINE.json north_star). The per-element relative
error on |ref| > 1e-3 max|ref| is reported; with
CTSM_PARITY_REPORT=<file> every case appends one JSON line there.

C4 (512^3, 1440 angles) evaluates the oracle on three z-slab bands (top,
centre, bottom; the outer slabs are where the atoms' cancellation is worst,
SURVEY.md §0 fact 5): x is nonzero only there for A x, and A^T y is compared
on those voxels. The GPU still runs the whole volume through the production
kernels.

The 3D CSR flip report compares GPU angle blocks of C2 with the reference AS
SHIPPED (glibc libm, `ref_glibc`, the unmodified reference sources): the GPU
CSR is bit-identical to the correctly rounded oracle (test_gpu_parity.py), and
against glibc every sparsity flip must lie in the cancellation-noise band
|w| < 1e-11 with |dw| <= 1e-10 on common entries (
drop threshold weights3d.cpp:453).
"""
import json
import os

import numpy as np
import pytest

import pyoracle
from paper_2511_12235_b200 import (CONFIGS, back_project_matrix_free, build_system_matrix,
                                   forward_project_matrix_free, sirt)
from paper_2511_12235_b200.phantoms import phantom_for
from paper_2511_12235_b200.projector import Context, last_kernel_path

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NTHREADS = max(1, os.cpu_count() or 1)
TOL32 = 1e-5
P_DIHEDRAL, P_ZMIRROR, P_F32VEC = 8, 16, 32


def sampled_angles(n: int) -> np.ndarray:
    """0, n/4, n/2, 3n/4 and 4 strided angles."""
    strided = [int(n * f) + 1 for f in (0.07, 0.31, 0.58, 0.86)]
    return np.array(sorted({0, n // 4, n // 2, 3 * n // 4, *strided}), np.int32)


def parity(got, ref, tol, name):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    mx = float(np.max(np.abs(ref)))
    err = float(np.max(np.abs(got - ref))) / max(1.0, mx)
    sig = np.abs(ref) > 1e-3 * mx
    rel = float(np.max(np.abs(got[sig] - ref[sig]) / np.abs(ref[sig]))) if sig.any() else 0.0
    line = {"case": name, "max_abs_err_over_max1": err, "tol": tol, "max_ref": mx,
            "max_rel_err_significant": rel, "n_significant": int(sig.sum()), "n": int(ref.size)}
    print(json.dumps(line))
    rep = os.environ.get("CTSM_PARITY_REPORT")
    if rep:
        with open(rep, "a") as fh:
            fh.write(json.dumps(line) + "\n")
    assert err <= tol, line
    return line


def rows_of(y, g, angles):
    rpa = g.rows_per_angle
    return torch.cat([y[int(a) * rpa:(int(a) + 1) * rpa] for a in angles])


def assert_production_path():
    p = last_kernel_path()
    assert p & P_DIHEDRAL and p & P_ZMIRROR, f"not the dihedral z-mirror kernels (path bits {p})"
    return p


# ---- C3: 256^3, 512x384, 720 angles, fp32 -----------------------------------
def test_c3_production_kernels_vs_oracle(oracle_glibc):
    g = CONFIGS["c3"]
    angles = sampled_angles(g.n_angles)
    x = torch.from_numpy(phantom_for("c3", g, dtype=np.float32)).cuda()
    y = forward_project_matrix_free(g, "consistent", 1, x)
    assert assert_production_path() & P_F32VEC  # red.global.add.v4.f32 row runs
    yref = oracle_glibc.forward_mf_angles(g, angles, x.double().cpu().numpy(), NTHREADS,
                                          split=True)
    parity(rows_of(y, g, angles).cpu().numpy(), yref, TOL32, "c3 fwd f32 (d8 + z mirror)")
    del y
    # A^T y of the sampled angles: y is U[0, 1) on their rows and 0 elsewhere,
    # so the full-scan production back-projection equals theirs
    gen = np.random.Generator(np.random.PCG64(12346))
    rpa = g.rows_per_angle
    yrows = gen.random(angles.size * rpa).astype(np.float32)
    ys = torch.zeros(g.n_measurements, dtype=torch.float32, device="cuda")
    for i, a in enumerate(angles):
        ys[int(a) * rpa:(int(a) + 1) * rpa] = torch.from_numpy(yrows[i * rpa:(i + 1) * rpa])
    xb = back_project_matrix_free(g, "consistent", 1, ys)
    assert_production_path()
    xref = oracle_glibc.back_mf_angles_slabs(g, angles, 0, g.n_z, yrows.astype(np.float64),
                                             NTHREADS)
    parity(xb.cpu().numpy(), xref, TOL32, "c3 bwd f32 (d8 + z mirror)")


# ---- C4: 512^3, 1024x768, 1440 angles, fp32 (three slab bands) ---------------
C4_BANDS = ((0, 16), (248, 264), (496, 512))


def test_c4_production_kernels_vs_oracle_slabs(oracle_glibc):
    g = CONFIGS["c4"]
    angles = sampled_angles(g.n_angles)
    plane = g.n_x * g.n_y
    gen = torch.Generator(device="cuda").manual_seed(12345)
    x = torch.zeros(g.n_voxels, dtype=torch.float32, device="cuda")
    for z0, z1 in C4_BANDS:  # seeded U[0.005, 0.02) attenuations in the bands
        x[z0 * plane:z1 * plane] = 0.005 + 0.015 * torch.rand(
            (z1 - z0) * plane, generator=gen, device="cuda")
    y = forward_project_matrix_free(g, "consistent", 1, x)
    assert assert_production_path() & P_F32VEC
    ysel = rows_of(y, g, angles).cpu().numpy()
    del y
    xh = x.double().cpu().numpy()
    yref = np.zeros(ysel.size)
    for z0, z1 in C4_BANDS:
        yref += oracle_glibc.forward_mf_angles_slabs(g, angles, z0, z1, xh, NTHREADS)
    parity(ysel, yref, TOL32, "c4 fwd f32 (d8 + z mirror), 3 slab bands")
    del x, xh
    rpa = g.rows_per_angle
    yrows = np.random.Generator(np.random.PCG64(12346)).random(angles.size * rpa).astype(np.float32)
    ys = torch.zeros(g.n_measurements, dtype=torch.float32, device="cuda")
    for i, a in enumerate(angles):
        ys[int(a) * rpa:(int(a) + 1) * rpa] = torch.from_numpy(yrows[i * rpa:(i + 1) * rpa])
    xb = back_project_matrix_free(g, "consistent", 1, ys)
    assert_production_path()
    del ys
    xb = xb.cpu().numpy()
    got, ref = [], []
    for z0, z1 in C4_BANDS:
        xr = oracle_glibc.back_mf_angles_slabs(g, angles, z0, z1, yrows.astype(np.float64),
                                               NTHREADS)
        got.append(xb[z0 * plane:z1 * plane])
        ref.append(xr[z0 * plane:z1 * plane])
    parity(np.concatenate(got), np.concatenate(ref), TOL32,
           "c4 bwd f32 (d8 + z mirror), 3 slab bands")


def test_c4_pitch_sirt_slab(oracle_glibc):
    """2 SIRT iterations at C4's voxel and detector pitch (depth / pitch ~ 2000,
    where the atoms cancel worst) on a reduced grid and angle count, through
    the production kernels, against the oracle's SIRT restatement."""
    g = CONFIGS["c4"].with_(n_x=128, n_y=128, n_z=16, n_angles=64)
    rng = np.random.default_rng(11)
    xt = rng.uniform(0.005, 0.02, g.n_voxels).astype(np.float32)
    y = forward_project_matrix_free(g, "consistent", 1, torch.from_numpy(xt).cuda())
    assert assert_production_path() & P_F32VEC
    yh = y.cpu().numpy()
    xg = sirt(g, y, None, iters=2)
    xref = oracle_glibc.sirt(g, yh.astype(np.float64), np.zeros(g.n_voxels), 2, NTHREADS)
    parity(xg.cpu().numpy(), xref, TOL32, "c4-pitch SIRT-2 f32 (128^2 x 16, 64 angles)")


# ---- 1 rank vs N ranks (orbit shards), C3 fp32 --------------------------------
@pytest.mark.parametrize("world", [2, 8])
def test_c3_shards_match_single_rank(world):
    """The N-rank results (orbit shards; A x rows disjoint, A^T y partials
    summed as the all-reduce would) match the 1-rank results within the fp32
    bar. Each shard runs the production kernels on this one GPU in turn."""
    g = CONFIGS["c3"]
    gen = torch.Generator(device="cuda").manual_seed(21)
    x = torch.rand(g.n_voxels, generator=gen, device="cuda")
    y = torch.rand(g.n_measurements, generator=gen, device="cuda")
    y1 = forward_project_matrix_free(g, "consistent", 1, x)
    x1 = back_project_matrix_free(g, "consistent", 1, y)
    yn = torch.zeros_like(y1)
    xn = torch.zeros_like(x1)
    for r in range(world):
        forward_project_matrix_free(g, "consistent", 1, x, angles=("orbits", r, world), out=yn)
        assert assert_production_path()
        xn += back_project_matrix_free(g, "consistent", 1, y, angles=("orbits", r, world))
    ey = float((yn - y1).abs().max()) / max(1.0, float(y1.abs().max()))
    ex = float((xn - x1).abs().max()) / max(1.0, float(x1.abs().max()))
    print(json.dumps({"case": f"c3 f32 {world} orbit shards vs 1", "fwd": ey, "bwd": ex}))
    assert ey <= TOL32 and ex <= TOL32


# ---- 3D CSR sparsity flips vs the reference as shipped (glibc) ----------------
@pytest.mark.parametrize("ip", [0, 37, 90, 111, 181, 300])
def test_csr_c2_flips_vs_reference_glibc(ip):
    if not pyoracle.available("ref_glibc"):
        pytest.skip("oracle/_ref not built")
    ref = pyoracle.load("ref_glibc")
    g = CONFIGS["c2"]
    w = build_system_matrix(g, angle_range=(ip, ip + 1), memory_budget_bytes=1 << 40)
    rs, col, val = w.to_host()
    rows = np.repeat(np.arange(rs.size - 1, dtype=np.uint64), np.diff(rs).astype(np.int64))
    kg = (rows << np.uint64(32)) | col.astype(np.uint64)
    rr, rc, rw = ref.angle_block_entries(g, ip, threads=NTHREADS)
    kr = (rr.astype(np.uint64) << np.uint64(32)) | rc.astype(np.uint64)
    o = np.argsort(kr, kind="stable")
    kr, rw = kr[o], rw[o]
    assert np.all(np.diff(kg.astype(np.int64)) > 0) or kg.size < 2  # rows ascending, cols ascending
    common, ig, ir = np.intersect1d(kg, kr, assume_unique=True, return_indices=True)
    only_g = np.setdiff1d(np.arange(kg.size), ig, assume_unique=True)
    only_r = np.setdiff1d(np.arange(kr.size), ir, assume_unique=True)
    dw = float(np.max(np.abs(val[ig] - rw[ir]))) if common.size else 0.0
    flip_w = np.concatenate([val[only_g], rw[only_r]])
    line = {"case": f"c2 CSR angle {ip} vs ref_glibc", "nnz_gpu": int(kg.size),
            "nnz_ref": int(kr.size), "only_gpu": int(only_g.size), "only_ref": int(only_r.size),
            "max_flipped_w": float(np.max(flip_w)) if flip_w.size else 0.0,
            "max_dw_common": dw}
    print(json.dumps(line))
    rep = os.environ.get("CTSM_PARITY_REPORT")
    if rep:
        with open(rep, "a") as fh:
            fh.write(json.dumps(line) + "\n")
    assert line["max_flipped_w"] < 1e-11, line
    assert dw <= 1e-10, line


def test_c2_full_matrix_hashes():
    """The WHOLE C2 system matrix (360 angle blocks, 4.6 G entries) against the
    unmodified reference compiled with the correctly rounded libm: entry count
    and an order-independent 64-bit hash of (row, column, weight bits) of
    every angle block (tests/golden/c2_block_hashes_ref_cr.npz, generated by
    tests/golden/make_c2_hashes.py from oracle/_ref). One differing bit in any
    of the 4.6 G weights, columns or row offsets changes a block hash."""
    fx_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "c2_block_hashes_ref_cr.npz")
    if not os.path.exists(fx_path):
        pytest.skip("fixture not generated")
    fx = np.load(fx_path)
    g = CONFIGS["c2"]
    w = build_system_matrix(g, memory_budget_bytes=1 << 40)
    assert w.nnz() == int(fx["nnz"].sum())
    rpa = g.rows_per_angle
    rs = w.row_start
    k1 = 0x9E3779B97F4A7C15 - (1 << 64)  # the fixture's constants as int64
    k2 = 0xC2B2AE3D27D4EB4F - (1 << 64)
    ar = torch.arange(rpa, device=rs.device, dtype=torch.int64)
    bad = []
    for ip in range(g.n_angles):
        blk = rs[ip * rpa:(ip + 1) * rpa + 1]
        lo, hi = int(blk[0].item()), int(blk[-1].item())
        if hi - lo != int(fx["nnz"][ip]):
            bad.append((ip, "nnz", hi - lo, int(fx["nnz"][ip])))
            continue
        raster = torch.repeat_interleave(ar, blk[1:] - blk[:-1])
        key = (raster << 32) | (w.col[lo:hi].to(torch.int64) & 0xFFFFFFFF)
        m = (w.val[lo:hi].view(torch.int64) * k1) ^ (key * k2)
        h = int(m.sum().item()) & ((1 << 64) - 1)
        if h != int(fx["hash"][ip]):
            bad.append((ip, "hash", hex(h), hex(int(fx["hash"][ip]))))
    line = {"case": "c2 full CSR vs ref_cr block hashes", "blocks": g.n_angles, "nnz": w.nnz(),
            "mismatching_blocks": len(bad)}
    print(json.dumps(line))
    rep = os.environ.get("CTSM_PARITY_REPORT")
    if rep:
        with open(rep, "a") as fh:
            fh.write(json.dumps(line) + "\n")
    assert not bad, bad[:5]
