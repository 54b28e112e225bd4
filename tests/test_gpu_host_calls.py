"""Host-buffer C-ABI calls (ctsm_{forward,back}_project_matrix_free_host, the
reference's value-semantics projector.cpp:235-260 shape, used by bench.py's
e2e leg): equal to the device-resident calls, also when A x and A^T y run
concurrently from two host threads on two contexts (each context owns its
scratch, status word and non-blocking stream)."""
import ctypes
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2511_12235_b200 import (CONFIGS, TEST_GEOMETRIES, back_project_matrix_free,
                                   forward_project_matrix_free, _lib)
from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
from paper_2511_12235_b200.projector import Context

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _host_fwd(ctx, g, x):
    y = np.empty(g.n_measurements, np.float64)
    cg = g.to_c()
    _lib.check(_lib.lib().ctsm_forward_project_matrix_free_host(
        ctx.handle, ctypes.byref(cg), ctypes.c_void_p(x.ctypes.data), ctypes.c_void_p(y.ctypes.data)))
    return y


def _host_bwd(ctx, g, y):
    x = np.empty(g.n_voxels, np.float64)
    cg = g.to_c()
    _lib.check(_lib.lib().ctsm_back_project_matrix_free_host(
        ctx.handle, ctypes.byref(cg), ctypes.c_void_p(y.ctypes.data), ctypes.c_void_p(x.ctypes.data)))
    return x


@pytest.mark.parametrize("name", ["proj2d", "c1"])
def test_host_calls_concurrent_bitequal(name):
    g = TEST_GEOMETRIES[name] if name in TEST_GEOMETRIES else CONFIGS[name]
    x = np.ascontiguousarray(phantom_for(name, g, dtype=np.float64)) if name in CONFIGS else \
        np.random.default_rng(7).random(g.n_voxels)
    y = np.ascontiguousarray(uniform_sinogram(g.n_measurements, 12346)) if name in CONFIGS \
        else np.random.default_rng(8).random(g.n_measurements)
    dev_y = forward_project_matrix_free(g, "consistent", 1, torch.from_numpy(x).cuda()).cpu().numpy()
    dev_x = back_project_matrix_free(g, "consistent", 1, torch.from_numpy(y).cuda()).cpu().numpy()
    ca, cb = Context(0), Context(0)
    try:
        # serial
        assert np.array_equal(_host_fwd(ca, g, x), dev_y)
        assert np.array_equal(_host_bwd(cb, g, y), dev_x)
        # concurrent, repeated (fp64 paths are deterministic on any schedule)
        with ThreadPoolExecutor(max_workers=1) as pool:
            for _ in range(3):
                fut = pool.submit(_host_bwd, cb, g, y)
                yf = _host_fwd(ca, g, x)
                xb = fut.result()
                assert np.array_equal(yf, dev_y)
                assert np.array_equal(xb, dev_x)
    finally:
        ca.close()
        cb.close()


def _host_f32(ctx, g, fn, src, n_out):
    out = np.empty(n_out, np.float32)
    cg = g.to_c()
    _lib.check(getattr(_lib.lib(), fn)(ctx.handle, ctypes.byref(cg),
                                       ctypes.c_void_p(src.ctypes.data),
                                       ctypes.c_void_p(out.ctypes.data)))
    return out


@pytest.mark.parametrize("name", ["cone16", "c3_slab"])
def test_host_calls_f32(name):
    """fp32 overloads (ctsm_*_project_matrix_free_host_f32) =
    the device-resident fp32 calls: A^T y bit-equal (fixed-order gathers), A x
    within 1e-6 (the fp32 3D forward's vector reductions are order-dependent
    at fp32 rounding)."""
    if name == "cone16":
        g = TEST_GEOMETRIES["cone3d"].with_(n_angles=16)
    else:
        g = CONFIGS["c3"].with_(n_x=64, n_y=64, n_z=32, n_det_z=96, n_angles=64)
    rng = np.random.default_rng(9)
    x = rng.random(g.n_voxels).astype(np.float32)
    y = rng.random(g.n_measurements).astype(np.float32)
    dev_y = forward_project_matrix_free(g, "consistent", 1, torch.from_numpy(x).cuda()).cpu().numpy()
    dev_x = back_project_matrix_free(g, "consistent", 1, torch.from_numpy(y).cuda()).cpu().numpy()
    ca, cb = Context(0), Context(0)
    try:
        with ThreadPoolExecutor(max_workers=1) as pool:
            fut = pool.submit(_host_f32, cb, g, "ctsm_back_project_matrix_free_host_f32", y,
                              g.n_voxels)
            yf = _host_f32(ca, g, "ctsm_forward_project_matrix_free_host_f32", x, g.n_measurements)
            xb = fut.result()
        assert np.max(np.abs(yf - dev_y)) <= 1e-6 * max(1.0, float(np.max(np.abs(dev_y))))
        assert np.array_equal(xb, dev_x)
    finally:
        ca.close()
        cb.close()


def test_bench_two_ranks_functional(tmp_path):
    """bench.py --gpus 2 launches two ranks (orbit shards, all-reduce of the
    A^T y volume, max-over-ranks timing, one JSON line from rank 0). On this
    one-GPU box both ranks share cuda:0 and reduce through gloo
    (CTSM_BENCH_SHARE_GPU=1): a check of the N-rank code path on the real
    kernels, not a measurement."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CTSM_BENCH_SHARE_GPU="1")
    for extra in (["--config", "c1", "--dtype", "f32"],
                  ["--config", "c1", "--mode", "sirt", "--no-e2e"]):
        r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps",
                            "2", "--warmup", "1", "--no-cpu", "--no-clocks"] + extra,
                           capture_output=True, text=True, timeout=900, env=env, cwd=root)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, r.stdout
        line = json.loads(lines[0])
        assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
        assert "x2" in line["config"]["parallelism"]
        if "--no-e2e" not in extra:
            assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
