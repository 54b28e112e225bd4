"""Host-buffer C-ABI calls (ctsm_{forward,back}_project_matrix_free_host, the
reference's value-semantics projector.cpp:235-260 shape, used by bench.py's
e2e leg): equal to the device-resident calls, also when A x and A^T y run
concurrently from two host threads on two contexts (each context owns its
scratch, status word and non-blocking stream)."""
import ctypes
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
