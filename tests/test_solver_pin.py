"""Pins the solver oracles (oracle/pyoracle.py: nag_tikhonov_np,
spectral_norm_power_np, csr_forward/csr_back) to the compiled reference
(solver.cpp:17-75, projector.cpp:203-280, phantoms.cpp:78-87) on CPU, and
the product's host-side normal_samples to the reference's."""
import numpy as np
import pytest

import pyoracle
from paper_2511_12235_b200.geometry import TEST_GEOMETRIES
from paper_2511_12235_b200.phantoms import normal_samples

needs_ref = pytest.mark.skipif(not pyoracle.available("ref_glibc"), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("seed", [7, 12345])
def test_normal_samples_match_reference(seed):
    ref = pyoracle.load("ref_glibc")
    assert np.array_equal(normal_samples(2000, seed), ref.normal_samples(2000, seed))


@needs_ref
def test_numpy_solver_restatement_is_bit_exact():
    ref = pyoracle.load("ref_glibc")
    g = TEST_GEOMETRIES["proj2d"]
    m = ref.build_system_matrix(g)
    n = g.n_voxels
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, n)
    y = rng.uniform(0, 1, g.n_measurements)
    # the appliers (projector.cpp:203-233)
    assert np.array_equal(pyoracle.csr_forward(m, x), ref.forward_project_matrix_free(g, x))
    # spectral norm (projector.cpp:262-280)
    v0 = ref.normal_samples(n, 7)
    nrm = ref.spectral_norm_power(g, 20, 7)
    assert pyoracle.spectral_norm_power_np(m, n, v0, 20) == nrm
    # NAG on the scaled matrix (solver.cpp:17-75)
    ms = pyoracle.Csr(m.row_start, m.col, m.val * (1.0 / nrm))
    p = pyoracle.csr_forward(ms, x)
    u_ref, it_ref, conv_ref, tr_ref = ref.nag_tikhonov(g, p, 1e-3, 40, 1e-30, scale=1.0 / nrm,
                                                        keep_trace=True)
    u, it, conv, tr = pyoracle.nag_tikhonov_np(ms, n, p, 1e-3, 40, 1e-30, keep_trace=True)
    assert (it, conv) == (it_ref, conv_ref) == (40, False)
    assert np.array_equal(u, u_ref)
    assert np.array_equal(tr, tr_ref)
    # the back projection used inside matches back_project bit for bit too
    assert np.array_equal(pyoracle.csr_back(m, y, n), ref.back_project_csr(g, y))
