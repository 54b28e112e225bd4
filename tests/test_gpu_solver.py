"""Device solver parity: spectral_norm_power and
nag_tikhonov through the C-ABI against the numpy restatement of
solver.cpp / projector.cpp:262-280 (oracle/pyoracle.py, pinned bit-exact to
the compiled reference in tests/test_solver_pin.py).

Tolerances: the device appliers sum in a different order than the
reference's serial loops (fixed-point A^T, tree reductions), so iterates
agree to rounding: 1e-10 relative after 40 iterations."""
import numpy as np
import pytest

import pyoracle
from paper_2511_12235_b200 import TEST_GEOMETRIES, CtsmError, build_system_matrix, scale_values
from paper_2511_12235_b200.phantoms import normal_samples
from paper_2511_12235_b200.projector import spectral_norm_power, spectral_norm_power_matrix_free
from paper_2511_12235_b200.solver import (SolveOptions, nag_tikhonov,
                                          nag_tikhonov_matrix_free)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def host_csr(w):
    rs, col, val = w.to_host()
    return pyoracle.Csr(rs, col, val)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b))))


@pytest.mark.parametrize("name", ["proj2d", "wide2d", "proj3d"])
def test_spectral_norm_and_nag_match_restatement(name):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    c = host_csr(w)
    n = g.n_voxels
    nrm_ref = pyoracle.spectral_norm_power_np(c, n, normal_samples(n, 7), 30)
    nrm = spectral_norm_power(w, 30, 7)
    assert abs(nrm - nrm_ref) <= 1e-12 * nrm_ref
    # matrix-free operator: same norm to rounding
    assert abs(spectral_norm_power_matrix_free(g, 30, 7) - nrm_ref) <= 1e-10 * nrm_ref
    # NAG on the normalised matrix
    scale_values(w, 1.0 / nrm)
    cs = pyoracle.Csr(c.row_start, c.col, c.val * (1.0 / nrm))
    x = np.random.default_rng(11).uniform(0, 1, n)
    p = pyoracle.csr_forward(cs, x)
    opt = SolveOptions(lam=1e-3, max_iter=40, tol=1e-30)
    u_ref, it_ref, conv_ref, tr_ref = pyoracle.nag_tikhonov_np(cs, n, p, 1e-3, 40, 1e-30, True)
    r = nag_tikhonov(w, p, opt, keep_trace=True)
    assert (r.iterations, r.converged) == (it_ref, conv_ref)
    assert rel(r.u.cpu().numpy(), u_ref) <= 1e-10
    tr = np.array([(t.iter, t.objective, t.grad_norm_sq) for t in r.trace])
    assert np.array_equal(tr[:, 0], tr_ref[:, 0])
    assert rel(tr[:, 1], tr_ref[:, 1]) <= 1e-10
    assert np.max(np.abs(tr[:, 2] - tr_ref[:, 2]) / tr_ref[:, 2]) <= 1e-8
    # with the CSC transpose kept beside the CSR the solvers' W^T gathers:
    # the same fixed-point integers, so the same iterates bit for bit
    from paper_2511_12235_b200 import build_transpose
    build_transpose(w)
    rt = nag_tikhonov(w, p, opt)
    assert torch.equal(rt.u, r.u) and rt.iterations == r.iterations
    assert spectral_norm_power(w, 30, 7) == 1.0 * spectral_norm_power(w, 30, 7)
    # matrix-free NAG on W = A / ||A||
    rm = nag_tikhonov_matrix_free(g, p, opt, scale=1.0 / nrm)
    assert rm.iterations == 40
    assert rel(rm.u.cpu().numpy(), u_ref) <= 1e-9


def test_nag_converges_like_reference():
    g = TEST_GEOMETRIES["proj2d"]
    w = build_system_matrix(g)
    nrm = spectral_norm_power(w, 50, 7)
    scale_values(w, 1.0 / nrm)
    c = host_csr(w)
    n = g.n_voxels
    p = pyoracle.csr_forward(c, np.random.default_rng(2).uniform(0, 1, n))
    u_ref, it_ref, conv_ref, _ = pyoracle.nag_tikhonov_np(c, n, p, 1e-2, 500, 1e-6)
    r = nag_tikhonov(w, p, SolveOptions(lam=1e-2, max_iter=500, tol=1e-6))
    assert conv_ref and r.converged
    assert abs(r.iterations - it_ref) <= 1  # the stop test compares rounded sums
    assert r.iterations < 500


def test_solver_errors():
    g = TEST_GEOMETRIES["proj2d"]
    w = build_system_matrix(g)
    p = np.zeros(g.n_measurements)
    with pytest.raises(CtsmError) as e:
        nag_tikhonov(w, p, SolveOptions(lam=-1.0))
    assert e.value.code == "InvalidConfig"
    with pytest.raises(CtsmError) as e:
        nag_tikhonov(w, p[:-1])
    assert e.value.code == "DimensionMismatch"
    scale_values(w, 0.0)
    with pytest.raises(CtsmError) as e:
        spectral_norm_power(w, 3, 7)
    assert e.value.code == "ZeroMatrix"
    with pytest.raises(CtsmError) as e:
        scale_values(w, float("inf"))
    assert e.value.code == "NonFinite"
