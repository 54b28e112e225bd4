"""K4 (back_project, projector.cpp:219-233) with the cached column-sum bound:
the bound is computed once per matrix and dropped when the values change
(scale_values through the C-ABI, or any in-place torch op on the arrays).
Power-of-two value scalings are exact end to end, so the results must scale
bit-exactly; a stale bound would break that (or overflow the fixed point)."""
import numpy as np
import pytest

from paper_2511_12235_b200 import TEST_GEOMETRIES, back_project, build_system_matrix
from paper_2511_12235_b200.projector import scale_values

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["proj2d", "proj3d"])
def test_back_project_cached_bound(name):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    y = torch.from_numpy(np.random.default_rng(3).random(g.n_measurements)).cuda()
    x1 = back_project(w, y).cpu().numpy()
    assert getattr(w, "_colsum_cache", None) is not None
    # repeated call on the cached bound: identical bits
    assert np.array_equal(back_project(w, y).cpu().numpy(), x1)
    # (parity with the oracle's CSR scatter: test_gpu_parity.py::test_spmv_and_transpose)
    scale_values(w, 2.0)
    assert np.array_equal(back_project(w, y).cpu().numpy(), 2.0 * x1)
    w.val.mul_(4.0)  # in-place torch op: version counter bump
    assert np.array_equal(back_project(w, y).cpu().numpy(), 8.0 * x1)
