"""Small-geometry tour of every kernel family for compute-sanitizer
(tools/sanitize.sh): CSR builds (single evaluation and count / fill), CSR
appliers, matrix-free projectors (general, quarter-turn, dihedral, z-mirror;
fp64 and fp32), SIRT, ray modes, the weight API, solver and CSM1 round trip."""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_12235_b200 import (TEST_GEOMETRIES, angle_block_entries, back_project,  # noqa: E402
                                   back_project_matrix_free, build_system_matrix, forward_project,
                                   forward_project_matrix_free, sirt, spectral_norm_power,
                                   weights_batch)
from paper_2511_12235_b200 import io as cio  # noqa: E402

rng = np.random.default_rng(3)
for name in ("proj2d", "wide2d", "proj3d", "cone3d"):
    g = TEST_GEOMETRIES[name]
    w = build_system_matrix(g)
    w2 = build_system_matrix(g, two_pass=True)
    assert torch.equal(w.col, w2.col)
    x = torch.tensor(rng.uniform(0, 1, g.n_voxels), device="cuda")
    y = torch.tensor(rng.uniform(0, 1, g.n_measurements), device="cuda")
    forward_project(w, x)
    back_project(w, y)
    for dt in (torch.float64, torch.float32):
        forward_project_matrix_free(g, "consistent", 1, x.to(dt))
        back_project_matrix_free(g, "consistent", 1, y.to(dt))
        forward_project_matrix_free(g, "consistent", 1, x.to(dt), angles=(1, g.n_angles, 2))
        back_project_matrix_free(g, "consistent", 1, y.to(dt), angles=(1, g.n_angles, 2))
        sirt(g, y.to(dt), None, 2)
    for mode, k in (("line", 1), ("multiline", 2)):
        build_system_matrix(g, mode, k)
        forward_project_matrix_free(g, mode, k, x)
        back_project_matrix_free(g, mode, k, y)
        angle_block_entries(g, mode, k, 1)
    angle_block_entries(g, "consistent", 1, 1)
    n = 64
    weights_batch(g, rng.integers(0, g.n_x, n), rng.integers(0, g.n_y, n),
                  rng.integers(0, g.n_z, n), rng.uniform(0, 6, n))
    spectral_norm_power(w, 5, 7)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.csm")
        cio.write_matrix(p, w)
        cio.read_matrix(p)
    torch.cuda.synchronize()
    print("ok", name, w.nnz(), flush=True)
print("sanitize tour done")
