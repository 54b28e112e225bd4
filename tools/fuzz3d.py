"""One-off fuzz of the symmetric 3D kernels on seeded random clipped
geometries (the generator of tests/test_gpu_parity.py::
test_symmetric_3d_random_clipped_geometries, more seeds, order 4 and 8):
python tools/fuzz3d.py [n_seeds]."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402
from paper_2511_12235_b200 import (TEST_GEOMETRIES, CtsmError, back_project_matrix_free,  # noqa: E402
                                   forward_project_matrix_free)

orc = pyoracle.load("port_cr")


def rel(a, b):
    return float(np.max(np.abs(a - b))) / max(1.0, float(np.max(np.abs(b))))


n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 60
worst = 0.0
skipped = 0
for seed in range(n_seeds):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.choice([4, 6, 8, 10]))
    a = float(rng.uniform(0.6, 2.0))
    g = TEST_GEOMETRIES["cone3d"].with_(
        n_x=n, n_y=n, a=a, b=a, n_z=int(rng.integers(1, 70)), c=float(rng.uniform(0.2, 2.5)),
        s=float(rng.uniform(60.0, 200.0)), d=float(rng.uniform(30.0, 150.0)),
        d_y=float(rng.uniform(0.8, 3.0)), d_z=float(rng.uniform(0.4, 3.0)),
        n_det_y=int(2 * rng.integers(3, 12)), n_det_z=int(2 * rng.integers(1, 20)),
        n_angles=int(rng.choice([4, 8, 12, 16, 24])))
    try:
        g.validate()
    except Exception:
        skipped += 1
        continue
    x = torch.tensor(rng.uniform(0, 1, g.n_voxels), dtype=torch.float64, device="cuda")
    y = torch.tensor(rng.uniform(0, 1, g.n_measurements), dtype=torch.float64, device="cuda")
    try:
        yg = forward_project_matrix_free(g, "consistent", 1, x).cpu().numpy()
        xg = back_project_matrix_free(g, "consistent", 1, y).cpu().numpy()
    except CtsmError as e:
        skipped += 1
        continue
    yr = orc.forward_project_matrix_free(g, x.cpu().numpy(), 8)
    xr = orc.back_project_matrix_free(g, y.cpu().numpy(), 8)
    e1, e2 = rel(yg, yr), rel(xg, xr)
    worst = max(worst, e1, e2)
    if max(e1, e2) > 1e-10:
        print("FAIL seed", seed, g, e1, e2)
print(f"{n_seeds} seeds, {skipped} skipped, worst relative error {worst:.3g}")
