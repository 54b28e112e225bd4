"""Profiling driver for the 3D matrix-free kernels: C3 geometry, a strided
shard of angles (default 16), fwd + bwd once each after a warm-up."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_12235_b200 import CONFIGS  # noqa: E402
from paper_2511_12235_b200.phantoms import phantom_for  # noqa: E402
from paper_2511_12235_b200.projector import (back_project_matrix_free,  # noqa: E402
                                             forward_project_matrix_free)

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n_ang = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = CONFIGS[cfg]
x = torch.from_numpy(phantom_for(cfg, g, dtype=np.float32)).cuda()
y = torch.rand(g.n_measurements, dtype=torch.float32, device="cuda")
from paper_2511_12235_b200.dist import shard_angles  # noqa: E402
from paper_2511_12235_b200.projector import symmetry_order  # noqa: E402

order = symmetry_order(g)
if order > 1:
    n_base = g.n_angles // 8 + 1 if order == 8 else g.n_angles // 4
    base_step = max(1, n_base // max(1, n_ang // order))
    shard = ("orbits", 0, base_step)  # base angles + their images under the group
    n_sel = len(shard_angles(g, shard, order))
else:
    step = max(1, g.n_angles // n_ang)
    shard = (0, g.n_angles, step)
    n_sel = len(range(*shard))
yo = torch.zeros_like(y)
xo = torch.zeros_like(x)
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    forward_project_matrix_free(g, "consistent", 1, x, angles=shard, out=yo)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    back_project_matrix_free(g, "consistent", 1, y, angles=shard, out=xo)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{cfg} {n_sel} angles ({shard[0] if shard[0] == 'orbits' else 'strided'}): "
          f"fwd {1e3*(t1-t0):.1f} ms  bwd {1e3*(t2-t1):.1f} ms  "
          f"-> per full projection fwd {1e3*(t1-t0)*g.n_angles/n_sel:.0f} ms, "
          f"bwd {1e3*(t2-t1)*g.n_angles/n_sel:.0f} ms")
