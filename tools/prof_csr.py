"""Profiling driver for the CSR emission (K1/K2) and appliers (K3/K4): the C2
matrix restricted to a strided block of angles (default 8), built twice
(warm-up + profiled), then A x and A^T y once each."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_12235_b200 import CONFIGS, back_project, build_system_matrix, forward_project  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_ang = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = CONFIGS[cfg]
for _ in range(2):
    w = build_system_matrix(g, memory_budget_bytes=1 << 40, angle_range=(0, n_ang))
    torch.cuda.synchronize()
x = torch.rand(g.n_voxels, dtype=torch.float64, device="cuda")
y = torch.rand(w.n_rows, dtype=torch.float64, device="cuda")
forward_project(w, x)
back_project(w, y)
torch.cuda.synchronize()
print(cfg, n_ang, "angles: nnz", w.nnz())
