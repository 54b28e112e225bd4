"""Angle-sharded multi-GPU drivers.

One process per GPU (torchrun). Rank r of N owns the strided angle shard
{r, r+N, r+2N, ...}: strided rather than contiguous because the per-angle cost
varies ~1.6x around the circle.

* A x: every rank writes its own sinogram rows -- no communication.
* A^T y: every rank back-projects its angles into a full-size partial volume;
  the partials are summed with one all-reduce (NCCL over NVLink on GPUs).
* SIRT: R = 1/(A 1) is row-local; C = 1/(A^T 1) needs one all-reduce; each
  iteration does local A x, the local residual R (y - A x), local A^T and one
  all-reduce of the back-projection, then the replicated update x += C bp.

The projector callables are injectable so the host logic can be exercised on
CPU ranks (gloo) with the oracle standing in for the kernels (tests only).
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from .geometry import ScanGeometry


def angle_shard(g: ScanGeometry, rank: int, world: int, symmetric: Optional[bool] = None):
    """Rank's angle shard. Symmetric scans are sharded by orbits
    ("orbits", rank, world): base angles rank, rank + world, ... (< n/4, or
    <= n/8 for dihedral scans) and their images under the symmetry group, so
    every rank keeps the 4x / 8x weight reuse;
    otherwise the strided shard (rank, n_angles, world)."""
    if symmetric is None:
        try:
            from .projector import quarter_symmetric
            symmetric = quarter_symmetric(g)
        except Exception:  # library unavailable (CPU-only tests)
            symmetric = False
    if symmetric:
        return ("orbits", rank, world)
    return rank, g.n_angles, world


def _symmetry_order(g: ScanGeometry) -> int:
    from .projector import symmetry_order
    return symmetry_order(g)


def shard_angles(g: ScanGeometry, shard, order: Optional[int] = None) -> torch.Tensor:
    """Angle indices of a shard, ascending. Orbit shards of a dihedral (order
    8) scan take base angles from [0, n/8] and add their reflections
    i -> n - i; quarter-turn (order 4) ones from [0, n/4)."""
    if shard[0] == "orbits":
        n = g.n_angles
        q = n // 4
        order = _symmetry_order(g) if order is None else order
        lim = n // 8 + 1 if order == 8 else q
        base = torch.arange(shard[1], lim, shard[2])
        if order == 8:
            base = torch.cat([base, (n - base) % n])
        allb = torch.cat([(base + k * q) % n for k in range(4)])
        return torch.unique(allb)  # sorted
    a0, a1, st = shard
    return torch.arange(a0, a1, st)


def shard_rows(g: ScanGeometry, shard) -> torch.Tensor:
    """Indices of the sinogram entries owned by a shard (angle-major rows)."""
    angles = shard_angles(g, shard)
    rpa = g.rows_per_angle
    return (angles[:, None] * rpa + torch.arange(rpa)[None, :]).reshape(-1)


def _default_fwd(g, x, shard, out):
    from .projector import forward_project_matrix_free
    return forward_project_matrix_free(g, "consistent", 1, x, angles=shard, out=out)


def _default_bwd(g, y, shard, out):
    from .projector import back_project_matrix_free
    return back_project_matrix_free(g, "consistent", 1, y, angles=shard, out=out)


def _world(group):
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def sharded_forward(g: ScanGeometry, x: torch.Tensor, group=None,
                    fwd: Callable = _default_fwd, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Local rows of A x (other rows zero / untouched). No communication."""
    rank, world = _world(group)
    if out is None:
        out = torch.zeros(g.n_measurements, dtype=x.dtype, device=x.device)
    return fwd(g, x, angle_shard(g, rank, world), out)


def sharded_back_project(g: ScanGeometry, y: torch.Tensor, group=None,
                         bwd: Callable = _default_bwd,
                         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """A^T y over all angles: local shard + all-reduce(sum) of the partials."""
    rank, world = _world(group)
    if out is None:
        out = torch.empty(g.n_voxels, dtype=y.dtype, device=y.device)
    part = bwd(g, y, angle_shard(g, rank, world), out)
    if world > 1:
        dist.all_reduce(part, group=group)
    return part


def _invert_nonzero(v: torch.Tensor) -> torch.Tensor:
    out = torch.zeros_like(v)
    nz = v != 0
    out[nz] = 1.0 / v[nz]
    return out


def sharded_sirt(g: ScanGeometry, y: torch.Tensor, x0: torch.Tensor, iters: int, group=None,
                 fwd: Callable = _default_fwd, bwd: Callable = _default_bwd) -> torch.Tensor:
    """SIRT x <- x + C A^T (R (y - A x)) with angle sharding (BASELINE configs[4]).

    y is the full sinogram on every rank (each rank reads only its rows); x is
    replicated and identical on all ranks after every iteration."""
    rank, world = _world(group)
    shard = angle_shard(g, rank, world)
    rows = shard_rows(g, shard).to(y.device)
    x = x0.clone()
    ax = torch.zeros(g.n_measurements, dtype=y.dtype, device=y.device)
    bp = torch.empty(g.n_voxels, dtype=y.dtype, device=y.device)
    # R = 1 / (A 1) on the local rows
    ones_v = torch.ones(g.n_voxels, dtype=y.dtype, device=y.device)
    fwd(g, ones_v, shard, ax)
    R = torch.zeros_like(ax)
    R[rows] = _invert_nonzero(ax[rows])
    # C = 1 / (A^T 1): local partial + all-reduce
    ones_m = torch.ones(g.n_measurements, dtype=y.dtype, device=y.device)
    colsum = bwd(g, ones_m, shard, bp)
    if world > 1:
        dist.all_reduce(colsum, group=group)
    C = _invert_nonzero(colsum)
    r = torch.zeros_like(ax)
    for _ in range(iters):
        fwd(g, x, shard, ax)
        r[rows] = R[rows] * (y[rows] - ax[rows])
        part = bwd(g, r, shard, bp)
        if world > 1:
            dist.all_reduce(part, group=group)
        x += C * part
    return x
