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


class DeviceElementwise:
    """K7/K8 elementwise steps of SIRT through the C-ABI kernels
    (ctsm_invert_nonzero, ctsm_sirt_residual, ctsm_sirt_update): the product
    path on CUDA tensors. R is zero on the rows a rank does not own, so the
    residual kernel runs over the full sinogram and leaves those rows zero."""

    def invert_nonzero(self, g, v: torch.Tensor) -> torch.Tensor:
        from . import _lib
        from .projector import Context, _dev_ptr, _dtype_code, _stream
        ctx = Context.get(v.device.index)
        _lib.check(_lib.lib().ctsm_invert_nonzero(ctx.handle, _dtype_code(v), v.numel(),
                                                  _dev_ptr(v), _stream(ctx.device)))
        return v

    def residual(self, g, y: torch.Tensor, rinv: torch.Tensor, ax: torch.Tensor) -> torch.Tensor:
        """ax <- rinv * (y - ax) in place; returns ax."""
        import ctypes
        from . import _lib
        from .projector import Context, _dev_ptr, _dtype_code, _stream
        ctx = Context.get(ax.device.index)
        cg = g.to_c()
        _lib.check(_lib.lib().ctsm_sirt_residual(ctx.handle, ctypes.byref(cg), _dtype_code(ax), 0,
                                                 g.n_angles, 1, _dev_ptr(y), _dev_ptr(rinv),
                                                 _dev_ptr(ax), _stream(ctx.device)))
        return ax

    def update(self, g, cinv: torch.Tensor, bp: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        """x += cinv * bp in place."""
        from . import _lib
        from .projector import Context, _dev_ptr, _dtype_code, _stream
        ctx = Context.get(x.device.index)
        _lib.check(_lib.lib().ctsm_sirt_update(ctx.handle, _dtype_code(x), x.numel(), _dev_ptr(cinv),
                                               _dev_ptr(bp), _dev_ptr(x), _stream(ctx.device)))
        return x


class SirtState:
    """Per-rank SIRT state of an angle shard: R = 1/(A 1) on the local rows (0
    elsewhere), C = 1/(A^T 1) (all-reduced), and the work arrays. step() is
    one iteration x <- x + C A^T (R (y - A x)): local A x, the fused residual
    (K8), local A^T, ONE all-reduce of the back-projection, the update."""

    def __init__(self, g: ScanGeometry, y: torch.Tensor, group=None, fwd: Callable = None,
                 bwd: Callable = None, ew=None):
        self.g, self.y, self.group = g, y, group
        self.fwd = fwd or _default_fwd
        self.bwd = bwd or _default_bwd
        self.ew = ew or DeviceElementwise()
        self.rank, self.world = _world(group)
        self.shard = angle_shard(g, self.rank, self.world)
        self.ax = torch.zeros(g.n_measurements, dtype=y.dtype, device=y.device)
        self.bp = torch.empty(g.n_voxels, dtype=y.dtype, device=y.device)
        # R = 1 / (A 1): rows of other ranks stay 0 in ax, hence in R
        ones_v = torch.ones(g.n_voxels, dtype=y.dtype, device=y.device)
        self.R = torch.zeros(g.n_measurements, dtype=y.dtype, device=y.device)
        self.fwd(g, ones_v, self.shard, self.R)
        self.ew.invert_nonzero(g, self.R)
        del ones_v
        # C = 1 / (A^T 1): local partial + all-reduce
        self.ax.fill_(1.0)
        self.C = torch.empty(g.n_voxels, dtype=y.dtype, device=y.device)
        self.bwd(g, self.ax, self.shard, self.C)
        if self.world > 1:
            dist.all_reduce(self.C, group=group)
        self.ew.invert_nonzero(g, self.C)

    def step(self, x: torch.Tensor) -> torch.Tensor:
        g = self.g
        self.fwd(g, x, self.shard, self.ax)
        self.ew.residual(g, self.y, self.R, self.ax)  # ax <- R (y - A x); 0 on foreign rows
        part = self.bwd(g, self.ax, self.shard, self.bp)
        if self.world > 1:
            dist.all_reduce(part, group=self.group)
        return self.ew.update(g, self.C, part, x)


def sharded_sirt(g: ScanGeometry, y: torch.Tensor, x0: torch.Tensor, iters: int, group=None,
                 fwd: Callable = _default_fwd, bwd: Callable = _default_bwd, ew=None) -> torch.Tensor:
    """SIRT x <- x + C A^T (R (y - A x)) with angle sharding (BASELINE configs[4]).

    y is the full sinogram on every rank (each rank reads only its rows); x is
    replicated and identical on all ranks after every iteration. ``ew`` swaps
    the elementwise kernels (tests on CPU ranks only)."""
    state = SirtState(g, y, group, fwd, bwd, ew)
    x = x0.clone()
    for _ in range(iters):
        state.step(x)
    return x
