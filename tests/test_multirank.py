"""World-size-2 gloo tests of the angle-sharded host logic (dist.py) on CPU.

The CUDA kernels are replaced by the CPU oracle (test-only injection), so the
test checks the sharding, row ownership and all-reduce plumbing: the sharded
A^T y and SIRT must equal the unsharded oracle results.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_12235_b200.geometry import TEST_GEOMETRIES


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_fns():
    import pyoracle
    orc = pyoracle.load("port_cr")

    from paper_2511_12235_b200.dist import shard_angles

    def fwd(g, x, shard, out):
        angles = shard_angles(g, shard).numpy().astype(np.int32)
        ysel = orc.forward_mf_angles(g, angles, x.numpy(), 1)
        rpa = g.rows_per_angle
        o = out.numpy()
        for k, a in enumerate(angles):
            o[a * rpa:(a + 1) * rpa] = ysel[k * rpa:(k + 1) * rpa]
        return out

    def bwd(g, y, shard, out):
        angles = shard_angles(g, shard).numpy().astype(np.int32)
        out.copy_(torch.from_numpy(orc.back_mf_angles(g, angles, y.numpy(), 1)))
        return out

    class TorchElementwise:
        """CPU stand-in for the K7/K8 C-ABI kernels (same contracts)."""

        def invert_nonzero(self, g, v):
            nz = v != 0
            v[nz] = 1.0 / v[nz]
            return v

        def residual(self, g, y, rinv, ax):
            ax.copy_(rinv * (y - ax))
            return ax

        def update(self, g, cinv, bp, x):
            x += cinv * bp
            return x

    return orc, fwd, bwd, TorchElementwise()


def _worker(rank, world, port, name, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_12235_b200 import dist as cdist
    orc, fwd, bwd, ew = _oracle_fns()
    g = TEST_GEOMETRIES[name]
    rng = np.random.default_rng(5)
    x = torch.from_numpy(rng.uniform(0, 1, g.n_voxels))
    y = torch.from_numpy(rng.uniform(0, 1, g.n_measurements))
    # forward: each rank owns disjoint rows; the sum over ranks is A x
    yl = cdist.sharded_forward(g, x, fwd=fwd)
    dist.all_reduce(yl)
    xb = cdist.sharded_back_project(g, y, bwd=bwd)
    ys = torch.from_numpy(orc.forward_project_matrix_free(g, x.numpy(), 1))
    xs = cdist.sharded_sirt(g, ys, torch.zeros(g.n_voxels, dtype=torch.float64), 3, fwd=fwd, bwd=bwd, ew=ew)
    if rank == 0:
        q.put((yl.numpy(), xb.numpy(), xs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["proj2d", "proj3d", "wide2d"])  # wide2d: orbit shards
def test_two_rank_sharding_matches_unsharded(name):
    import pyoracle
    orc = pyoracle.load("port_cr")
    g = TEST_GEOMETRIES[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    yl, xb, xs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, g.n_voxels)
    y = rng.uniform(0, 1, g.n_measurements)
    y_ref = orc.forward_project_matrix_free(g, x, 1)
    x_ref = orc.back_project_matrix_free(g, y, 1)
    s_ref = orc.sirt(g, y_ref, np.zeros(g.n_voxels), 3, 1)
    assert np.array_equal(yl, y_ref)  # disjoint rows: exact
    assert np.max(np.abs(xb - x_ref)) <= 1e-12 * max(1.0, np.max(np.abs(x_ref)))
    assert np.max(np.abs(xs - s_ref)) <= 1e-10 * max(1.0, np.max(np.abs(s_ref)))


@pytest.mark.parametrize("symmetric", [False, True])
def test_shard_rows_partition(symmetric):
    from paper_2511_12235_b200.dist import angle_shard, shard_rows
    g = TEST_GEOMETRIES["cone3d"]  # 8 angles, square grid: both shardings apply
    world = 2
    rows = torch.cat([shard_rows(g, angle_shard(g, r, world, symmetric)) for r in range(world)])
    assert torch.equal(torch.sort(rows).values, torch.arange(g.n_measurements))


@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("order", [4, 8])
def test_orbit_shards_partition_angles(world, order):
    from paper_2511_12235_b200.dist import shard_angles
    g = TEST_GEOMETRIES["wide2d"].with_(n_angles=48)
    got = torch.cat([shard_angles(g, ("orbits", r, world), order) for r in range(world)])
    assert torch.equal(torch.sort(got).values, torch.arange(g.n_angles))


def test_shard_angles_c_abi_matches_dist():
    """ctsm_shard_angles (the partition of the library's multi-GPU context)
    and dist.shard_angles (the torch.distributed drivers) agree, cover every
    angle exactly once, and are balanced to within one orbit."""
    import ctypes

    from paper_2511_12235_b200 import CONFIGS, _lib
    from paper_2511_12235_b200.dist import shard_angles

    L = _lib.lib()
    odd = CONFIGS["c1"].with_(n_angles=90, angle_end=3.0)  # no symmetry: strided shards
    for g in (CONFIGS["c1"], CONFIGS["c3"], CONFIGS["c0"], odd):
        cg = g.to_c()
        for world in (1, 2, 3, 8):
            seen = []
            sizes = []
            for rank in range(world):
                buf = (ctypes.c_int * g.n_angles)()
                n = ctypes.c_int(0)
                orb = ctypes.c_int(0)
                assert L.ctsm_shard_angles(ctypes.byref(cg), rank, world, buf, ctypes.byref(n),
                                           ctypes.byref(orb)) == 0
                got = list(buf[:n.value])
                order = 8 if (orb.value and g.angle_start == 0.0 and g.n_angles % 8 == 0) else 4
                shard = ("orbits", rank, world) if orb.value else (rank, g.n_angles, world)
                assert got == shard_angles(g, shard, order=order).tolist()
                seen += got
                sizes.append(n.value)
            assert sorted(seen) == list(range(g.n_angles))
            assert max(sizes) - min(sizes) <= 8
