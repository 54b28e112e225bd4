#!/usr/bin/env python3
"""Benchmark of the consistent-system-matrix hot path on B200.

Workload (default, --config c1): BASELINE.json configs[1] -- 2D fan-beam
512x512 grid, 0.5 mm pixels, s=500, sdd=1000, 1024 cells of 0.6 mm, 720
angles; one step = matrix-free A x (40-ellipse phantom) + A^T y (U[0,1)
sinogram), fp64 storage and FP64 weights. Metric: voxel-ray updates/s, where
one projection performs nnz(A) = 591,345,624 updates, so
a step is 2 * nnz updates. Multi-GPU (torchrun): angles are sharded
round-robin (rank::N); A x needs no communication, the A^T y partial volumes
are summed with an NCCL all-reduce.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libctsm_ref_glibc.so: forward_project_matrix_free and the
angle_block_entries adjoint) on all host cores over a bounded angle sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# nnz(A) per projection (voxel-ray updates); C1/C2 are
# re-verified by tests/test_gpu_parity.py::test_nnz_counts.
NNZ = {"c0": 18_291_648, "c1": 591_345_624, "c2": 4_604_879_490}
# sampled estimates for the matrix-free 3D configs; the
# GPU arm counts its updates live, the CPU reference arm uses these.
NNZ_EST = {"c3": 7.22e10, "c4": 1.158e12}
# FP64 operations per pixel/voxel-angle as executed by the reference
# (add/sub/mul/div each 1, libm calls excluded).
F_REF = {"2d": 247.0, "3d": 1513.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed steps (default: 50 for proj, 5 for sirt, 3 for csr)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c1")
    p.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    p.add_argument("--no-clocks", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--mode", default="proj", choices=["proj", "sirt", "csr"],
                   help="proj: one A x + A^T y per step; sirt: one SIRT iteration per step "
                        "(BASELINE configs[4]: y = A x_true + 1%% noise)")
    a = p.parse_args()
    if a.steps is None:
        a.steps = {"proj": 50, "sirt": 5, "csr": 3}[a.mode]
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    from paper_2511_12235_b200 import CONFIGS
    from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram

    cfg = args.config
    g = CONFIGS[cfg]
    variant = "ref_glibc" if pyoracle.available("ref_glibc") else "port_glibc"
    orc = pyoracle.load(variant)
    cores = os.cpu_count() or 1
    x = phantom_for(cfg, g)
    y = uniform_sinogram(g.n_measurements, 12346)
    # bounded sample: strided angles sized so that the whole --warmup W
    # --steps K run stays within ~2 minutes (<= 10 s of CPU work per step)
    step_budget = min(10.0, 120.0 / max(1, args.warmup + args.steps))
    probe = np.array([0, g.n_angles // 2], np.int32)
    t0 = time.perf_counter()
    orc.forward_mf_angles(g, probe, x, cores)
    orc.back_mf_angles(g, probe, y, cores)
    tau = time.perf_counter() - t0  # ~ one angle's fwd+bwd (the 2 probes run in parallel)
    # the reference parallelises over angles: use >= one angle per core
    n_sample = int(min(g.n_angles, cores * max(1, int(step_budget / max(tau, 1e-6)))))
    angles = np.linspace(0, g.n_angles, n_sample, endpoint=False).astype(np.int32)
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        orc.forward_mf_angles(g, angles, x, cores)
        orc.back_mf_angles(g, angles, y, cores)
        t = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(t)
    t_sample = float(np.mean(times))
    t_full = t_sample * g.n_angles / angles.size  # extrapolated fwd+bwd time
    value = 2.0 * NNZ.get(cfg, NNZ_EST.get(cfg, 0.0)) / t_full
    line = {
        "impl": "reference",
        "metric": "voxel-ray updates/s (A x + A^T y)",
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_full * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{cfg}: BASELINE.json configs[{cfg[1]}]", "sample_angles": int(angles.size)},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": "reference" if variant == "ref_glibc" else "port",
                         "sample": f"{angles.size} of {g.n_angles} strided angles, fwd+bwd, extrapolated x{g.n_angles / angles.size:.0f}"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def measure_dfma_peak(torch):
    """Measured FP64 FMA throughput (TFLOP/s, FMA = 2 flops) with a DFMA
    microkernel in the library's own context."""
    from paper_2511_12235_b200 import _lib
    import ctypes

    L = _lib.lib()
    f = getattr(L, "ctsm_bench_dfma", None)
    if f is None:
        return None
    f.restype = ctypes.c_double
    f.argtypes = [ctypes.c_int]
    best = 0.0
    for _ in range(3):
        best = max(best, f(torch.cuda.current_device()))
    return best


class ClockSampler:
    def __init__(self, gpu_index: int, enabled: bool):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        if not enabled:
            return
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # wait (<= 5 s) for the sampler's first line so the timed region is covered
        t_end = time.time() + 5.0
        while time.time() < t_end and os.path.getsize(self.path) == 0:
            time.sleep(0.02)
        self.t0 = self.t1 = None

    def mark(self, start: bool):
        """Wall-clock bounds of the timed region (samples outside are dropped)."""
        if start:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for line in open(self.path):
            f = [v.strip() for v in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]),
                             {n for n, v in zip(names, f[5:9]) if v.lower().startswith("active")}))
            except ValueError:
                continue
        if not rows:
            return None
        t0 = self.t0 if self.t0 is not None else rows[0][0]
        t1 = self.t1 if self.t1 is not None else rows[-1][0]
        inside = [r for r in rows if t0 - 0.025 <= r[0] <= t1 + 0.025]
        sel = inside or [min(rows, key=lambda r: abs(r[0] - 0.5 * (t0 + t1)))]
        reasons = set().union(*(r[3] for r in sel))
        return {"sm_mhz": float(np.median([r[1] for r in sel])),
                "sm_max_mhz": float(max(r[2] for r in sel)),
                "reasons": sorted(reasons), "samples": len(inside),
                "timed_region_s": round(t1 - t0, 4)}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2511_12235_b200 import CONFIGS, Context, _lib
    from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
    from paper_2511_12235_b200.projector import (back_project_matrix_free,
                                                 forward_project_matrix_free)

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    g = CONFIGS[cfg]
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    ctx = Context.get(local)
    x_h = phantom_for(cfg, g, dtype=np.float32 if not g.is_2d() else np.float64)
    y_h = uniform_sinogram(g.n_measurements, 12346)
    x = torch.from_numpy(x_h).to(tdt).to(dev)
    y = torch.from_numpy(y_h).to(tdt).to(dev)
    yout = torch.zeros(g.n_measurements, dtype=tdt, device=dev)
    xout = torch.zeros(g.n_voxels, dtype=tdt, device=dev)
    from paper_2511_12235_b200.dist import angle_shard
    shard = angle_shard(g, rank, world)  # orbit shards for quarter-turn symmetric scans
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)  # > 126 MB L2

    ev_f0, ev_f1, ev_b1, ev_r1 = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    def step():
        forward_project_matrix_free(g, "consistent", 1, x, angles=shard, out=yout)
        ev_f1.record()
        back_project_matrix_free(g, "consistent", 1, y, angles=shard, out=xout)
        ev_b1.record()
        if world > 1:
            dist.all_reduce(xout)
        ev_r1.record()

    clocks = ClockSampler(local, not args.no_clocks)
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    t_total = t_fwd = t_bwd = 0.0
    clocks.mark(True)
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ev_f0.record()
        step()
        torch.cuda.synchronize()
        t_total += ev_f0.elapsed_time(ev_r1)
        t_fwd += ev_f0.elapsed_time(ev_f1)
        t_bwd += ev_f1.elapsed_time(ev_b1)
    launches = _lib.launch_count() - launches0
    clocks.mark(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t_total / args.steps
    ms_t = torch.tensor([ms, t_fwd / args.steps, t_bwd / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms, ms_f, ms_b = [float(v) for v in ms_t.cpu()]
    # voxel-ray updates of this step, counted live by the forward kernel
    # (nonzero weights of the shard's rows); A^T y applies the same weights.
    cnt = torch.tensor([float(_lib.lib().ctsm_last_update_count(ctx.handle))], dtype=torch.float64,
                       device=dev)
    if world > 1:
        dist.all_reduce(cnt)
    nnz_live = int(cnt.item())
    updates_per_step = 2.0 * nnz_live
    value = updates_per_step / (ms * 1e-3)

    # ---- end-to-end through the reference-facing host-buffer C-ABI ----
    e2e = None
    if not args.no_e2e and world == 1 and args.dtype == "f64":
        import ctypes
        L = _lib.lib()
        xh = torch.from_numpy(x_h.astype(np.float64)).pin_memory()
        yh = torch.from_numpy(y_h).pin_memory()
        yo = torch.empty(g.n_measurements, dtype=torch.float64).pin_memory()
        xo = torch.empty(g.n_voxels, dtype=torch.float64).pin_memory()
        cg = g.to_c()
        # A x and A^T y are independent calls: a user thread each, one
        # context (scratch, status word, non-blocking stream) per thread, so
        # one call's host<->device copies overlap the other's kernels
        from concurrent.futures import ThreadPoolExecutor
        from paper_2511_12235_b200.projector import Context as _Ctx
        ctx_b = _Ctx(local)
        pool = ThreadPoolExecutor(max_workers=1)

        def bwd_call():
            _lib.check(L.ctsm_back_project_matrix_free_host(ctx_b.handle, ctypes.byref(cg),
                                                            ctypes.c_void_p(yh.data_ptr()),
                                                            ctypes.c_void_p(xo.data_ptr())))

        def e2e_step():
            fut = pool.submit(bwd_call)
            _lib.check(L.ctsm_forward_project_matrix_free_host(ctx.handle, ctypes.byref(cg),
                                                               ctypes.c_void_p(xh.data_ptr()),
                                                               ctypes.c_void_p(yo.data_ptr())))
            fut.result()
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / args.steps
        e2e = {"value": updates_per_step / te, "unit": "updates/s",
               "h2d_bytes_per_step": 8 * (g.n_voxels + g.n_measurements),
               "d2h_bytes_per_step": 8 * (g.n_measurements + g.n_voxels),
               "ms_per_step": te * 1e3,
               "calls": "ctsm_forward_project_matrix_free_host and ctsm_back_project_matrix_free_host "
                        "(pinned host buffers), issued concurrently from two host threads"}
        pool.shutdown()
        ctx_b.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak = measure_dfma_peak(torch)
    # roofline of the dominant kernel (the slower of fwd / bwd). Units are the
    # pixel/voxel-angle weight evaluations the kernel actually performs: with
    # the dihedral (quarter-turn) symmetry each evaluation serves 8 (4)
    # pixel-angles of the workload, and in 3D the z mirror doubles that, so
    # units = voxel-angles / reuse (the workload-equivalent figure is reported
    # beside it).
    from paper_2511_12235_b200.projector import symmetry_order
    reuse = symmetry_order(g)
    npix = g.n_x * g.n_y * g.n_z
    if reuse == 8:  # base angles 0..n/8 (the two self-symmetric ones reuse 4x)
        n_eval = g.n_angles // 8 + 1
    elif reuse == 4:
        n_eval = g.n_angles // 4
    else:
        n_eval = g.n_angles
    units = npix * n_eval / (world if world > 1 else 1)
    reuse = g.n_angles / n_eval
    if not g.is_2d() and symmetry_order(g) > 1 and g.n_z % 2 == 0:
        # z mirror of the symmetric 3D kernels: only the lower half of every
        # voxel column is evaluated, each weight also serves voxel n_z-1-iz
        units /= 2
        reuse *= 2
    per_unit = F_REF["2d"] if g.is_2d() else F_REF["3d"]
    dom_ms = max(ms_f, ms_b)
    achieved = units * per_unit / (dom_ms * 1e-3) / 1e12
    suffix = {8: "_d8", 4: "_sym"}.get(symmetry_order(g), "")
    kname = ("fwd2d" if ms_f >= ms_b else "bwd2d") + suffix
    if not g.is_2d():
        kname = kname.replace("2d", "3d")
    # DRAM traffic of the same kernel and workload from one committed
    # `ncu --set full` capture (profiles/ncu_kernels.json, tools/ncu_kernels.py)
    traffic, ncu_pipe = None, None
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernels.json")))
        tname = "double" if args.dtype == "f64" else "float"
        # kernel names as ncu prints them: fwd2d_d8_kernel<double>,
        # bwd2d_d8_kernel<float, 1>, fwd3d_sym_kernel<float, 8>, ...
        kbase = kname.replace("3d_d8", "3d_sym")
        prefix = f"{cfg}_{args.dtype}:{kbase}_kernel<{tname}"
        hits = [k for k in sorted(ncu) if k == prefix + ">" or k.startswith(prefix + ",")]
        if hits:
            traffic = ncu[hits[0]]["dram_bytes"]
            ncu_pipe = ncu[hits[0]].get("fp64_pipe_pct")
    except (OSError, ValueError, KeyError):
        pass
    roof = {"bound": "fp64", "kernel": kname,
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": (achieved / peak) if peak else None, "traffic": traffic,
            "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/ncu_kernels.json)",
            "ncu_fp64_pipe_active_pct": ncu_pipe,
            "peak_source": "measured DFMA microkernel (MEASURED_PEAKS.json has no FP64 entry)",
            "work_per_unit": f"{per_unit:g} FP64 flops per weight evaluation (reference op count, SURVEY.md §8(d))",
            "units_per_launch": units, "symmetry_reuse": reuse,
            "workload_equivalent_TFLOPs": achieved * reuse,
            "fwd_ms": ms_f, "bwd_ms": ms_b}
    line = {
        "metric": "voxel-ray updates/s (A x + A^T y)",
        "value": value,
        "unit": "updates/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": f"{cfg}: BASELINE.json configs[{cfg[1]}] matrix-free A x + A^T y",
                   "parallelism": f"angle-shard x{world}", "l2": "flushed (256 MB write) before each step"},
        "roofline": roof,
        "updates_per_projection": nnz_live,
        "nnz_reference": NNZ.get(cfg),  # reference nnz; the live count may differ by noise-band (<1e-13) entries
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and os.environ.get("CTSM_BENCH_NO_CPU") is None:
        line["cpu_baseline"] = cpu_baseline_quick(cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_quick(cfg):
    """The reference's CPU path on a bounded sample (rank 0, N=1)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import pyoracle
        from paper_2511_12235_b200 import CONFIGS
        from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}
    variant = "ref_glibc" if pyoracle.available("ref_glibc") else "port_glibc"
    if not pyoracle.available(variant):
        return {"error": "oracle not built"}
    orc = pyoracle.load(variant)
    g = CONFIGS[cfg]
    cores = os.cpu_count() or 1
    x = phantom_for(cfg, g)
    y = uniform_sinogram(g.n_measurements, 12346)
    # bounded sample sized to ~10 s of CPU work: time 2 angles, then scale
    probe = np.array([0, g.n_angles // 2], np.int32)
    t0 = time.perf_counter()
    orc.forward_mf_angles(g, probe, x, cores)
    orc.back_mf_angles(g, probe, y, cores)
    tau = time.perf_counter() - t0  # ~ one angle's fwd+bwd (the 2 probes run in parallel)
    # the reference parallelises over angles: use >= one angle per core
    n_sample = int(min(g.n_angles, cores * max(1, int(10.0 / max(tau, 1e-6)))))
    angles = np.linspace(0, g.n_angles, n_sample, endpoint=False).astype(np.int32)
    t0 = time.perf_counter()
    orc.forward_mf_angles(g, angles, x, cores)
    orc.back_mf_angles(g, angles, y, cores)
    t = time.perf_counter() - t0
    t_full = t * g.n_angles / angles.size
    return {"value": 2.0 * NNZ.get(cfg, NNZ_EST.get(cfg, 0.0)) / t_full, "unit": "updates/s", "cores": cores,
            "kind": "reference" if variant == "ref_glibc" else "port",
            "sample": f"fwd+bwd over {angles.size} of {g.n_angles} strided angles ({t:.1f} s), extrapolated"}


def run_sirt(args):
    """SIRT iterations (x <- x + C A^T (R (y - A x))), angle-sharded; one step =
    one iteration = one A x + one A^T r + the all-reduce. The setup (y = A
    x_true + noise, R = 1/(A 1), C = 1/(A^T 1)) runs once, untimed."""
    import torch
    import torch.distributed as dist

    from paper_2511_12235_b200 import CONFIGS, Context, _lib
    from paper_2511_12235_b200.dist import angle_shard
    from paper_2511_12235_b200.phantoms import phantom_for
    from paper_2511_12235_b200.projector import (back_project_matrix_free,
                                                 forward_project_matrix_free)

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    g = CONFIGS[cfg]
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    ctx = Context.get(local)
    shard = angle_shard(g, rank, world)
    t_setup0 = time.perf_counter()
    x_true = torch.from_numpy(phantom_for(cfg, g, dtype=np.float32)).to(tdt).to(dev)
    y = torch.zeros(g.n_measurements, dtype=tdt, device=dev)
    forward_project_matrix_free(g, "consistent", 1, x_true, angles=shard, out=y)
    ymax = y.abs().max()
    if world > 1:
        dist.all_reduce(ymax, op=dist.ReduceOp.MAX)
    # noise on every row (a rank reads only its own rows: R is zero elsewhere)
    gen = torch.Generator(device=dev).manual_seed(12347 + rank)
    y += 0.01 * ymax * torch.randn(y.numel(), dtype=tdt, device=dev, generator=gen)
    R = torch.zeros_like(y)
    forward_project_matrix_free(g, "consistent", 1, torch.ones_like(x_true), angles=shard, out=R)
    R = torch.where(R != 0, 1.0 / R, torch.zeros_like(R))  # rows of other ranks stay 0
    Cc = back_project_matrix_free(g, "consistent", 1, torch.ones_like(y), angles=shard)
    if world > 1:
        dist.all_reduce(Cc)
    Cc = torch.where(Cc != 0, 1.0 / Cc, torch.zeros_like(Cc))
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup0
    x = torch.zeros_like(x_true)
    ax = torch.zeros_like(y)
    r = torch.zeros_like(y)
    bp = torch.empty_like(x)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def iteration():
        forward_project_matrix_free(g, "consistent", 1, x, angles=shard, out=ax)
        torch.mul(R, y - ax, out=r)  # R = 0 on rows of other ranks
        back_project_matrix_free(g, "consistent", 1, r, angles=shard, out=bp)
        if world > 1:
            dist.all_reduce(bp)
        x.add_(Cc * bp)

    clocks = ClockSampler(local, not args.no_clocks)
    for _ in range(args.warmup):
        iteration()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    ms_total = 0.0
    clocks.mark(True)
    for _ in range(args.steps):
        torch.cuda.synchronize()
        ev0.record()
        iteration()
        ev1.record()
        torch.cuda.synchronize()
        ms_total += ev0.elapsed_time(ev1)
    launches = _lib.launch_count() - launches0
    clocks.mark(False)
    clk = clocks.stop()
    ms = ms_total / args.steps
    cnt = torch.tensor([float(_lib.lib().ctsm_last_update_count(ctx.handle)), ms],
                       dtype=torch.float64, device=dev)
    if world > 1:
        upd = cnt[0:1].clone()
        dist.all_reduce(upd)
        msx = cnt[1:2].clone()
        dist.all_reduce(msx, op=dist.ReduceOp.MAX)
        cnt = torch.cat([upd, msx])
    nnz_live, ms = int(cnt[0].item()), float(cnt[1].item())
    if rank == 0:
        # residual over the rows rank 0 solves for (R != 0; empty rows excluded)
        resid = float((torch.where(R != 0, y - ax, torch.zeros_like(ax)) ** 2).sum().sqrt())
        line = {
            "metric": "voxel-ray updates/s (SIRT iterations)",
            "value": 2.0 * nnz_live / (ms * 1e-3),
            "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{cfg}: BASELINE.json configs[{cfg[1]}] SIRT (one iteration per step)",
                       "parallelism": f"angle-shard x{world}", "setup_s": t_setup,
                       "iterations_total": args.warmup + args.steps},
            "updates_per_projection": nnz_live,
            "rank0_residual_norm": resid,
            "gpu_launches": int(launches), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_csr(args):
    """K1/K2 consistent CSR assembly (bit-exact path) + K3 SpMV on one GPU.
    One step = build_system_matrix (count, scan, fill, per-row sort) of the
    whole config; metric SM weights/s = nnz / build time. K3 A x on the built
    matrix is timed separately (HBM roofline: 12 B/nnz + 16 B/row)."""
    import torch

    from paper_2511_12235_b200 import CONFIGS, _lib
    from paper_2511_12235_b200.phantoms import phantom_for
    from paper_2511_12235_b200.projector import build_system_matrix, forward_project

    cfg = args.config
    g = CONFIGS[cfg]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    budget = 1 << 40
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w = None
    for _ in range(args.warmup):
        w = build_system_matrix(g, memory_budget_bytes=budget)
        del w
        torch.cuda.synchronize()
    clocks = ClockSampler(0, not args.no_clocks)
    launches0 = _lib.launch_count()
    ms = 0.0
    clocks.mark(True)
    for _ in range(args.steps):
        w = None
        torch.cuda.synchronize()
        ev0.record()
        w = build_system_matrix(g, memory_budget_bytes=budget)
        ev1.record()
        torch.cuda.synchronize()
        ms += ev0.elapsed_time(ev1)
    launches = _lib.launch_count() - launches0
    clocks.mark(False)
    ms /= args.steps
    nnz = w.nnz()
    x = torch.from_numpy(phantom_for(cfg, g, dtype=np.float64 if g.is_2d() else np.float32)).double().to(dev)
    for _ in range(3):
        forward_project(w, x)
    torch.cuda.synchronize()
    ms_spmv = 0.0
    for _ in range(5):
        ev0.record()
        forward_project(w, x)
        ev1.record()
        torch.cuda.synchronize()
        ms_spmv += ev0.elapsed_time(ev1) / 5
    # K4 (reference back_project, projector.cpp:219-233) on a U[0, 1) sinogram
    from paper_2511_12235_b200.projector import back_project
    from paper_2511_12235_b200.phantoms import uniform_sinogram
    yb = torch.from_numpy(uniform_sinogram(w.n_rows, 12346)).to(dev)
    for _ in range(3):
        back_project(w, yb)
    torch.cuda.synchronize()
    ms_spmvt = 0.0
    for _ in range(5):
        ev0.record()
        back_project(w, yb)
        ev1.record()
        torch.cuda.synchronize()
        ms_spmvt += ev0.elapsed_time(ev1) / 5
    clk = clocks.stop()
    bytes_spmv = 12.0 * nnz + 16.0 * w.n_rows + 8.0 * w.n_cols
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    gbs = bytes_spmv / (ms_spmv * 1e-3) / 1e9
    line = {
        "metric": "SM weights/s (consistent CSR assembly)", "value": nnz / (ms * 1e-3),
        "unit": "weights/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg}: BASELINE.json configs[{cfg[1]}] build_system_matrix"},
        "nnz": nnz, "nnz_reference": NNZ.get(cfg),
        "spmv": {"ms": ms_spmv, "GB/s": gbs, "algorithmic_bytes": bytes_spmv,
                 "hbm_peak_gbs": peaks.get("hbm_gbs"), "frac": gbs / peaks.get("hbm_gbs", 6650.0)},
        "spmv_t": {"ms": ms_spmvt, "GB/s": bytes_spmv / (ms_spmvt * 1e-3) / 1e9,
                   "algorithmic_bytes": bytes_spmv,
                   "frac": bytes_spmv / (ms_spmvt * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                   "note": "back_project: int64 fixed-point scatter (deterministic) with the matrix's "
                           "column-sum bound, computed once per matrix (cached, outside the timed calls)"},
        "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "sirt":
        run_sirt(args)
    elif args.mode == "csr":
        run_csr(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
