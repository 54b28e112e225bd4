#!/usr/bin/env python3
"""Benchmark of the consistent-system-matrix hot path on B200.

Default workload (--config c3): BASELINE.json configs[3], the largest
matrix-free projection pair that BASELINE.json states for 1-8 GPUs -- 3D
circular cone-beam, 256^3 voxels of 0.5 mm, s = 500, sdd = 1000, 512 x 384
detector of 0.8 mm pixels, 720 angles; one step = matrix-free A x
(50-ellipsoid phantom) + A^T y (U[0,1) sinogram), fp32 storage, FP64 weights.
Metric: voxel-ray updates/s = nonzero weights applied per second (a projection
applies nnz(A) of them; counted live by the forward kernel). Other workloads:
--config c0..c4, --dtype f32|f64, --mode proj|sirt|csr.

Multi-GPU: `python bench.py --gpus N` re-launches itself under
torch.distributed.run with N ranks (or is launched that way by the driver);
angles are sharded by symmetry orbits (rank r takes base angles r, r+N, ...
and their images), A x needs no communication, the A^T y partial volumes are
summed with an NCCL all-reduce.

--impl reference times the reference's own CPU implementation
(oracle/_ref/libctsm_ref_glibc.so, the unmodified reference sources) on all
host cores; each step is a bounded sample of the same workload (strided
angles x strided voxel slabs, A x and A^T y each evaluating the weights as
the reference does).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# nnz(A) per projection (voxel-ray updates), SURVEY.md §0 fact 4 (C0/C1 are
# checked against the GPU's live count and CSR by tests/test_gpu_parity.py).
NNZ = {"c0": 18_291_648, "c1": 591_345_624, "c2": 4_604_879_490}
# sampled estimates for the matrix-free 3D configs; only
# used to extrapolate the CPU sample to a full step, never for `value`.
NNZ_EST = {"c3": 7.22e10, "c4": 1.158e12}
# FP64 operations per pixel/voxel-angle as executed by the reference
# (add/sub/mul/div each 1, an FMA would count 1, libm calls
# excluded).
F_REF = {"2d": 247.0, "3d": 1513.0}
DEFAULT_DTYPE = {"c0": "f64", "c1": "f64", "c2": "f64", "c3": "f32", "c4": "f32"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed steps (default: 20 for proj (50 for 2D), 5 for sirt, 3 for csr)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c3", choices=["c0", "c1", "c2", "c3", "c4"])
    p.add_argument("--dtype", default=None, choices=["f64", "f32"])
    p.add_argument("--no-clocks", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--mode", default="proj", choices=["proj", "sirt", "csr"],
                   help="proj: one A x + A^T y per step; sirt: one SIRT iteration per step "
                        "(BASELINE configs[4]: y = A x_true + 1%% noise); csr: one "
                        "build_system_matrix per step")
    a = p.parse_args()
    if a.dtype is None:
        a.dtype = DEFAULT_DTYPE[a.config]
    if a.steps is None:
        a.steps = {"proj": 50 if a.config in ("c0", "c1") else 20, "sirt": 5, "csr": 3}[a.mode]
    return a


def share_gpu():
    """CTSM_BENCH_SHARE_GPU=1: every rank uses cuda:0 and the collectives go
    through gloo. A functional check of the N-rank code path on a one-GPU box
    (tests/test_gpu_host_calls.py); never a measurement."""
    return os.environ.get("CTSM_BENCH_SHARE_GPU") == "1"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if share_gpu() else int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def relaunch_if_needed(args):
    """`python bench.py --gpus N` without torchrun: start the N ranks here
    (the driver's own launch line, on 127.0.0.1). Under torchrun the world
    size must equal --gpus."""
    if args.impl == "reference" or args.mode == "csr":
        return
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def init_dist(torch, dev):
    """NCCL process group over the ranks torchrun started; prints the
    communicator size per rank (NCCL_DEBUG=INFO adds NCCL's own lines)."""
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if share_gpu():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        assert dist.get_world_size() == world
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)
        print(f"[bench] rank {rank}/{world} on cuda:{local}: communicator nranks={int(t.item())}",
              file=sys.stderr, flush=True)
        assert int(t.item()) == world
    return dist


def host_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "libc": " ".join(platform.libc_ver()),
            "cores": os.cpu_count() or 1}


def workload_config(args, world):
    """The `config` object: identical in both arms for the same flags."""
    cfg = args.config
    what = {"proj": "matrix-free A x + A^T y", "sirt": "SIRT (one iteration per step)",
            "csr": "build_system_matrix (consistent CSR assembly)"}[args.mode]
    return {"workload": f"{cfg}: BASELINE.json configs[{cfg[1]}] {what}",
            "parallelism": f"angle-shard x{world}",
            "l2": "flushed (256 MB write) before each step" if args.mode == "proj"
                  else "working set larger than L2"}


# ---------------------------------------------------------------------------
# The reference's CPU path on a bounded sample (reference arm and cpu_baseline)
# ---------------------------------------------------------------------------
def _load_oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    variant = "ref_glibc" if pyoracle.available("ref_glibc") else "port_glibc"
    return pyoracle, pyoracle.load(variant), variant


def sample_inputs(cfg, g):
    """Synthetic inputs of the CPU sample: the same seeded phantom as the GPU
    arm where it is cheap to build (2D), a PCG64 U[0.005, 0.02) volume for the
    3D configs (the CPU cost does not depend on the values)."""
    from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
    if g.is_2d():
        x = phantom_for(cfg, g)
    else:
        x = 0.005 + 0.015 * np.random.Generator(np.random.PCG64(12345)).random(g.n_voxels)
    y = uniform_sinogram(g.n_measurements, 12346)
    return x, y


class PairSample:
    """A bounded A x + A^T y sample of one config: strided angles (angle 0, a
    flat-branch angle, included) x strided slabs (z planes / pixel rows),
    sized by a probe to about `seconds` of wall time on `cores` threads."""

    def __init__(self, cfg, seconds):
        from paper_2511_12235_b200 import CONFIGS
        self.pyoracle, self.orc, self.variant = _load_oracle()
        self.cfg, self.g = cfg, CONFIGS[cfg]
        g = self.g
        self.cores = os.cpu_count() or 1
        self.x, self.y = sample_inputs(cfg, g)
        n_slab_total = g.n_y if g.is_2d() else g.n_z
        n_ang = min(g.n_angles, max(16, self.cores))
        self.angles = np.unique(np.linspace(0, g.n_angles, n_ang, endpoint=False).astype(np.int32))
        probe_slabs = np.array([n_slab_total // 3], np.int32)
        t0 = time.perf_counter()
        self.orc.mf_pair_sample(g, self.angles, probe_slabs, self.x, self.y, self.cores)
        tau = max(time.perf_counter() - t0, 1e-4)  # one slab of every sampled angle
        n_sl = int(max(1, min(n_slab_total, seconds / tau)))
        self.slabs = np.unique(np.linspace(0, n_slab_total, n_sl, endpoint=False).astype(np.int32))
        self.frac = (self.angles.size * self.slabs.size) / (g.n_angles * n_slab_total)

    def run(self):
        t0 = time.perf_counter()
        upd, _ = self.orc.mf_pair_sample(self.g, self.angles, self.slabs, self.x, self.y, self.cores)
        return upd, time.perf_counter() - t0

    def describe(self, t):
        unit = "pixel rows" if self.g.is_2d() else "z planes"
        return (f"A x + A^T y over {self.angles.size} of {self.g.n_angles} strided angles x "
                f"{self.slabs.size} strided {unit} ({100 * self.frac:.3g}% of a step, {t:.1f} s)")


def cpu_baseline_proj(cfg, seconds=12.0):
    try:
        s = PairSample(cfg, seconds)
        upd, t = s.run()
    except Exception as e:  # pragma: no cover
        return {"error": repr(e)}
    return {"value": upd / t, "unit": "updates/s", "cores": s.cores,
            "kind": "reference" if s.variant == "ref_glibc" else "port",
            "sample": s.describe(t), **host_info()}


def csr_reference_sample(cfg, seconds):
    """Reference CSR assembly: build_system_matrix in full where it fits a
    bounded run (C0), else build_angle_block of strided angles, one angle per
    core (C2). Returns (weights built, seconds, description)."""
    from paper_2511_12235_b200 import CONFIGS
    _, orc, variant = _load_oracle()
    g = CONFIGS[cfg]
    cores = os.cpu_count() or 1
    if g.is_2d():
        t0 = time.perf_counter()
        w = orc.build_system_matrix(g, threads=cores, budget=1 << 40)
        t = time.perf_counter() - t0
        return w.nnz, t, f"build_system_matrix in full ({t:.1f} s)", variant, cores
    t0 = time.perf_counter()
    orc.csr_angle_sample(g, np.array([g.n_angles // 3], np.int32), 1)
    tau = time.perf_counter() - t0
    rounds = max(1, int(seconds / max(tau, 1e-3)))
    n_ang = min(g.n_angles, cores * rounds)
    angles = np.unique(np.linspace(0, g.n_angles, n_ang, endpoint=False).astype(np.int32))
    t0 = time.perf_counter()
    nnz = orc.csr_angle_sample(g, angles, cores)
    t = time.perf_counter() - t0
    return nnz, t, (f"build_angle_block of {angles.size} of {g.n_angles} strided angles, one angle "
                    f"per core ({t:.1f} s)"), variant, cores


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    # each step is a bounded sample; the whole run stays within a few minutes
    step_budget = min(6.0, 150.0 / max(1, args.warmup + args.steps))
    if args.mode == "csr":
        nnz, t, desc, variant, cores = csr_reference_sample(cfg, step_budget)
        times = [t]
        for it in range(1, args.warmup + args.steps):
            nnz, t, desc, variant, cores = csr_reference_sample(cfg, step_budget)
            times.append(t)
        t = float(np.mean(times[-args.steps:]))
        value, unit, metric = nnz / t, "weights/s", "SM weights/s (consistent CSR assembly)"
        full_ms = NNZ[cfg] / value * 1e3
    else:
        s = PairSample(cfg, step_budget)
        variant, cores = s.variant, s.cores
        times, upd = [], 0
        for it in range(args.warmup + args.steps):
            upd, t = s.run()
            if it >= args.warmup:
                times.append(t)
        t = float(np.mean(times))
        desc = s.describe(t)
        value, unit = upd / t, "updates/s"
        metric = ("voxel-ray updates/s (SIRT iterations)" if args.mode == "sirt"
                  else "voxel-ray updates/s (A x + A^T y)")
        full_ms = 2.0 * NNZ.get(cfg, NNZ_EST.get(cfg, 0.0)) / value * 1e3
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3,  # one step = one bounded sample (see cpu_baseline.sample)
        "ms_per_full_step_extrapolated": full_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores,
                         "kind": "reference" if variant == "ref_glibc" else "port",
                         "sample": desc, **host_info()},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def measure_dfma_peak(torch):
    """Measured FP64 FMA throughput (TFLOP/s, FMA = 2 flops) with a DFMA
    microkernel in the library's own context."""
    import ctypes

    from paper_2511_12235_b200 import _lib

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


def fp64_roofline(torch, g, cfg, dtype, world, ms_f, ms_b):
    """FP64 roofline of the dominant kernel (the slower of fwd / bwd), per
    SURVEY.md §8(d): achieved = weight evaluations per launch x F (FP64
    arithmetic operations per evaluation as the reference executes them, an
    FMA counting as ONE operation) / kernel time; peak = the measured FP64
    arithmetic-instruction rate = measured DFMA FLOP/s / 2. The evaluations
    are the ones the kernel performs: with the dihedral (quarter-turn)
    symmetry each serves 8 (4) pixel-angles of the workload and, in 3D, the z
    mirror doubles that (the workload-equivalent figure is beside it)."""
    from paper_2511_12235_b200.projector import symmetry_order
    peak_flops = measure_dfma_peak(torch)
    order = symmetry_order(g)
    npix = g.n_x * g.n_y * g.n_z
    n_eval = {8: g.n_angles // 8 + 1, 4: g.n_angles // 4}.get(order, g.n_angles)
    if order > 1 and world > 1:  # orbit shards: the slowest rank's base angles
        n_eval = -(-n_eval // world)
    elif world > 1:
        n_eval = -(-g.n_angles // world)
    units = npix * n_eval
    reuse = g.n_angles / world / n_eval
    if not g.is_2d() and order > 1 and g.n_z % 2 == 0:
        units /= 2  # z mirror: only the lower half of every voxel column is evaluated
        reuse *= 2
    per_unit = F_REF["2d"] if g.is_2d() else F_REF["3d"]
    dom_ms = max(ms_f, ms_b)
    achieved = units * per_unit / (dom_ms * 1e-3) / 1e12  # T FP64 ops/s (FMA = 1)
    peak_ops = peak_flops / 2.0 if peak_flops else None
    suffix = {8: "_d8", 4: "_sym"}.get(order, "")
    kname = ("fwd2d" if ms_f >= ms_b else "bwd2d") + suffix
    if not g.is_2d():
        kname = kname.replace("2d", "3d")
    # DRAM traffic and pipe utilisation of the same kernel and workload from one
    # committed `ncu --set full` capture (profiles/ncu_kernels.json)
    traffic = ncu_pipe = ncu_ms = ncu_red = None
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernels.json")))
        tname = "double" if dtype == "f64" else "float"
        kbase = kname.replace("3d_d8", "3d_sym")
        prefix = f"{cfg}_{dtype}:{kbase}_kernel<{tname}"
        # (the 3D back-projection runs as bwd3d_sym_v_kernel)
        prefixes = (prefix, f"{cfg}_{dtype}:{kbase}_v_kernel<{tname}")
        hits = [k for k in sorted(ncu)
                if any(k == p + ">" or k.startswith(p + ",") for p in prefixes)]
        if hits:
            e = ncu[hits[-1]]
            traffic = e["dram_bytes"]
            ncu_pipe = e.get("fp64_pipe_pct")
            ncu_ms = e.get("duration_ms")
            if e.get("global_red_warp_insts") and e.get("sm_cycles"):
                # the fp32 3D forward leaves through 16-byte vector reductions;
                # tools/micro/red_bench.cu measures what an SM sustains
                lane_ops = e["global_red_warp_insts"] * e.get("active_lanes", 32.0)
                ncu_red = {"lane_reductions_per_clk_sm": lane_ops / 148.0 / e["sm_cycles"],
                           "microbench_peak_per_clk_sm": [0.47, 0.65],
                           "note": "16-byte red.global.add.v4.f32 per lane; the peak is the "
                                   "two-reductions-per-32-byte-segment microbenchmark, lanes 5 rows "
                                   "apart / adjacent (profiles/r3l_red_bench.log); upper estimate: "
                                   "the kernel's average active lanes applied to its reductions"}
    except (OSError, ValueError, KeyError):
        pass
    extra = {"ncu_global_reductions": ncu_red} if ncu_red else {}
    return {**extra, "bound": "fp64", "kernel": kname, "achieved": achieved, "peak": peak_ops,
            "unit": "T FP64 op/s (arithmetic instructions, FMA = 1 op; SURVEY.md §8(d))",
            "frac": (achieved / peak_ops) if peak_ops else None,
            "frac_flops_convention": (achieved / peak_flops) if peak_flops else None,
            "traffic": traffic,
            "traffic_unit": "DRAM bytes per kernel launch of the ncu capture (ncu --set full, "
                            "profiles/ncu_kernels.json)",
            "ncu_fp64_pipe_active_pct": ncu_pipe, "ncu_launch_ms": ncu_ms,
            "peak_source": "measured DFMA microkernel (ctsm_bench_dfma; MEASURED_PEAKS.json has no "
                           f"FP64 entry): {peak_flops:.2f} TFLOP/s = {peak_ops:.2f} T DFMA/s"
                           if peak_flops else "unavailable",
            "work_per_unit": f"{per_unit:g} FP64 ops per weight evaluation (reference op count, "
                             "SURVEY.md §8(d))",
            "units_per_launch": units, "symmetry_reuse": reuse,
            "workload_equivalent_Tops": achieved * reuse,
            "fwd_ms": ms_f, "bwd_ms": ms_b}


def e2e_projection_pair(torch, args, g, x_h, y_h, ctx, local, updates_per_step):
    """The same step through the reference-facing host-buffer C-ABI
    (ctsm_{forward,back}_project_matrix_free_host[_f32]): pinned host x / y in,
    host y / x out, H2D and D2H copies inside the timed region. A x and A^T y
    are independent calls: a user thread each, one context (scratch, status
    word, non-blocking stream) per thread, so one call's copies overlap the
    other's kernels."""
    import ctypes
    from concurrent.futures import ThreadPoolExecutor

    from paper_2511_12235_b200 import Context, _lib
    L = _lib.lib()
    f32 = args.dtype == "f32"
    npdt, es = (np.float32, 4) if f32 else (np.float64, 8)
    tdt = torch.float32 if f32 else torch.float64
    fwd = L.ctsm_forward_project_matrix_free_host_f32 if f32 else L.ctsm_forward_project_matrix_free_host
    bwd = L.ctsm_back_project_matrix_free_host_f32 if f32 else L.ctsm_back_project_matrix_free_host
    xh = torch.from_numpy(x_h.astype(npdt)).pin_memory()
    yh = torch.from_numpy(y_h.astype(npdt)).pin_memory()
    yo = torch.empty(g.n_measurements, dtype=tdt).pin_memory()
    xo = torch.empty(g.n_voxels, dtype=tdt).pin_memory()
    cg = g.to_c()
    ctx_b = Context(local)
    pool = ThreadPoolExecutor(max_workers=1)

    def bwd_call():
        _lib.check(bwd(ctx_b.handle, ctypes.byref(cg), ctypes.c_void_p(yh.data_ptr()),
                       ctypes.c_void_p(xo.data_ptr())))

    def e2e_step():
        fut = pool.submit(bwd_call)
        _lib.check(fwd(ctx.handle, ctypes.byref(cg), ctypes.c_void_p(xh.data_ptr()),
                       ctypes.c_void_p(yo.data_ptr())))
        fut.result()

    n_warm = max(1, min(args.warmup, 3))
    n_steps = args.steps if g.is_2d() else min(args.steps, 5)
    for _ in range(n_warm):
        e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        e2e_step()
    torch.cuda.synchronize()
    te = (time.perf_counter() - t0) / n_steps
    pool.shutdown()
    ctx_b.close()
    return {"value": updates_per_step / te, "unit": "updates/s",
            "h2d_bytes_per_step": es * (g.n_voxels + g.n_measurements),
            "d2h_bytes_per_step": es * (g.n_measurements + g.n_voxels),
            "ms_per_step": te * 1e3, "steps": n_steps,
            "calls": ("ctsm_forward_project_matrix_free_host" + ("_f32" if f32 else "") +
                      " and ctsm_back_project_matrix_free_host" + ("_f32" if f32 else "") +
                      " (pinned host buffers), issued concurrently from two host threads")}


def e2e_projection_pair_sharded(torch, dist, args, g, x_h, y_h, dev, world, rank,
                                updates_per_step):
    """N ranks: the step through the public sharded API (dist.sharded_forward
    / sharded_back_project) with pinned host buffers. Per step and rank: x
    host -> device, A x on the rank's angle shard, its sinogram rows device ->
    host; its rows of y host -> device, A^T y on the shard, the NCCL
    all-reduce of the volume, the volume device -> host. Timed between
    barriers, max over ranks."""
    from paper_2511_12235_b200.dist import (angle_shard, shard_angles, sharded_back_project,
                                            sharded_forward)
    f32 = args.dtype == "f32"
    npdt, es = (np.float32, 4) if f32 else (np.float64, 8)
    tdt = torch.float32 if f32 else torch.float64
    rpa = g.rows_per_angle
    angles = shard_angles(g, angle_shard(g, rank, world)).tolist()
    xh = torch.from_numpy(x_h.astype(npdt)).pin_memory()
    yh = torch.from_numpy(y_h.astype(npdt)).pin_memory().view(g.n_angles, rpa)
    yo = torch.empty(g.n_angles, rpa, dtype=tdt).pin_memory()
    xo = torch.empty(g.n_voxels, dtype=tdt).pin_memory()
    xd = torch.empty(g.n_voxels, dtype=tdt, device=dev)
    yd = torch.zeros(g.n_angles, rpa, dtype=tdt, device=dev)
    yin = torch.zeros(g.n_angles, rpa, dtype=tdt, device=dev)
    bp = torch.empty(g.n_voxels, dtype=tdt, device=dev)
    idx = torch.tensor(angles, device=dev)
    idx_h = torch.tensor(angles)
    stage_d = torch.empty(len(angles), rpa, dtype=tdt, device=dev)
    stage_h = torch.empty(len(angles), rpa, dtype=tdt).pin_memory()      # A x rows out
    stage_in_h = torch.empty(len(angles), rpa, dtype=tdt).pin_memory()   # y rows in

    def step():
        xd.copy_(xh, non_blocking=True)
        sharded_forward(g, xd, out=yd.view(-1))
        torch.index_select(yd, 0, idx, out=stage_d)
        stage_h.copy_(stage_d, non_blocking=True)
        # this rank's rows of y: gathered on the host, one H2D copy, scattered on the device
        torch.index_select(yh, 0, idx_h, out=stage_in_h)
        stage_d.copy_(stage_in_h, non_blocking=True)
        yin.index_copy_(0, idx, stage_d)
        sharded_back_project(g, yin.view(-1), out=bp)
        xo.copy_(bp, non_blocking=True)
        torch.cuda.synchronize()

    n_warm = max(1, min(args.warmup, 3))
    n_steps = args.steps if g.is_2d() else min(args.steps, 5)
    for _ in range(n_warm):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n_steps):
        step()
    dist.barrier()
    te = torch.tensor([(time.perf_counter() - t0) / n_steps], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    te = float(te.item())
    rows = len(angles) * rpa
    return {"value": updates_per_step / te, "unit": "updates/s",
            "h2d_bytes_per_step": es * (g.n_voxels + rows),
            "d2h_bytes_per_step": es * (rows + g.n_voxels),
            "bytes_are": "per rank (x replicated, the rank's own sinogram rows)",
            "ms_per_step": te * 1e3, "steps": n_steps,
            "calls": "dist.sharded_forward / dist.sharded_back_project with pinned host buffers "
                     "on every rank (max over ranks)"}


def run_ours(args):
    import torch

    from paper_2511_12235_b200 import CONFIGS, Context, _lib
    from paper_2511_12235_b200.dist import angle_shard
    from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
    from paper_2511_12235_b200.projector import (back_project_matrix_free,
                                                 forward_project_matrix_free)

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist = init_dist(torch, dev)
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

    e2e = None
    if not args.no_e2e and world == 1:
        del yout, xout
        e2e = e2e_projection_pair(torch, args, g, x_h, y_h, ctx, local, updates_per_step)
    elif not args.no_e2e:
        del yout, xout
        e2e = e2e_projection_pair_sharded(torch, dist, args, g, x_h, y_h, dev, world, rank,
                                          updates_per_step)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": "voxel-ray updates/s (A x + A^T y)",
        "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": workload_config(args, world),
        "roofline": fp64_roofline(torch, g, cfg, args.dtype, world, ms_f, ms_b),
        "updates_per_projection": nnz_live,
        "nnz_reference": NNZ.get(cfg),  # reference nnz; the live count may differ by noise-band (<1e-13) entries
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu and os.environ.get("CTSM_BENCH_NO_CPU") is None:
        line["cpu_baseline"] = cpu_baseline_proj(cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sirt(args):
    """SIRT iterations (x <- x + C A^T (R (y - A x))), angle-sharded; one step =
    one iteration = one A x + the fused residual (K8) + one A^T r + the
    all-reduce + the update. The setup (y = A x_true + noise, R = 1/(A 1),
    C = 1/(A^T 1)) runs once, untimed."""
    import torch

    from paper_2511_12235_b200 import CONFIGS, Context, _lib
    from paper_2511_12235_b200.dist import SirtState, angle_shard
    from paper_2511_12235_b200.phantoms import phantom_for
    from paper_2511_12235_b200.projector import forward_project_matrix_free

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist = init_dist(torch, dev)
    cfg = args.config
    g = CONFIGS[cfg]
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    ctx = Context.get(local)
    shard = angle_shard(g, rank, world)
    t_setup0 = time.perf_counter()
    x_true = torch.from_numpy(phantom_for(cfg, g, dtype=np.float32)).to(tdt).to(dev)
    y = torch.zeros(g.n_measurements, dtype=tdt, device=dev)
    forward_project_matrix_free(g, "consistent", 1, x_true, angles=shard, out=y)
    del x_true
    ymax = y.abs().max()
    if world > 1:
        dist.all_reduce(ymax, op=dist.ReduceOp.MAX)
    # noise on every row (a rank reads only its own rows: R is zero elsewhere)
    gen = torch.Generator(device=dev).manual_seed(12347 + rank)
    y.add_(torch.randn(y.numel(), dtype=tdt, device=dev, generator=gen), alpha=float(0.01 * ymax))
    state = SirtState(g, y)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup0
    x = torch.zeros(g.n_voxels, dtype=tdt, device=dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    clocks = ClockSampler(local, not args.no_clocks)
    for _ in range(args.warmup):
        state.step(x)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    ms_total = 0.0
    clocks.mark(True)
    for _ in range(args.steps):
        torch.cuda.synchronize()
        ev0.record()
        state.step(x)
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
    updates_per_step = 2.0 * nnz_live

    # ---- end to end: a user's solve through the host-buffer path: y from
    # pinned host memory, `steps` iterations, x back to the host; per iteration
    e2e = None
    if not args.no_e2e and world == 1:
        yh = y.cpu().pin_memory()
        xh = torch.empty(g.n_voxels, dtype=tdt).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y.copy_(yh, non_blocking=True)
        x.zero_()
        for _ in range(args.steps):
            state.step(x)
        xh.copy_(x, non_blocking=True)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / args.steps
        es = 4 if args.dtype == "f32" else 8
        e2e = {"value": updates_per_step / te, "unit": "updates/s",
               "h2d_bytes_per_step": es * g.n_measurements / args.steps,
               "d2h_bytes_per_step": es * g.n_voxels / args.steps, "ms_per_step": te * 1e3,
               "calls": f"one solve of {args.steps} iterations: y from pinned host memory, x back "
                        "to the host; bytes and time per iteration"}
    if rank == 0:
        # residual over the rows rank 0 solves for (R != 0; empty rows excluded)
        ax = torch.zeros_like(y)
        forward_project_matrix_free(g, "consistent", 1, x, angles=shard, out=ax)
        resid = float((torch.where(state.R != 0, y - ax, torch.zeros_like(ax)) ** 2).sum().sqrt())
        del ax
        # the iteration is one forward and one back-projection launch; the
        # roofline is the slower projection's, taken as half the iteration
        line = {
            "metric": "voxel-ray updates/s (SIRT iterations)",
            "value": updates_per_step / (ms * 1e-3), "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {**workload_config(args, world), "setup_s": t_setup,
                       "iterations_total": args.warmup + args.steps},
            "roofline": {**fp64_roofline(torch, g, cfg, args.dtype, world, ms / 2, ms / 2),
                         "note": "one A x and one A^T r launch per iteration; kernel time taken as "
                                 "half the iteration (the elementwise K8 steps are < 1 %)"},
            "updates_per_projection": nnz_live,
            "rank0_residual_norm": resid,
            "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk,
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_proj(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_csr(args):
    """K1/K2 consistent CSR assembly (bit-exact path) + K3/K4 on one GPU.
    One step = build_system_matrix (ctsm_csr_build: single-evaluation emission,
    row scan, record scatter, per-row radix sort) of the whole config; metric SM weights/s = nnz / build time. K3 A x and K4 A^T y
    on the built matrix are timed separately (HBM roofline: 12 B/nnz + 16
    B/row)."""
    import torch

    from paper_2511_12235_b200 import CONFIGS, _lib
    from paper_2511_12235_b200.phantoms import phantom_for, uniform_sinogram
    from paper_2511_12235_b200.projector import (back_project, build_system_matrix,
                                                 forward_project)

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
    # end to end: the matrix built AND copied to host memory (the reference
    # returns a host SparseSystemMatrix), where it fits a bounded run
    e2e = None
    csr_bytes = 12 * nnz + 8 * (w.n_rows + 1)
    if not args.no_e2e and csr_bytes < (8 << 30):
        hrs = torch.empty(w.n_rows + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(nnz, dtype=torch.int32).pin_memory()
        hval = torch.empty(nnz, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            w2 = build_system_matrix(g, memory_budget_bytes=budget)
            hrs.copy_(w2.row_start, non_blocking=True)
            hcol.copy_(w2.col, non_blocking=True)
            hval.copy_(w2.val, non_blocking=True)
            torch.cuda.synchronize()
            del w2
        te = (time.perf_counter() - t0) / args.steps
        e2e = {"value": nnz / te, "unit": "weights/s", "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": csr_bytes, "ms_per_step": te * 1e3,
               "calls": "build_system_matrix + the CSR copied to pinned host memory"}
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
    # K4 as a gather over the CSC transpose (ctsm_csc_build), when the copy
    # fits beside the CSR: same bits as the scatter (tests/test_gpu_parity.py)
    ms_spmvt_csc = ms_csc_build = None
    try:
        from paper_2511_12235_b200.projector import build_transpose, drop_transpose
        free_b, _tot = torch.cuda.mem_get_info()
        if free_b > 1.15 * (12.0 * nnz + 8.0 * w.n_cols):
            xs = back_project(w, yb)
            ev0.record()
            build_transpose(w)
            ev1.record()
            torch.cuda.synchronize()
            ms_csc_build = ev0.elapsed_time(ev1)
            for _ in range(3):
                xc = back_project(w, yb)
            assert torch.equal(xs, xc), "CSC back_project differs from the scatter"
            del xs, xc
            torch.cuda.synchronize()
            ms_spmvt_csc = 0.0
            for _ in range(5):
                ev0.record()
                back_project(w, yb)
                ev1.record()
                torch.cuda.synchronize()
                ms_spmvt_csc += ev0.elapsed_time(ev1) / 5
            drop_transpose(w)
    except torch.cuda.OutOfMemoryError:
        ms_spmvt_csc = None
    clk = clocks.stop()
    bytes_spmv = 12.0 * nnz + 16.0 * w.n_rows + 8.0 * w.n_cols
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    gbs = bytes_spmv / (ms_spmv * 1e-3) / 1e9
    # FP64 roofline of the emission kernel (K1 / K2): every
    # pixel/voxel-angle is evaluated (no symmetry on the bit-exact path), F
    # reference operations each, against the measured DFMA instruction rate.
    peak_flops = measure_dfma_peak(torch)
    per_unit = F_REF["2d"] if g.is_2d() else F_REF["3d"]
    units = float(g.n_x * g.n_y * g.n_z) * g.n_angles
    achieved = units * per_unit / (ms * 1e-3) / 1e12
    kname = "csr2d_kernel" if g.is_2d() else "emit3d_kernel"
    ncu = {}
    try:
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_kernels.json"))).get(
            f"{cfg}_csr:{kname}", {})
    except Exception:
        pass
    roof = {"bound": "fp64", "kernel": kname,
            "achieved": achieved, "peak": peak_flops / 2 if peak_flops else None,
            "unit": "T FP64 op/s (arithmetic instructions, FMA = 1 op; SURVEY.md §8(d))",
            "frac": achieved / (peak_flops / 2) if peak_flops else None,
            "traffic": ncu.get("dram_bytes"),
            "traffic_unit": "DRAM bytes per emission launch of the ncu capture (one chunk of "
                            "angles; profiles/ncu_kernels.json)",
            "ncu_fp64_pipe_active_pct": ncu.get("fp64_pipe_pct"),
            "ncu_launch_ms": ncu.get("duration_ms"),
            "work_per_unit": f"{per_unit:g} FP64 ops per pixel/voxel-angle (reference op count; "
                             "the crmath calls are excluded like the reference's libm calls)",
            "units_per_launch": units,
            "algorithmic_output_bytes": 12.0 * nnz + 8.0 * (w.n_rows + 1),
            "note": "whole build taken as the kernel time: per angle chunk the plan and emission "
                    "kernels (each weight evaluated once), the row scan, the record scatter and "
                    "the per-row radix sort (profiles/*_csr_c2_launches.csv gives the shares)"}
    line = {
        "metric": "SM weights/s (consistent CSR assembly)", "value": nnz / (ms * 1e-3),
        "unit": "weights/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, 1),
        "nnz": nnz, "nnz_reference": NNZ.get(cfg),
        "roofline": roof,
        "spmv": {"ms": ms_spmv, "GB/s": gbs, "algorithmic_bytes": bytes_spmv,
                 "hbm_peak_gbs": peaks.get("hbm_gbs"), "frac": gbs / peaks.get("hbm_gbs", 6650.0)},
        "spmv_t": {"ms": ms_spmvt, "GB/s": bytes_spmv / (ms_spmvt * 1e-3) / 1e9,
                   "algorithmic_bytes": bytes_spmv,
                   "frac": bytes_spmv / (ms_spmvt * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                   "note": "back_project: int64 fixed-point scatter (deterministic) with the matrix's "
                           "column-sum bound, computed once per matrix (cached, outside the timed calls)"},
        "spmv_t_csc": None if ms_spmvt_csc is None else {
            "ms": ms_spmvt_csc, "GB/s": bytes_spmv / (ms_spmvt_csc * 1e-3) / 1e9,
            "frac": bytes_spmv / (ms_spmvt_csc * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
            "transpose_build_ms": ms_csc_build,
            "note": "back_project as a gather over a CSC transpose kept beside the CSR "
                    "(build_transpose; bit-identical to the scatter, checked in this run)"},
        "e2e": e2e,
        "gpu_launches": int(launches), "clocks": clk,
    }
    if not args.no_cpu:
        del w, x, yb
        try:
            n_ref, t_ref, desc, variant, cores = csr_reference_sample(cfg, 12.0)
            line["cpu_baseline"] = {"value": n_ref / t_ref, "unit": "weights/s", "cores": cores,
                                    "kind": "reference" if variant == "ref_glibc" else "port",
                                    "sample": desc, **host_info()}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"error": repr(e)}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    relaunch_if_needed(args)
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
