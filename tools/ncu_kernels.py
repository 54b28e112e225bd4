"""Extract per-kernel ncu figures (one --set full capture) into
profiles/ncu_kernels.json, which bench.py reads for roofline.traffic.

Usage: python tools/ncu_kernels.py gpurun_out/prof_r1n.ncu-rep <config> [<config> ...]
(config labels the workload the capture ran, e.g. c1_f64; one per kernel in
capture order, or one for all). Entries are keyed by config and kernel name
(the template signature up to the first '('), e.g. "c1_f64:fwd2d_d8_kernel<double>".
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_kernels.json")
METRICS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__inst_executed_op_global_red.sum": "global_red_warp_insts",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_lanes",
    "sm__cycles_elapsed.max": "sm_cycles",
}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "%": 1.0, "inst": 1.0, "cycle": 1.0}


def main():
    rep, cfgs = sys.argv[1], sys.argv[2:]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for n, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").split("::")[-1]
        cfg = cfgs[min(n, len(cfgs) - 1)] if cfgs else "unlabelled"
        e = {"report": os.path.basename(rep)}
        for m, key in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                unit = units[i]
                v *= SCALE.get(unit, 1.0)
                if key == "duration_ms" and unit in ("ns", "us", "ms", "s"):
                    pass
                e[key] = v
        e["dram_bytes"] = e.get("dram_read_bytes", 0.0) + e.get("dram_write_bytes", 0.0)
        data[f"{cfg}:{short}"] = e
        print(f"{cfg}:{short}", e)
    json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
