"""Summarise an ncu report (.ncu-rep) into profiles/<tag>_ncu_summary.md.

Usage: python tools/ncu_summary.py gpurun_out/prof_r1c.ncu-rep r1c
"""
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "FP64 pipe % (elapsed)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / warp-instr"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 RED sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local-memory load sectors"),
]


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    out = [f"# ncu summary {tag} ({os.path.basename(rep)}, --set full --clock-control none)", ""]
    for d in data:
        name = d[idx["Kernel Name"]]
        out.append(f"## {name[:110]}")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for key, label in METRICS:
            if key in idx:
                out.append(f"| {label} (`{key}`) | {d[idx[key]]} {units[idx[key]]} |")
        st = [(h, float(d[idx[h]] or 0)) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        st = sorted([x for x in st if x[1] > 0], key=lambda x: -x[1])[:6]
        out.append("| top stall reasons (pc sampling) | " +
                   ", ".join(f"{h[len('smsp__pcsamp_warps_issue_stalled_'):]} {100 * v / tot:.0f}%"
                             for h, v in st) + " |")
        out.append("")
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        f"{tag}_ncu_summary.md")
    open(path, "w").write("\n".join(out) + "\n")
    print(path)


if __name__ == "__main__":
    main()
