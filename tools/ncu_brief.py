"""Prints the headline metrics of every kernel in an .ncu-rep (raw page):
duration, FP64 pipe, issue active, active lanes, occupancy, DRAM bytes, local
memory sectors and the stall-reason shares of the PC samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
keys = [("gpu__time_duration.sum", "time"), ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "registers"), ("smsp__inst_executed.sum", "warp instructions"),
        ("dram__bytes_read.sum", "dram read"), ("dram__bytes_write.sum", "dram write"),
        ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local ld sectors"),
        ("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", "local st sectors"),
        ("lts__t_sectors_op_atom.sum", "L2 atom sectors"), ("lts__t_sectors_op_red.sum", "L2 red sectors")]
for r in rows[2:]:
    print("==", r[idx["Kernel Name"]][:90])
    for k, label in keys:
        if k in idx:
            print("  %-20s %s %s" % (label, r[idx[k]], rows[1][idx[k]]))
    total = float(r[idx["smsp__pcsamp_sample_count"]]) if "smsp__pcsamp_sample_count" in idx else 0
    stalls = []
    for h, i in idx.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(v for v, _ in stalls) or 1
    print("  stalls: " + ", ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in stalls[:7]))
