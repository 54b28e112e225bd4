"""Per-source-line breakdown (warp-stall samples, executed warp instructions)
of the kernels in an ncu report (needs -lineinfo + --import-source on).

Usage: python tools/ncu_lines.py gpurun_out/prof_r1c.ncu-rep [kernel-substring] [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    want = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    cur_file = cur_fn = hdr = None
    agg = collections.defaultdict(lambda: [0, 0, "", 0])
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "Line No" and "--header" in sys.argv:
            print(list(enumerate(r)))
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            cur_fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit() or (want and want not in (cur_fn or "")):
            continue
        try:
            s, ie = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        # thread-level instruction count (active lanes per line), when present
        ti_col = next((i for i, h in enumerate(hdr) if h.strip() == "Thread Instructions Executed"), None)
        try:
            te = int(r[ti_col] or 0) if ti_col is not None else 0
        except ValueError:
            te = 0
        key = (cur_fn[:60], cur_file, int(r[0]))
        agg[key][0] += s
        agg[key][1] += ie
        agg[key][2] = r[1][:90]
        agg[key][3] += te
    for fn in sorted(set(k[0] for k in agg)):
        sub = [(k, v) for k, v in agg.items() if k[0] == fn]
        ts = sum(v[0] for _, v in sub) or 1
        ti = sum(v[1] for _, v in sub) or 1
        print(f"===== {fn}  samples={ts} warp_instr={ti}")
        for k, v in sorted(sub, key=lambda x: -x[1][0])[:top]:
            lanes = f"{v[3] / v[1]:5.1f} ln " if v[3] and v[1] else ""
            print(f"{100 * v[0] / ts:5.1f}% samp {100 * v[1] / ti:5.1f}% inst {lanes} {k[1]}:{k[2]}  {v[2]}")


if __name__ == "__main__":
    main()
