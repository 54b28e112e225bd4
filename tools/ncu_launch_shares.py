"""Kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv):
python tools/ncu_launch_shares.py profiles/x_launches.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= mv:
        continue
    v = float(r[mv].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r[mu], 1e-6)
    name = r[kn].split("(")[0].split("::")[-1][-44:]
    agg[name] += v
    cnt[name] += 1
tot = sum(agg.values())
print(f"total {tot:.2f} ms in {sum(cnt.values())} launches")
for k, v in agg.most_common(top):
    print(f"{100 * v / tot:6.1f}% {v:10.2f} ms {cnt[k]:6d}  {k}")
