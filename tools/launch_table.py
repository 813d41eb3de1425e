"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
total and per-kernel time.  Usage: python tools/launch_table.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mi = h.index("Metric Name") if "Metric Name" in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(r[ui], 1.0)
    short = r[ki].split("(")[0][:80]
    agg[short][0] += 1
    agg[short][1] += v
    tot += v
print(f"total {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{t / 1e3:8.3f} ms {n:5d}  {k}")
