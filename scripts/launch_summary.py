"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): per-kernel
count, total and mean time, share.  usage: launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:40]:40s} {n:8d} {t / 1e3:10.2f} {t / n:10.1f} {t / tot:6.3f}")
print(f"{'total':40s} {sum(a[0] for a in agg.values()):8d} {tot / 1e3:10.2f}")
