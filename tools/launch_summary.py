"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel: count, total, share, average.  python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total_us':>11} {'share':>6} {'avg_us':>9}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t / 1e3:11.1f} {100 * t / tot:5.1f}% {t / n / 1e3:9.2f}  {k}")
