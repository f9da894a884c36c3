"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: launches, total us, share.

usage: python scripts/launch_summary.py launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) > 5 and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
        k = r[hdr["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r[hdr["Metric Value"]].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:30s} {n:5d} {t / 1e3:11.1f} us {100 * t / tot:5.1f}%")
print(f"{'total':30s} {'':5s} {tot / 1e3:11.1f} us")
