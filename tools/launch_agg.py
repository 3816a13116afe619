"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel.

    python tools/launch_agg.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"]) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1)
    a = agg.setdefault(d["Kernel Name"][:70], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, t) in agg.items():
    print(f"{n:5d} {t / n / 1000:9.2f} us avg {100 * t / tot:5.1f}%  {k}")
print(f"total {tot / 1000:.1f} us")
