"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = None
    agg = collections.defaultdict(list)
    for r in rows:
        if h is None:
            if "Kernel Name" in r:
                h = r
            continue
        if len(r) < len(h):
            continue
        k = r[h.index("Kernel Name")].split("(")[0]
        agg[k[:40]].append(float(r[h.index("Metric Value")]) / 1e3)
    print(path)
    for k, v in agg.items():
        v2 = sorted(v)
        big = [x for x in v if x > 5.0] or v
        print(f"  {k:40s} n={len(v):3d} median={v2[len(v2)//2]:8.1f}us  median(>5us)={sorted(big)[len(big)//2]:8.1f}us")
