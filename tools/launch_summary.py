"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total us and
launch count per kernel, largest first.  python tools/launch_summary.py FILE"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if len(r) > 10 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"][:70]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"])
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t / 1e3:10.1f} us  {c:5d}  {t / 1e3 / c:8.2f} us/launch  {k}")
