"""Top source lines by warp-stall samples from `ncu --page source --csv
--print-source cuda,sass` output: python tools/ncu_lines.py file.csv [N]."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
fname = "?"
hdr = None
agg = defaultdict(lambda: [0, 0, "", defaultdict(int)])
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or not r[0].isdigit() or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0))
    except ValueError:
        continue
    key = (fname, int(r[0]))
    a = agg[key]
    a[0] += s
    a[2] = r[1][:90]
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                a[3][k] += int(float(v or 0))
            except ValueError:
                pass
tot = sum(a[0] for a in agg.values()) or 1
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    top = sorted(a[3].items(), key=lambda kv: -kv[1])[:3]
    print(f"{a[0] / tot * 100:5.1f}% {f}:{ln:<5} {a[2]:<90} {' '.join(f'{k[6:]}={v}' for k, v in top)}")
