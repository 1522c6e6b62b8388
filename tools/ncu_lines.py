"""Summarise an `ncu --page source --print-source=cuda,sass --csv` export:
per source line warp-stall samples and executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
path = None
hdr = None
agg = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or not r[0].isdigit():
        continue
    try:
        s = float(r[4] or 0)
        ie = float(r[7] or 0)
    except ValueError:
        continue
    key = (path, int(r[0]))
    a = agg.setdefault(key, [0.0, 0.0, r[1][:100]])
    a[0] += s
    a[1] += ie
tot = sum(v[0] for v in agg.values()) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for (f, l), (s, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * s / tot:5.1f}% {ie / 1e6:8.2f}M {f}:{l:<4d} {src}")
