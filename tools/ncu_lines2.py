"""Per source line of one file from an ncu source-page CSV: warp instr (M),
avg lanes, samples%. usage: ncu_lines2.py export.csv file.cuh lo hi"""
import csv, sys, os
csv.field_size_limit(1 << 30)
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2]; lo = int(sys.argv[3]); hi = int(sys.argv[4])
path = None; agg = {}; tot = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": path = os.path.basename(r[1]); continue
    if not r[0].isdigit(): continue
    try: s = float(r[4] or 0); wi = float(r[7] or 0); ti = float(r[8] or 0)
    except ValueError: continue
    tot += s
    if path != want: continue
    a = agg.setdefault(int(r[0]), [0, 0, 0, r[1][:90]])
    a[0] += s; a[1] += wi; a[2] += ti
for l in sorted(agg):
    if lo <= l <= hi:
        s, wi, ti, src = agg[l]
        print(f"{l:5d} {100*s/tot:5.2f}% {wi/1e6:8.1f}M lanes {ti/wi if wi else 0:5.1f}  {src}")
