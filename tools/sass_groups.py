"""Group the SASS of an `ncu --page source --print-source=cuda,sass --csv`
export by execution count (instructions executed the same number of times
form one basic-block family -- loop bodies show up as large groups):
    python tools/sass_groups.py <source.csv> [top] [show_count]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
path = cur = None
sass = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Function Name"):
        continue
    if r[0].isdigit():
        cur = (path, int(r[0]))
        continue
    if r[2].startswith("0x") and r[7] not in ("-", ""):
        a = int(r[2], 16)
        if a in sass:
            sass[a][0].append(cur[1])
        else:
            sass[a] = [[cur[1]], r[3].strip(), int(r[7])]
items = sorted(sass.items())
tot = sum(v[2] for _, v in items)
print(f"warp instructions executed: {tot}")
hist = collections.Counter(v[2] for _, v in items)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
for n, k in sorted(hist.items(), key=lambda x: -x[0] * x[1])[:top]:
    print(f"{n:10d} x {k:4d} = {n * k:11d}  {100 * n * k / tot:5.1f}%")
if len(sys.argv) > 3:
    show = int(sys.argv[3])
    for a, v in items:
        if v[2] == show:
            print(hex(a)[-5:], v[0], v[1][:70])
