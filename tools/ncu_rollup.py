"""Roll an `ncu --page source --csv --print-source=cuda,sass` export up by
function (line ranges of the csrc files): warp-stall samples and thread
instructions executed per region.
    python tools/ncu_rollup.py <source.csv>"""
import csv
import re
import sys
from collections import defaultdict

CSRC = "paper_2507_14624_b200/csrc/"


def regions(path):
    """(first_line, name) of each top-level function in a .cuh/.cu file."""
    out = []
    pat = re.compile(r"^(?:template <[^>]*>\s*)?(?:__device__|__global__|static|"
                     r"inline|[A-Za-z_][\w:<>, ]*\s)[^;{]*?\b([A-Za-z_]\w*)\s*\(")
    lines = open(path).read().split("\n")
    for i, l in enumerate(lines, 1):
        if l.startswith((" ", "\t", "/", "#", "}")) or not l.strip():
            continue
        m = re.search(r"\b([A-Za-z_]\w*)\s*\(", l)
        if m and m.group(1) not in ("if", "for", "while", "return", "sizeof"):
            out.append((i, m.group(1)))
    return out


def locate(regs, line):
    name = "?"
    for first, n in regs:
        if first <= line:
            name = n
        else:
            break
    return name


rows = list(csv.reader(open(sys.argv[1])))
path = None
agg = defaultdict(lambda: [0.0, 0.0])
regcache = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]
        continue
    if r[0] in ("Line No", "Function Name") or not r[0].isdigit():
        continue
    try:
        samples = float(r[4] or 0)
        tinst = float(r[8] or 0)
    except (ValueError, IndexError):
        continue
    fname = path.split("/")[-1]
    if CSRC in path:
        if path not in regcache:
            try:
                regcache[path] = regions(path)
            except OSError:
                regcache[path] = []
        key = f"{fname}:{locate(regcache[path], int(r[0]))}"
    else:
        key = fname
    agg[key][0] += samples
    agg[key][1] += tinst
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{'stall%':>7} {'inst%':>7} {'thread-inst':>14}  region")
for k, (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if s / ts < 0.002 and i / ti < 0.002:
        continue
    print(f"{100 * s / ts:6.1f}% {100 * i / ti:6.1f}% {i:14.0f}  {k}")
print(f"total thread instructions {ti:.4g}")
