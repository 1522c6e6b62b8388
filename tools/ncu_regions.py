"""Per-function roll-up of an `ncu --page source --csv --print-source=cuda,sass`
export: share of warp-stall samples, executed warp / thread instructions and
average active lanes, with source lines assigned to the enclosing (inlined)
device function of the repo's .cu/.cuh files.
usage: ncu_regions.py export.csv [csrc_dir]"""
import csv
import os
import re
import sys

csv.field_size_limit(1 << 30)
src_dir = sys.argv[2] if len(sys.argv) > 2 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_2507_14624_b200", "csrc")


def functions(path):
    """line -> function name (header line search; good enough for roll-ups)"""
    out = {}
    cur = "(file scope)"
    pend = False
    for n, line in enumerate(open(path, errors="replace"), 1):
        s = line.rstrip()
        if re.match(r"^(template|__device__|__global__|static\s+__device__)", s):
            pend = True
        if pend:
            m = re.search(r"([A-Za-z_][A-Za-z_0-9]*)\s*\($", s) or \
                re.search(r"([A-Za-z_][A-Za-z_0-9]*)\s*\([^;]*$", s)
            if m and m.group(1) not in ("__launch_bounds__", "__forceinline__"):
                cur = m.group(1)
                pend = False
        out[n] = cur
    return out


rows = list(csv.reader(open(sys.argv[1])))
path = None
hdr = None
agg = {}
fmap = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1]
        base = os.path.basename(path)
        cand = os.path.join(src_dir, base)
        fmap[base] = functions(cand) if os.path.exists(cand) else {}
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        s = float(r[4] or 0)
        wi = float(r[7] or 0)
        ti = float(r[8] or 0)
    except ValueError:
        continue
    base = os.path.basename(path)
    fn = fmap.get(base, {}).get(int(r[0]), base)
    a = agg.setdefault((base, fn), [0.0, 0.0, 0.0])
    a[0] += s
    a[1] += wi
    a[2] += ti
ts = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
tt = sum(v[2] for v in agg.values()) or 1
print(f"total: {tw / 1e6:.1f} M warp instr, {tt / 1e6:.1f} M thread instr, "
      f"avg active lanes {tt / tw:.2f}")
print(" samples%  warp-instr%  thread-instr%  lanes  function")
for (f, fn), (s, wi, ti) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    if wi / tw < 0.002 and s / ts < 0.002:
        continue
    print(f"  {100 * s / ts:6.2f}    {100 * wi / tw:6.2f}      {100 * ti / tt:6.2f}     "
          f"{ti / wi if wi else 0:5.1f}  {f}:{fn}")
