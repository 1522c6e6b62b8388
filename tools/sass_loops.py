"""List the loops of one kernel's SASS (nvdisasm -g -c output): backward
branches, instruction count of the loop body and what it contains (local
memory traffic, fp64 ops, conversions). Usage:
    python tools/sass_loops.py kernel.sass [min_len]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
min_len = int(sys.argv[2]) if len(sys.argv) > 2 else 10
labels, insts = {}, []
cur_line = None
for l in lines:
    m = re.match(r"^(\.L_x_\d+):", l.strip())
    if m:
        labels[m.group(1)] = len(insts)
        continue
    m = re.search(r'line (\d+)', l)
    if "//##" in l and m:
        cur_line = (l.split('"')[1].split("/")[-1], int(m.group(1)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        insts.append((m.group(1), m.group(2).strip(), cur_line))
for i, (addr, txt, src) in enumerate(insts):
    m = re.search(r"BRA (?:!?U?P\d+, )?`\((\.L_x_\d+)\)", txt)
    if not m or m.group(1) not in labels:
        continue
    j = labels[m.group(1)]
    if j > i or i - j < min_len:
        continue
    body = insts[j:i + 1]
    ops = Counter(t.split()[0].lstrip("@!P0123456789T ").split(".")[0]
                  if not t.startswith("@") else t.split()[1].split(".")[0]
                  for _, t, _ in body)
    srcs = Counter(s for _, _, s in body if s)
    top = ", ".join(f"{f}:{ln}" for (f, ln), _ in srcs.most_common(4))
    interesting = {k: v for k, v in ops.items()
                   if k in ("LDL", "STL", "I2F", "F2F", "DMUL", "DADD", "DFMA",
                            "DSETP", "LDG", "LDS", "STS", "MUFU", "CALL")}
    print(f"loop {insts[j][0]}..{addr} len {i - j + 1:4d} {interesting} | {top}")
