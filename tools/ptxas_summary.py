"""Registers / spills of the main kernel instances from a ptxas -v log
(tools/build_variants.py writes <lib>.ptxas.txt):
    python tools/ptxas_summary.py build/variants/<lib>.so.ptxas.txt"""
import re
import subprocess
import sys

KEYS = ("render_cameras_kernel<1, 0", "wave_kernel<1", "render_hierarchy_kernel<1",
        "persistent_kernel<1", "trace_rays_kernel<1")
t = open(sys.argv[1]).read()
for b in re.split(r"ptxas info\s+: Compiling entry function '", t)[1:]:
    name = b.split("'")[0]
    dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    if not any(k in dn for k in KEYS):
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", b)
    r = re.search(r"Used (\d+) registers", b)
    short = re.search(r"(\w+_kernel<[^>]*>)", dn).group(1)
    print(f"{short:40s} regs {r.group(1):>4s} stack {m.group(1):>4s} "
          f"spill st {m.group(2):>4s} ld {m.group(3):>4s}")
