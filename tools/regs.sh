#!/bin/bash
# Registers / spills per kernel instance of lfp_capi.cu (ptxas -v), demangled-ish.
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
  -Xptxas -v -Xcompiler -fPIC -shared $@ -o /tmp/regs_probe.so paper_2507_14624_b200/csrc/lfp_capi.cu 2>&1 |
python3 -c '
import sys,re
name=None
for l in sys.stdin:
    m=re.search(r"Function properties for (\S+)",l)
    if m: name=m.group(1); st=""; continue
    m=re.search(r"(\d+) bytes spill stores",l)
    if m and name: st=m.group(1); continue
    m=re.search(r"Used (\d+) registers",l)
    if m and name:
        k=re.search(r"(render_cameras_kernel|persistent_kernel|trace_rays_kernel|render_hierarchy_kernel|render_probes_kernel|trace_source_kernel)I(\w+?)EEv",name)
        if k: print(f"{k.group(1):28s} {k.group(2):20s} regs={m.group(1):4s} spill={st}")
        name=None
'
