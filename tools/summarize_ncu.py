"""Write the committed summary of an ncu --set full capture:
    python tools/summarize_ncu.py <report.ncu-rep> <out_prefix>
-> <out_prefix>_details.txt (sections), _stalls.txt (warp stall sampling,
   pipe utilisation, DRAM bytes), _hot_lines.txt (per source line) and
   prints the DRAM bytes per launch (for profiles/ncu_traffic.json)."""
import csv
import os
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]


def ncu_csv(*args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True,
                         text=True).stdout
    return list(csv.reader(out.splitlines()))


rows = ncu_csv("--page", "details")
h = rows[0]
si, mi, ui, vi = (h.index(k) for k in ("Section Name", "Metric Name",
                                        "Metric Unit", "Metric Value"))
kname = rows[1][h.index("Kernel Name")] if "Kernel Name" in h else "?"
with open(prefix + "_details.txt", "w") as f:
    f.write(f"ncu --set full: {os.path.basename(rep)}\nkernel: {kname}\n")
    for r in rows[1:]:
        if r[mi]:
            f.write(f"{r[si][:28]:28s} {r[mi][:55]:55s} {r[vi]:>14s} {r[ui]}\n")

raw = ncu_csv("--page", "raw")
h, u, v = raw[0], raw[1], raw[2]
stalls = []
dram = 0.0
with open(prefix + "_stalls.txt", "w") as f:
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled") and \
                not name.endswith("not_issued"):
            stalls.append((float(v[i].replace(",", "") or 0), name))
    tot = sum(x for x, _ in stalls) or 1
    f.write("warp stall sampling (share of samples)\n")
    for val, name in sorted(stalls, reverse=True):
        if val:
            f.write(f"{100 * val / tot:6.2f}%  {name}\n")
    f.write("\nselected raw metrics\n")
    for i, name in enumerate(h):
        if any(k in name for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                   "lts__t_bytes.sum", "pipe_fp64_cycles_active.avg.pct",
                                   "inst_executed_pipe_fma.avg.pct",
                                   "inst_executed_pipe_alu.avg.pct",
                                   "inst_executed_pipe_xu.avg.pct",
                                   "inst_executed_pipe_lsu.avg.pct",
                                   "thread_inst_executed_per_inst_executed.ratio",
                                   "launch__registers_per_thread",
                                   "sm__warps_active.avg.pct")):
            f.write(f"{name:90s} {v[i]:>16s} {u[i]}\n")
            if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[i], 1)
                dram += float(v[i].replace(",", "")) * scale

src = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source",
                      "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
tmp = prefix + "_src.tmp.csv"
open(tmp, "w").write(src)
lines = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__),
                                                     "ncu_lines.py"), tmp, "40"],
                       capture_output=True, text=True).stdout
os.remove(tmp)
with open(prefix + "_hot_lines.txt", "w") as f:
    f.write("share of warp-stall samples | executed warp instructions | line\n")
    f.write(lines)
print(int(dram))
