"""Per-kernel DRAM bytes and serialised time of an
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv`
launch log (tools/evidence.sh: c5_traffic.csv), one line per kernel name:
    python tools/ncu_traffic_sum.py <log.csv>"""
import csv
import sys
from collections import OrderedDict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3, "B": 1, "KB": 1e3, "MB": 1e6,
         "GB": 1e9, "TB": 1e12}

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
hdr = rows[0]
col = {k: i for i, k in enumerate(hdr)}
agg = OrderedDict()
for r in rows[1:]:
    if len(r) != len(hdr) or not r[col["ID"]].isdigit():
        continue
    name = r[col["Kernel Name"]][:48]
    a = agg.setdefault(name, {"n": set(), "read": 0.0, "write": 0.0, "ms": 0.0})
    a["n"].add(r[col["ID"]])
    v = float(r[col["Metric Value"]].replace(",", ""))
    unit = r[col["Metric Unit"]]
    m = r[col["Metric Name"]]
    if m == "dram__bytes_read.sum":
        a["read"] += v * SCALE[unit]
    elif m == "dram__bytes_write.sum":
        a["write"] += v * SCALE[unit]
    elif m == "gpu__time_duration.sum":
        a["ms"] += v * SCALE[unit]
tot = {"read": 0.0, "write": 0.0, "ms": 0.0}
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"{name:48s} launches {len(a['n']):4d}  read {a['read'] / 1e9:9.2f} GB  "
          f"write {a['write'] / 1e9:8.2f} GB  time {a['ms']:9.2f} ms")
    for k in tot:
        tot[k] += a[k]
print(f"{'total':48s} {'':14s} read {tot['read'] / 1e9:9.2f} GB  "
      f"write {tot['write'] / 1e9:8.2f} GB  time {tot['ms']:9.2f} ms")
