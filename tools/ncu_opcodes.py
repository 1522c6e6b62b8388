"""Opcode histogram (warp instructions, average active lanes, stall samples)
of an ncu source-page CSV export, plus the stall-reason totals.
usage: ncu_opcodes.py export.csv"""
import csv, os, re, sys
csv.field_size_limit(1 << 30)
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; opc = {}; tot_w = 0; stalls = {}
for r in rows:
    if not r: continue
    if r[0] == "Line No": hdr = r; continue
    if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
        try: wi = float(r[7] or 0); ti = float(r[8] or 0); s = float(r[4] or 0)
        except ValueError: continue
        tot_w += wi
        m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_.]+)", r[3].strip())
        op = m.group(2).split('.')[0] if m else '?'
        if op in ("LDG", "LD", "LDL", "STL", "LDS", "STS", "STG", "MUFU", "F2F", "I2F", "F2I"):
            op = ".".join(m.group(2).split('.')[:2]) if op in ("MUFU", "F2F") else op
        o = opc.setdefault(op, [0, 0, 0]); o[0] += wi; o[1] += ti; o[2] += s
        for i, k in enumerate(hdr):
            if k.startswith("stall_") and "Not Issued" not in k and i < len(r):
                try: stalls[k] = stalls.get(k, 0) + float(r[i] or 0)
                except ValueError: pass
ts = sum(v[2] for v in opc.values()) or 1
print("total warp instr %.1fM" % (tot_w / 1e6))
st = sum(stalls.values()) or 1
print("stalls:", {k[6:]: round(100 * v / st, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:9]})
for op, (wi, ti, s) in sorted(opc.items(), key=lambda kv: -kv[1][0])[:32]:
    print(f"{op:12s} {100*wi/tot_w:5.1f}%  lanes {ti/wi if wi else 0:5.1f}  samples {100*s/ts:5.1f}%")
