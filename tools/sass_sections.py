"""Summarise an ncu --page source --csv (SASS) dump: instructions and stall
samples per section (sections split at barriers), plus opcode totals."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
ii = hdr.index("Instructions Executed")
src = hdr.index("Source")
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ii] or 0) for r in data)
tots = sum(float(r[si] or 0) for r in data)
print(f"{sys.argv[1]}: {len(data)} SASS lines, {tot:.3e} warp-instructions")
cum = cs = last = lasts = 0.0
lastk = 0
for k, r in enumerate(data):
    cum += float(r[ii] or 0)
    cs += float(r[si] or 0)
    s = r[src]
    if "BAR.SYNC" in s or "EXIT" in s or k == len(data) - 1:
        if (cum - last) / tot > 0.02 or (cs - lasts) / tots > 0.02:
            print(f"  [{lastk:5d}-{k:5d}] inst {(cum - last) / tot * 100:5.1f}%  stall {(cs - lasts) / tots * 100:5.1f}%  {s.strip()[:40]}")
        last, lasts, lastk = cum, cs, k
op = collections.Counter()
for r in data:
    t = r[src].split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    op[o.split(".")[0]] += float(r[ii] or 0)
print("  top opcodes:", ", ".join(f"{o} {v / tot * 100:.0f}%" for o, v in op.most_common(12)))
