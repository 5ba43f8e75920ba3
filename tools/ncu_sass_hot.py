"""Summarise an ncu --page source --csv export (SASS view): stall samples
and executed instructions per opcode, plus the hottest instructions."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
S = hdr.index("Warp Stall Sampling (All Samples)")
E = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[S] or 0) for r in data)
print(f"samples {tot}  warp-instructions {sum(int(r[E] or 0) for r in data)}")
op, opi = collections.Counter(), collections.Counter()
reasons = collections.Counter()
for r in data:
    toks = r[1].split()
    o = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    o = o.split(".")[0]
    op[o] += int(r[S] or 0)
    opi[o] += int(r[E] or 0)
    for i in stall_cols:
        reasons[hdr[i]] += int(r[i] or 0)
for o, v in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 18):
    print(f"  {o:10s} samples {v:7d} ({100 * v / max(1, tot):5.1f}%)  instr {opi[o]}")
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / max(1, tot):.1f}%" for k, v in reasons.most_common(8)))
