"""Stall samples and executed warp instructions per CUDA source line from an
ncu `--page source --csv --print-source cuda,sass` export (per kernel)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))


def num(v):
    try:
        return int(v)
    except ValueError:  # "-", or a source line whose quotes broke the CSV
        return 0


top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
fn = fp = None
hdr = None
agg = collections.defaultdict(collections.Counter)
ex = collections.defaultdict(collections.Counter)
reasons = collections.defaultdict(lambda: collections.defaultdict(collections.Counter))
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fp = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        fn = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    key = (fp, int(r[0]), r[1].strip()[:80])
    agg[fn][key] += num(r[4])
    ex[fn][key] += num(r[7])
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("-", ""):
            reasons[fn][key][h[6:]] += num(r[i])
for f in agg:
    tot = sum(agg[f].values())
    print(f"== {f}  samples {tot}  warp-instructions {sum(ex[f].values())}")
    for key, v in agg[f].most_common(top):
        rs = ", ".join(f"{k} {100 * c / max(1, v):.0f}%" for k, c in reasons[f][key].most_common(2))
        print(f"  {key[0][:14]}:{key[1]:<5d} {100 * v / max(1, tot):5.1f}%  ex {ex[f][key]:>10d}  [{rs}]  {key[2]}")
