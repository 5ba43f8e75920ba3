"""Static SASS section sizes of the kernels in liblopc.so (split at BAR.SYNC),
a fast local proxy for per-warp instruction counts of straight-line code."""
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_26968_b200/liblopc.so"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat and pat not in name:
        continue
    ins = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
    secs, cur = [], 0
    for l in ins:
        cur += 1
        if "BAR.SYNC" in l or "EXIT" in l:
            secs.append(cur)
            cur = 0
    secs.append(cur)
    print(f"{name[:70]:70s} total {len(ins):5d}  sections {secs}")
