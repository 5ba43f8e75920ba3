"""Run bench.py once per liblopc variant (LOPC_LIB) and print the step and
per-kernel times side by side."""
import glob
import json
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
for so in sorted(glob.glob("variants/liblopc_*.so")):
    env = dict(os.environ, LOPC_LIB=os.path.abspath(so))
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "5", "--warmup", "3", "--no-cpu-baseline"],
                       env=env, capture_output=True, text=True, timeout=600)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        pk = {k: round(v["ms"], 4) for k, v in d["per_kernel"].items()}
        print(os.path.basename(so), f"value {d['value']:.1f} comp {d['compress_GBps']:.1f} dec {d['decompress_GBps']:.1f}"
              f" e2e {d['e2e']['value']:.2f}",
              pk, "viol", d["order_violations"], d["bound_violations"], flush=True)
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(so), "FAILED", e, r.stderr[-2000:], flush=True)
