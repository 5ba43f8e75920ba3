"""Summarise a round's ncu captures into profiles/ (tracked).

  python tools/ncu_summary.py TAG [--config cfg2]

Reads gpurun_out/full_TAG.ncu-rep (ncu --set full, one launch of every kernel
of one compress+decompress step) and gpurun_out/launches_TAG.csv (ncu
gpu__time_duration launch list of `bench.py --steps 2 --warmup 1`), writes
  profiles/TAG_ncu_summary.json   per-kernel metrics (duration, DRAM bytes,
                                  throughput, IPC, occupancy, top stalls, pipes)
  profiles/TAG_launches.csv       the launch list (our kernels only)
  profiles/traffic_CONFIG.json    dram read+write bytes per launch (bench.py's
                                  roofline.traffic)
  profiles/warpinst_CONFIG.json   warp instructions per launch (bench.py's
                                  issue roofline)
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "cfg2"
rep = os.path.join(ROOT, "gpurun_out", f"full_{tag}.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("lopc::", "")
    return n.split("<")[0]


def num(d, k):
    v = d.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


out = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    k = short(d["Kernel Name"])
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}

    def nbytes(key):
        v = num(d, key)
        return None if v is None else v * mult.get(u.get(key, "byte"), 1)

    dur_ns = num(d, "gpu__time_duration.sum") * {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(
        u.get("gpu__time_duration.sum"), 1)
    stalls = sorted(((kk.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      num(d, kk)) for kk in d if kk.startswith("smsp__average_warps_issue_stalled_")
                     and kk.endswith("_per_issue_active.ratio") and num(d, kk) is not None), key=lambda t: -t[1])
    pipes = {kk.replace("sm__inst_executed_pipe_", "").replace(".avg.pct_of_peak_sustained_active", ""): num(d, kk)
             for kk in d if kk.startswith("sm__inst_executed_pipe_") and kk.endswith(".avg.pct_of_peak_sustained_active")
             and (num(d, kk) or 0) > 5}
    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    entry = {
        "kernel": d["Kernel Name"], "grid": d.get("Grid Size"), "block": d.get("Block Size"),
        "duration_us": dur_ns / 1e3,
        "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_GBps": (rd + wr) / dur_ns if rd is not None and wr is not None else None,
        "dram_pct_peak": num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "ipc_active": num(d, "sm__inst_executed.avg.per_cycle_active"),
        "warp_instructions": num(d, "smsp__inst_executed.sum"),
        "achieved_occupancy_pct": num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num(d, "launch__registers_per_thread"),
        "smem_per_block": num(d, "launch__shared_mem_per_block_dynamic"),
        "top_stalls": stalls[:6],
        "pipes_pct": pipes,
        "shared_bank_conflicts_ld": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "shared_bank_conflicts_st": num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"),
    }
    key = k if k not in out else k + "_2"
    out[key] = entry

prof = os.path.join(ROOT, "profiles")
os.makedirs(prof, exist_ok=True)
json.dump({"source": f"ncu --set full --clock-control none, tools/prof_step.py {config} (second step)",
           "kernels": out}, open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w"), indent=1)
traffic = {}
for k, v in out.items():
    name = k[:-2] if k.endswith("_2") and k.startswith("k_encode") else k  # the two encode roles: one step's encode
    traffic[name] = traffic.get(name, 0) + (v["dram_read_bytes"] or 0) + (v["dram_write_bytes"] or 0)
json.dump(traffic, open(os.path.join(prof, f"traffic_{config}.json"), "w"), indent=1)
winst = {}
for k, v in out.items():
    name = k[:-2] if k.endswith("_2") and k.startswith("k_encode") else k
    winst[name] = winst.get(name, 0) + (v["warp_instructions"] or 0)
json.dump({"source": f"{tag}_ncu_summary.json smsp__inst_executed.sum per launch", "kernels": winst},
          open(os.path.join(prof, f"warpinst_{config}.json"), "w"), indent=1)

# launch list: our kernels only, plus each kernel's share of the step
lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(lp):
    lines = [ln for ln in open(lp) if ln.startswith('"')]
    lr = list(csv.reader(lines))
    h = lr[0]
    keep = [h] + [r for r in lr[1:] if short(r[h.index("Kernel Name")]).startswith("k_")]
    with open(os.path.join(prof, f"{tag}_launches.csv"), "w", newline="") as f:
        csv.writer(f).writerows(keep)
    tot = {}
    for r in keep[1:]:
        k = short(r[h.index("Kernel Name")])
        tot[k] = tot.get(k, 0) + float(r[h.index("Metric Value")])
    s = sum(tot.values())
    print("launch-list share of the step:", {k: round(v / s, 3) for k, v in tot.items()})
for k, v in out.items():
    print(f"{k:14s} {v['duration_us']:8.1f} us  dram {((v['dram_read_bytes'] or 0) + (v['dram_write_bytes'] or 0)) / 1e6:8.1f} MB"
          f"  ipc {v['ipc_active']}  occ {v['achieved_occupancy_pct']}  stalls {v['top_stalls'][:3]}")
