"""NEXT f3: error-bound sweep on the synthetic suite (the paper's Fig. 3/4
axes): for each config and NOA bound 1e0..1e-6, GPU compress /
decompress time (CUDA events, median of 5 after 2 warm-ups), ratio, bin vs
subbin bytes, repair passes, max error / PSNR / order and bound violations
from k_check.  Also the repair-engine ablation (NEXT f2): tile engine vs the
paper's point worklist on the same bytes.  Writes results/eb_sweep.json."""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS  # noqa: E402

RELS = [1e0, 1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6]


def timed(fn, reps=5, warm=2):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(warm):
        r = fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        ev[0].record()
        r = fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts), r


def main():
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg3"]
    out = {"sweep": [], "engine_ablation": []}
    for name in names:
        cfg = CONFIGS[name]
        x_np = cfg.generate()
        x = torch.from_numpy(x_np).cuda()
        raw = x_np.nbytes
        lo, hi, _ = lopc.value_range(x)
        for rel in RELS:
            eps = lopc.noa_eps(lo, hi, x_np.size, rel) if hasattr(lopc, "noa_eps") else rel * (hi - lo)
            buf = torch.empty(lopc.compress_bound(x.shape, x.dtype), dtype=torch.uint8, device="cuda")
            tc, st = timed(lambda: lopc.compress(x, eps, out=buf))
            s = lopc.last_stats()
            y = torch.empty_like(x)
            td, _ = timed(lambda: lopc.decompress(st, out=y))
            chk = lopc.check(x, y, eps)
            cp = lopc.critical_points(x, y)
            row = {"config": name, "rel": rel, "eps": eps, "compress_ms": tc, "decompress_ms": td,
                   "compress_GBps": raw / tc / 1e6, "decompress_GBps": raw / td / 1e6,
                   "ratio": raw / st.numel(), "bin_bytes": s["bin_bytes"], "sub_bytes": s["sub_bytes"],
                   "sweep_passes": s["sweep_passes"], "worklist_points": s["worklist_points"],
                   "max_subbin": s["max_subbin"], "escapes": s["escapes"],
                   "max_abs_err_over_eps": chk["max_abs_err"] / eps, "psnr_db": chk["psnr_db"],
                   "order_violations": chk["order_violations"], "bound_violations": chk["bound_violations"],
                   "critical_points": cp["critical_x"], "fp_fn_ft": [cp["false_positives"], cp["false_negatives"],
                                                                     cp["false_types"]],
                   "pair_mismatches": cp["pair_mismatches"]}
            out["sweep"].append(row)
            print(json.dumps(row), flush=True)
            if rel in (1e-2, 1e-3, 1e-4) and name in ("cfg2", "cfg4"):
                lopc.set_timing(True)
                res = {}
                for eng in (0, 1):
                    lopc.set_repair_engine(eng)
                    ms = []
                    for _ in range(5):
                        st2 = lopc.compress(x, eps, out=buf)
                        ss = lopc.last_stats()
                        ms.append(ss["ms_sweep"] + ss["ms_quant_repair"])
                    res[eng] = (statistics.median(ms), ss["sweep_passes"], ss["worklist_points"],
                                st2.cpu().numpy().tobytes() == st.cpu().numpy().tobytes())
                lopc.set_repair_engine(0)
                lopc.set_timing(False)
                ab = {"config": name, "rel": rel,
                      "tile_engine": {"repair_ms": res[0][0], "passes": res[0][1], "worklist_points": res[0][2]},
                      "paper_worklist_engine": {"repair_ms": res[1][0], "passes": res[1][1],
                                                "worklist_points": res[1][2]},
                      "same_bytes": bool(res[0][3] and res[1][3])}
                out["engine_ablation"].append(ab)
                print(json.dumps(ab), flush=True)
        del x
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "results"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "results", "eb_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
