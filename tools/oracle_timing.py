"""SURVEY §8(d.7) oracle timing protocol, run on the GPU box's host.

One thread pinned to one core (os.sched_setaffinity): the single-thread
oracle's ref_compress / ref_decompress and the paper's serial Alg. 1/2
(ref_alg12_serial: bins + flags + the worklist repair, the "Ser" column of
Tables IV/V) on the FULL cfg1, cfg2 and cfg4 (median of 3) and
on cfg3 (one run; 6 min) when --cfg3; crops only for cfg5 (labelled).  The
OpenMP baseline (all cores: compress and decompress) beside it.  Writes one
JSON record per config to stdout."""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth.fields import CONFIGS, eps_noa, sha256  # noqa: E402


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return "unknown"


def timed(fn, reps):
    ts, out = [], None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts), ts, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["cfg1", "cfg4", "cfg2"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--core", type=int, default=None)
    args = ap.parse_args()
    oracle.build()
    oracle.build_omp()
    allowed = sorted(os.sched_getaffinity(0))
    core = args.core if args.core is not None else allowed[-1]
    host = {"cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(), "affinity_cores": len(allowed)}
    for name in args.configs:
        cfg = CONFIGS[name]
        x = cfg.generate()
        eps = eps_noa(x, cfg.rel)
        reps = 1 if name == "cfg3" else args.reps
        os.sched_setaffinity(0, {core})
        try:
            tc, tcs, st = timed(lambda: oracle.compress(x, eps), reps)
            td, tds, _ = timed(lambda: oracle.decompress(st), reps)
            ta, tas, (_, stats) = timed(lambda: oracle.subbins(x, eps, "alg12"), reps)
        finally:
            os.sched_setaffinity(0, set(allowed))
        tmc, _, (st2, sweeps) = timed(lambda: oracle.omp_compress(x, eps), reps)
        tmd, _, _ = timed(lambda: oracle.omp_decompress(st2), reps)
        assert st2 == st
        gb = x.nbytes / 1e9
        rec = {"config": name, "dims": list(x.shape), "input_sha256": sha256(x), "eps": eps, "host": host,
               "single_thread": {"core": core, "runs": reps,
                                 "compress_s": tc, "compress_runs": tcs, "compress_GBps": gb / tc,
                                 "decompress_s": td, "decompress_runs": tds, "decompress_GBps": gb / td,
                                 "round_trip_GBps": gb / (tc + td),
                                 "alg12_serial_s": ta, "alg12_runs": tas, "alg12_stats": stats},
               "openmp": {"threads": len(allowed), "compress_s": tmc, "decompress_s": tmd,
                          "round_trip_GBps": gb / (tmc + tmd), "relaxation_sweeps": sweeps}}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
