"""bench.py — LOPC hot path on B200: compress + decompress throughput.

One step (default cfg3, 512^3 f32) = one pass of the whole hot path over one
synthetic field: lopc_compress (quantize -> repair to the fixpoint -> chunked
encode with look-back placement) followed by lopc_decompress, input resident
in HBM.  value = raw input GB (all ranks) / (max over ranks of the summed
device time of the K timed steps), in GB/s.  L2 (126 MB) is flushed between
steps by writing a 512 MB buffer outside the timed events.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
  python bench.py --impl reference ...   # the CPU oracle arm (rank 0 only)

Multi-GPU (torchrun): the slab mode — one global field, the
config tiled N times along z (cfg1-4) or the cfg5 turbulence field with 256 z
planes of 2048^2 f64 per rank (N = 8 is cfg5 itself), NCCL halo exchange per
repair round; weak scaling, barrier + max-over-ranks device time.
`--config cfg5` at N = 1 runs one rank's slab (2048 x 2048 x 256 f64).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from synth.fields import CONFIGS, eps_noa, sha256  # noqa: E402

METRIC = "compress/decompress GB/s at 1/2/4/8 B200 (%HBM roofline); ratio; 0 order violations"
WORKLOAD = {
    "cfg1": "cfg1: 2D f32 64x64 sum-of-Gaussians with plateaus/ties, NOA 1e-2",
    "cfg2": "cfg2: 3D f32 100x500x500 Isabel-shaped synthetic field, NOA 1e-3",
    "cfg3": "cfg3: 3D f32 512^3 NYX-shaped log-normal density, NOA 1e-4",
    "cfg4": "cfg4: 2D f32 1800x3600 CESM-ATM-shaped field with near-ties, NOA 1e-3",
    "cfg5": "cfg5: 3D f64 turbulence (Kolmogorov mode sum), 2048x2048 planes, 256 z-planes per GPU "
            "(N=8: the 2048^3 field), NOA 1e-5 of the global range",
}
CFG5_PLANES = 256  # z-planes of 2048^2 per rank
# per-kernel keys -> the kernel that runs them (single-GPU engine 0; the slab
# mode's repair is k_sweep + k_ghost_inject)
KERNEL_NAMES = {"quant_flags": "k_quant_flags", "sweep": "k_tiles", "encode": "k_encode", "place": "k_place",
                "decode_scan": "k_chunk_scan", "decode": "k_decode"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region through
    NVML (a background thread polling every ~2 ms), so that even a short timed
    region gets samples."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = None
        self.err = None

    def _run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.ready.set()
            while not self.stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, r))
                time.sleep(0.002)
        except Exception as e:  # no NVML: reported as unsampled
            self.err = repr(e)
            self.ready.set()

    def __enter__(self):
        self.ready = threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        self.ready.wait(10)
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "error": self.err}
        sm = [v for v, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": getattr(self, "max_mhz", None),
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, 2 ms polling"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def crop_planes(x) -> int:
    """Leading z-planes (3D) / rows (2D) of the bounded oracle sample: about
    2-8 M points, a few seconds of single-thread oracle work."""
    per = int(np.prod(x.shape[1:]))
    return max(1, min(x.shape[0] // 12 if x.ndim == 3 else x.shape[0] // 8, (2 << 20) // per))


def oracle_sample(cfg_name: str, x: np.ndarray, eps: float, budget_s: float):
    """The CPU oracle (single thread) on a bounded crop of the same field:
    leading z-planes (3D) or rows (2D), compress + decompress, repeated until
    ~budget_s.  Returns (GB/s, description)."""
    import oracle

    oracle.build()
    planes = crop_planes(x)
    crop = np.ascontiguousarray(x[:planes])
    allowed = sorted(os.sched_getaffinity(0))
    core = allowed[-1]
    os.sched_setaffinity(0, {core})  # one thread, pinned
    try:
        t0 = time.perf_counter()
        done = 0
        reps = 0
        while True:
            st = oracle.compress(crop, eps)
            oracle.decompress(st)
            done += crop.nbytes
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, set(allowed))
    desc = (f"oracle compress+decompress of the leading {planes} of {x.shape[0]} "
            f"{'z-planes' if x.ndim == 3 else 'rows'} of {cfg_name} ({crop.nbytes / 1e6:.1f} MB, a crop) x{reps}, "
            f"{dt:.1f} s, 1 thread pinned to core {core} of {os.cpu_count()} on {cpu_model()}; "
            f"full-size single-thread timings: tools/oracle_timing.py -> results/")
    return done / dt / 1e9, desc


def omp_sample(cfg_name: str, x: np.ndarray, eps: float, budget_s: float):
    """NEXT f4: the OpenMP CPU baseline (oracle/lopc_omp.c, all host cores) on
    the same bounded crop, compress + decompress (GB/s of raw input), the
    same round trip as cpu_baseline."""
    import oracle

    planes = crop_planes(x)
    crop = np.ascontiguousarray(x[:planes])
    st, _ = oracle.omp_compress(crop, eps)  # warm-up (thread pool, build)
    oracle.omp_decompress(st)
    t0 = time.perf_counter()
    reps = 0
    while True:
        st, sweeps = oracle.omp_compress(crop, eps)
        oracle.omp_decompress(st)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": crop.nbytes * reps / dt / 1e9, "unit": "GB/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle_omp", "metric": "compress + decompress",
            "sample": f"OpenMP compress+decompress of the leading {planes} of {x.shape[0]} planes of {cfg_name} "
                      f"({crop.nbytes / 1e6:.1f} MB, a crop) x{reps}, {sweeps} relaxation sweeps, {cpu_model()}"}


def cfg5_eps(world: int) -> float:
    """a0 for the cfg5 weak-scaling field (256 planes per rank): 1e-5 x its
    range, found block by block on the device (same value on every rank)."""
    from synth import turbulence as turb

    lo, hi = turb.field_range(CFG5_PLANES * world, 2048, 2048)
    return turb.eps_noa_range(lo, hi, turb.CFG5_REL)


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.config == "cfg5":
        # the oracle's sample: the leading planes of the same field, built on
        # the host (the crop is all the reference arm touches); eps of the
        # N-rank field, as the lopc arm uses
        from synth import turbulence as turb

        x = turb.planes_torch(0, 1, 2048, 2048, device="cpu").numpy()
        try:
            eps = cfg5_eps(world)
        except Exception:  # no GPU on this host: the range of the crop
            eps = eps_noa(x, turb.CFG5_REL)
    else:
        cfg = CONFIGS[args.config]
        x = cfg.generate()
        eps = eps_noa(x, cfg.rel)
    times = []
    desc = ""
    per = max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for i in range(args.warmup + args.steps):
        v, desc = oracle_sample(args.config, x, eps, per)
        if i >= args.warmup:
            times.append(v)
    value = statistics.median(times)
    nbytes = x[:crop_planes(x)].nbytes
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": nbytes / (value * 1e9) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if x.dtype == np.float32 else "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD[args.config], "sample": "bounded crop, see cpu_baseline"},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def tiled_config(cfg_name: str, world: int):
    """Weak-scaling workload for N ranks: the config's field tiled N times
    along z (dims[0]), every other copy mirrored so the field stays continuous
    across copies (same value range, so the same NOA eps)."""
    cfg = CONFIGS[cfg_name]
    base = cfg.generate()
    eps = eps_noa(base, cfg.rel)
    shape = (base.shape[0] * world,) + base.shape[1:]
    return base, eps, shape


def slab_values(base: np.ndarray, shape, e0: int, e1: int) -> np.ndarray:
    """Elements [e0, e1) of the tiled field (only the planes they touch are built)."""
    P = int(np.prod(shape[1:]))
    nz = base.shape[0]
    z0, z1 = e0 // P, -(-e1 // P)
    planes = [base[z % nz] if (z // nz) % 2 == 0 else base[nz - 1 - z % nz] for z in range(z0, z1)]
    flat = np.ascontiguousarray(np.stack(planes)).reshape(-1)
    return np.ascontiguousarray(flat[e0 - z0 * P:e1 - z0 * P])


def run_slabs(args, rank, world, local):
    """N > 1: the slab mode — one global field (the config
    tiled N times along z), chunk-aligned ranges, NCCL halo exchange of the
    subbins every repair round, allgathered payload offsets.  Weak scaling:
    every rank owns one config's worth of points."""
    import torch
    import torch.distributed as dist

    import paper_2603_26968_b200 as lopc
    from paper_2603_26968_b200 import dist as ldist

    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lopc.load()
    uid = [lopc.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = lopc.Comm(world, rank, uid[0])
    if args.config == "cfg5":
        from synth import turbulence as turb

        shape = (CFG5_PLANES * world, 2048, 2048)
        dt = torch.float64
        b = lopc.slab_partition(shape, dt, world)
        e0, e1 = b[rank], b[rank + 1]
        P = shape[1] * shape[2]
        assert e0 % P == 0 and e1 % P == 0
        xs = turb.planes_torch(e0 // P, e1 // P, shape[1], shape[2]).reshape(-1)
        mm = torch.stack([-xs.min(), xs.max()])
        dist.all_reduce(mm, op=dist.ReduceOp.MAX)  # a0: the global range
        eps = turb.eps_noa_range(-float(mm[0]), float(mm[1]), turb.CFG5_REL)
        xs_np = None
        k = 8
    else:
        base, eps, shape = tiled_config(args.config, world)
        dt = torch.float32 if base.dtype == np.float32 else torch.float64
        b = lopc.slab_partition(shape, dt, world)
        e0, e1 = b[rank], b[rank + 1]
        xs_np = slab_values(base, shape, e0, e1)
        xs = torch.from_numpy(xs_np).cuda()
        k = xs_np.itemsize
    W = 16384 // k
    n_chunks = -(-int(np.prod(shape)) // W)
    out = torch.empty(lopc.slab_bound(shape, dt, e0, e1), dtype=torch.uint8, device="cuda")
    y = torch.empty(e1 - e0, dtype=dt, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    hdr = {}

    def step():
        loc, po, tot = lopc.compress_slab(comm, xs, shape, eps, e0, e1, out=out)
        if "h" not in hdr:
            hdr["h"] = lopc.write_header(shape, dt, eps, tot)
        lopc.decompress_slab(hdr["h"], loc, e0, e1, dt, out=y)
        return loc, po, tot

    for _ in range(args.warmup):
        loc, po, tot = step()
    torch.cuda.synchronize()
    if xs_np is not None:
        import oracle  # test infrastructure, outside the timed region: per-rank bound check

        y_np = y.cpu().numpy().reshape(1, -1)
        bound_bad = oracle.bound_violations(xs_np.reshape(1, -1), y_np, eps)
        order_bad = None
    else:  # cfg5 slab (1 G points): the device checker (k_check, pinned to the oracle's checkers)
        lsh = ((e1 - e0) // (shape[1] * shape[2]),) + tuple(shape[1:])
        chk = lopc.check(xs.view(lsh), y.view(lsh), eps)
        bound_bad, order_bad = chk["bound_violations"], chk["order_violations"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    comp_ms, dec_ms = [], []
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ev[0].record()
            loc, po, tot = lopc.compress_slab(comm, xs, shape, eps, e0, e1, out=out)
            ev[1].record()
            lopc.decompress_slab(hdr["h"], loc, e0, e1, dt, out=y)
            ev[2].record()
            torch.cuda.synchronize()
            comp_ms.append(ev[0].elapsed_time(ev[1]))
            dec_ms.append(ev[1].elapsed_time(ev[2]))
    dist.barrier()
    torch.cuda.synchronize()
    lopc.compress_slab(comm, xs, shape, eps, e0, e1, out=out)
    st = lopc.last_stats()
    t = torch.tensor([sum(comp_ms) + sum(dec_ms), sum(comp_ms), sum(dec_ms), float(bound_bad),
                      float(order_bad or 0)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, cm, dm, bad, obad = (float(v) for v in t.tolist())
    K = args.steps
    raw_total = int(np.prod(shape)) * k
    value = raw_total * K / (total_ms / 1e3) / 1e9
    # per-kernel breakdown (library events, a separate loop)
    lopc.set_timing(True)
    kern = {kk: [] for kk in ("quant_flags", "sweep", "encode", "place", "decode_scan", "decode")}
    launches = 0
    for _ in range(K):
        loc, po, tot = lopc.compress_slab(comm, xs, shape, eps, e0, e1, out=out)
        sc = lopc.last_stats()
        lopc.decompress_slab(hdr["h"], loc, e0, e1, dt, out=y)
        sd = lopc.last_stats()
        for kk, v in (("quant_flags", sc["ms_quant_repair"]), ("sweep", sc["ms_sweep"]), ("encode", sc["ms_encode"]),
                      ("place", sc["ms_place"]), ("decode_scan", sd["ms_place"]), ("decode", sd["ms_decode"])):
            kern[kk].append(v)
        launches += sc["launches"] + sd["launches"]
    lopc.set_timing(False)
    # e2e: pinned host slab in, local stream out and back, values out
    xh = torch.from_numpy(xs_np).pin_memory() if xs_np is not None else xs.cpu().pin_memory()
    oh = torch.empty(out.numel(), dtype=torch.uint8).pin_memory()
    yh = torch.empty(e1 - e0, dtype=dt).pin_memory()
    e2e = []
    for i in range(max(3, K // 2) + 1):
        flush.fill_(1)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        xd = xh.cuda(non_blocking=True)
        loc, po, tot = lopc.compress_slab(comm, xd, shape, eps, e0, e1, out=out)
        oh[:loc.numel()].copy_(loc)
        ld = oh[:loc.numel()].cuda(non_blocking=True)
        yd = lopc.decompress_slab(hdr["h"], ld, e0, e1, dt)
        yh.copy_(yd)
        torch.cuda.synchronize()
        if i:
            e2e.append((time.perf_counter() - t0) * 1e3)
    te = torch.tensor([statistics.median(e2e), float(loc.numel())], device="cuda", dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te[0])
    sizes = [None] * world
    dist.all_gather_object(sizes, int(loc.numel()))
    if rank == 0:
        peak, peak_src = load_peaks()
        med = {kk: statistics.median(v) for kk, v in kern.items()}
        n_loc = e1 - e0
        F = 2 if len(shape) == 3 else 1
        # slab mode: tile pass 1 (F + 1 B/point) + the planes widened to u32
        # after the repair (1 + 4; later tile passes not counted: a lower
        # bound); the encoder reads x and the u32 subbins
        alg = {"quant_flags": n_loc * (k + F), "sweep": n_loc * (F + 6), "encode": n_loc * (k + 4) + sizes[0],
               "place": 2 * sizes[0], "decode_scan": 16 * (-(-n_loc // W)), "decode": sizes[0] + n_loc * k}
        dom = max(med, key=lambda kk: med[kk])
        achieved = alg[dom] / (med[dom] / 1e3) / 1e9 if med[dom] > 0 else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(f"k_{dom}")
        stream_total = sum(sizes) + 64  # tables are inside the locals
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if k == 4 else "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config] + (
                           ", slab mode" if args.config == "cfg5" else f", tiled x{world} along z (mirrored), slab mode"),
                       "dims": list(shape), "eps": eps, "ranges": b, "l2": "flushed (512 MB write) between steps",
                       "parallelism": f"slabs x{world}: NCCL halo exchange per repair round"},
            "compress_GBps": raw_total * K / (cm / 1e3) / 1e9, "decompress_GBps": raw_total * K / (dm / 1e3) / 1e9,
            "ratio": raw_total / stream_total, "stream_bytes": stream_total, "bound_violations": int(bad),
            "order_violations": None if xs_np is not None else int(obad),
            "order_check": "per-rank slab, device k_check" if xs_np is None else None,
            "repair_rounds": st["inner_iters"],
            "per_kernel_rank0": {kk: {"ms": med[kk], "alg_bytes": alg[kk]} for kk in med},
            "roofline": {"kernel": f"k_{dom}", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src},
            "cpu_baseline": None,
            "e2e": {"value": raw_total / (e2e_ms / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": (e1 - e0) * k + int(loc.numel()),
                    "d2h_bytes_per_step": (e1 - e0) * k + int(loc.numel()),
                    "note": "per rank: pinned slab H2D, compress_slab, local stream D2H + H2D, decompress_slab, D2H"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    comm.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    # cfg3 (512^3 f32): the largest single-GPU config of BASELINE.json (cfg5
    # is the 8-GPU one); its metric names no config, so the bench line is on it
    ap.add_argument("--config", default="cfg3", choices=sorted(WORKLOAD))
    ap.add_argument("--impl", default="lopc", choices=["lopc", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--slab", action="store_true", help="use the slab mode even at N=1 (tests the N>1 path)")
    ap.add_argument("--engine", type=int, default=0, choices=[0, 1, 2],
                    help="repair engine (diagnostic; 0 = tile engine, the default; see lopc.set_repair_engine); "
                         "the per-kernel alg bytes of 'sweep' assume engine 0")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1 or args.slab:
        return run_slabs(args, rank, world, local)

    import torch

    import paper_2603_26968_b200 as lopc

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lopc.load()
    if args.engine:
        lopc.set_repair_engine(args.engine)
    big = args.config == "cfg5"
    if big:  # one rank's slab of cfg5, generated on the device (8.6 GB f64)
        from synth import turbulence as turb

        x = turb.planes_torch(0, CFG5_PLANES, 2048, 2048)
        eps = cfg5_eps(1)
        x_np = None
    else:
        cfg = CONFIGS[args.config]
        x_np = cfg.generate()
        eps = eps_noa(x_np, cfg.rel)
        x = torch.from_numpy(x_np).cuda()
    raw = x.numel() * x.element_size()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    st_buf = torch.empty(lopc.compress_bound(x.shape, x.dtype), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)

    def step():
        st = lopc.compress(x, eps, out=st_buf)
        lopc.decompress(st, out=y)
        return st

    for _ in range(args.warmup):
        st = step()
    torch.cuda.synchronize()
    # correctness of the benchmarked configuration: order / bound / stability
    if big:  # 1 G points: the device checker (k_check == the oracle's checkers, tests/test_gpu_check.py)
        chk = lopc.check(x, y, eps)
        violations, bound_bad = chk["order_violations"], chk["bound_violations"]
    else:
        import oracle  # test infrastructure, outside the timed region

        y_np = y.cpu().numpy()
        violations = oracle.order_violations(x_np, y_np) if rank == 0 else 0
        bound_bad = oracle.bound_violations(x_np, y_np, eps) if rank == 0 else 0
    nbytes_stream = int(st.numel())

    # (1) the timed region: K steps, CUDA events around the C-ABI calls
    comp_ms, dec_ms = [], []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ev[0].record()
            st = lopc.compress(x, eps, out=st_buf)
            ev[1].record()
            lopc.decompress(st, out=y)
            ev[2].record()
            torch.cuda.synchronize()
            comp_ms.append(ev[0].elapsed_time(ev[1]))
            dec_ms.append(ev[1].elapsed_time(ev[2]))
    torch.cuda.synchronize()
    st = lopc.compress(x, eps, out=st_buf)  # launches per step of the timed schedule (timing off)
    launches_timed = lopc.last_stats()["launches"]
    lopc.decompress(st, out=y)
    launches_timed = K_launch = (launches_timed + lopc.last_stats()["launches"]) * args.steps
    # (2) per-kernel breakdown: the same K steps again with the library's own
    # per-launch events on (lopc_set_timing), not part of `value`
    lopc.set_timing(True)
    kern = {k: [] for k in ("quant_flags", "sweep", "encode", "place", "decode_scan", "decode")}
    tiles, launches = [], 0
    for _ in range(args.steps):
        flush.fill_(1)
        st = lopc.compress(x, eps, out=st_buf)
        sc = lopc.last_stats()
        lopc.decompress(st, out=y)
        sd = lopc.last_stats()
        kern["quant_flags"].append(sc["ms_quant_repair"])
        kern["sweep"].append(sc["ms_sweep"])
        kern["encode"].append(sc["ms_encode"])
        kern["place"].append(sc["ms_place"])
        kern["decode_scan"].append(sd["ms_place"])
        kern["decode"].append(sd["ms_decode"])
        launches += sc["launches"] + sd["launches"]
        tiles.append(sc["worklist_points"])
        rep = {k: sc[k] for k in ("sweep_passes", "worklist_points", "inner_iters", "raised", "max_subbin",
                                  "escapes", "n_tiles", "bin_bytes", "sub_bytes")}
        rep["pass_items"] = [v for v in sc["pass_items"][1:] if v]
    torch.cuda.synchronize()
    lopc.set_timing(False)
    total_ms = sum(comp_ms) + sum(dec_ms)
    if dist:
        t = torch.tensor([total_ms, sum(comp_ms), sum(dec_ms)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, cm, dm = (float(v) for v in t.tolist())
    else:
        cm, dm = sum(comp_ms), sum(dec_ms)
    K = args.steps
    value = raw * world * K / (total_ms / 1e3) / 1e9

    # ---- e2e through the C-ABI with HOST (pinned) buffers -------------------
    xh = x.cpu().pin_memory()
    sth = torch.empty(st_buf.numel(), dtype=torch.uint8).pin_memory()
    yh = torch.empty(x.shape, dtype=x.dtype).pin_memory()
    for _ in range(2):
        s2 = lopc.compress(xh, eps, out=sth)
        lopc.decompress(s2, out=yh)
    e2e_ms = []
    for _ in range(max(3, K // 2)):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s2 = lopc.compress(xh, eps, out=sth)
        lopc.decompress(s2, out=yh)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_step = statistics.median(e2e_ms)
    if dist:
        t = torch.tensor([e2e_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())
    e2e_val = raw * world / (e2e_step / 1e3) / 1e9

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----------------------------------
    # algorithmic bytes per launch: x is k bytes/point, the
    # bit-plane flags F = 2 (3D) / 1 (2D) bytes/point, s is u32.
    peak, peak_src = load_peaks()
    n = x.numel()
    k = x.element_size()
    F = 2 if x.dim() == 3 else 1
    med = {kk: statistics.median(v) for kk, v in kern.items()}
    alg = {
        "quant_flags": n * (k + F),                                        # read x, write flags
        # tile engine (k_tiles): pass 1 reads the flags and writes the subbin
        # planes (F + 1 B/point); every later tile visit (1024 points) reads
        # flags + planes and writes planes (F + 2 B/point)
        "sweep": n * (F + 1) + max(0, statistics.median(tiles) - rep["pass_items"][0]) * 1024 * (F + 2),
        # planes mode (tile engine): the bin CTAs read x, the subbin CTAs the
        # subbin planes (1 B/point) and the flags' escape words (1/8 B/point);
        # both write their payloads
        "encode": n * (k + 1) + n // 8 + nbytes_stream,
        "place": 2 * nbytes_stream,                                        # staged payloads -> stream
        "decode_scan": 16 * ((n * k + 16383) // 16384),                   # size table in, offsets out
        "decode": nbytes_stream + n * k,                                   # read stream, write x^
    }
    dom = max(med, key=lambda kk: med[kk])
    kname = KERNEL_NAMES[dom]
    achieved = alg[dom] / (med[dom] / 1e3) / 1e9 if med[dom] > 0 else 0.0
    per_kernel = {kk: {"ms": med[kk], "alg_bytes": alg[kk],
                       "GBps": (alg[kk] / (med[kk] / 1e3) / 1e9) if med[kk] > 0 else None} for kk in med}
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(kname)

    # the bound these kernels actually hit: instruction issue.  Peak = 4
    # schedulers x 1 warp-instruction/clk x 148 SMs x the sampled SM clock
    # (B200_PROFILING.md / blackwell guide unit counts); instructions per
    # launch from the committed ncu capture of the same kernel and config.
    issue = None
    wp = os.path.join(ROOT, "profiles", f"warpinst_{args.config}.json")
    if os.path.exists(wp) and med[dom] > 0:
        wi = json.load(open(wp))["kernels"].get(kname)
        if wi:
            mhz = clk.summary().get("sm_mhz") or 1965.0
            ipk = 4 * 148 * mhz * 1e6
            ach = wi / (med[dom] / 1e3)
            issue = {"kernel": kname, "bound": "issue", "achieved": ach, "peak": ipk,
                     "unit": "warp-instructions/s", "frac": ach / ipk, "warp_instructions": wi,
                     "source": os.path.relpath(wp, ROOT)}

    cpu = cpu_omp = None
    if not args.no_cpu_baseline:
        xs_host = x_np if x_np is not None else x[:1].cpu().numpy()  # cfg5: the leading plane
        v, desc = oracle_sample(args.config, xs_host, eps, args.cpu_budget)
        cpu = {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc}
        cpu_omp = omp_sample(args.config, xs_host, eps, max(2.0, args.cpu_budget / 2))

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if k == 4 else "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config] + (", one rank's slab at N=1" if big else ""),
                   "dims": list(x.shape), "eps": eps,
                   "input_sha256": sha256(x_np) if x_np is not None else "generated on the device (synth/turbulence.py)",
                   "l2": "flushed (512 MB write) between steps" if not big else "inputs (8.6 GB) larger than L2",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   **({"repair_engine": args.engine} if args.engine else {})},
        "compress_GBps": raw * world * K / (cm / 1e3) / 1e9,
        "step_ms": {"compress": [round(v, 4) for v in comp_ms], "decompress": [round(v, 4) for v in dec_ms]},
        "decompress_GBps": raw * world * K / (dm / 1e3) / 1e9,
        "ratio": raw / nbytes_stream, "stream_bytes": nbytes_stream,
        "order_violations": int(violations), "bound_violations": bound_bad,
        "repair": rep,
        "per_kernel": per_kernel,
        "roofline": {"kernel": kname, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": alg[dom], "launch_ms": med[dom]},
        "roofline_issue": issue,
        "cpu_baseline": cpu,
        "cpu_baseline_multicore": cpu_omp,
        "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": raw + nbytes_stream,
                "d2h_bytes_per_step": nbytes_stream + raw,
                "note": "lopc_compress/lopc_decompress on pinned host buffers: staging copies inside the calls, "
                         "decompress pipelined over chunk ranges (H2D / decode / D2H overlap)"},
        "gpu_launches": launches_timed,
        "clocks": clk.summary(),
        "notes": "per_kernel/roofline: the library's per-launch events (lopc_set_timing) in a second loop; "
                 "launches run in stream order in both loops",
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
