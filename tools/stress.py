"""Randomised GPU-vs-oracle stress (not part of the default suite): random
2D/3D shapes (ragged against the 32-point segments and 16 KiB chunks), both
dtypes, every random-field kind, NOA bounds 1e-1..1e-5, escapes sprinkled in
(NaN, +-Inf, out-of-range values), through the plain calls (device I/O), the
host-I/O path, and slab mode (2-4 random-partitioned slabs, tile engine);
every stream must equal the oracle's bytes and every decode the oracle's
values.  Usage: python tools/stress.py [cases] [seed]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import eps_noa, random_field  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
kinds = ["noise", "smooth", "ties", "plateau", "ramp_down", "grid16", "signed_zero_subnormal"]
bad = 0
stats = {"plain": 0, "host": 0, "slab": 0}
for i in range(cases):
    nd = int(rng.integers(2, 4))
    shape = tuple(int(v) for v in (rng.integers(1, 40, 3) if nd == 3 else rng.integers(1, 400, 2)))
    if nd == 3:
        shape = (shape[0], shape[1], int(rng.integers(1, 130)))
    dt = "f32" if rng.random() < 0.6 else "f64"
    kind = kinds[int(rng.integers(len(kinds)))]
    x = random_field(shape, dt, kind, int(rng.integers(1 << 30)))
    rel = 10.0 ** -float(rng.integers(1, 6))
    eps = eps_noa(x, rel)
    if not (eps > 0 and np.isfinite(eps)):
        continue
    if rng.random() < 0.3:  # escapes
        big = 3e38 if dt == "f32" else 1e300
        for _ in range(int(rng.integers(1, 6))):
            x.ravel()[int(rng.integers(x.size))] = [np.nan, np.inf, -np.inf, big, -big][int(rng.integers(5))]
    ref = oracle.compress(x, eps)
    xref = oracle.decompress(ref)
    tdt = torch.float32 if dt == "f32" else torch.float64
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    st = lopc.compress(xt, eps)
    y = lopc.decompress(st)
    ok = st.cpu().numpy().tobytes() == ref and y.cpu().numpy().tobytes() == xref.tobytes()
    stats["plain"] += 1
    if i % 3 == 0:  # host I/O
        sh = lopc.compress(torch.from_numpy(np.ascontiguousarray(x)).pin_memory(), eps)
        yh = lopc.decompress(sh, out=torch.empty(x.shape, dtype=tdt).pin_memory())
        ok = ok and sh.numpy().tobytes() == ref and yh.numpy().tobytes() == xref.tobytes()
        stats["host"] += 1
    if i % 2 == 0:  # slab mode, when the shape allows the ranges
        world = int(rng.integers(2, 5))
        try:
            bounds = lopc.slab_partition(x.shape, tdt, world)
        except Exception:  # noqa: BLE001  (too small for that many ranges)
            bounds = None
        if bounds is not None:
            try:
                ss = lopc.compress_slabs_local(xt, eps, bounds).cpu().numpy().tobytes()
                ok = ok and ss == ref
                stats["slab"] += 1
            except lopc.LopcError as e:  # a middle range shorter than the halo: not a slab layout
                if e.code != -2:
                    raise
    if not ok:
        bad += 1
        print(f"MISMATCH case {i}: shape {shape} {dt} {kind} rel {rel}", flush=True)
torch.cuda.synchronize()
print(f"stress: {cases} cases ({stats}), {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
