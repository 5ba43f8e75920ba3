"""Round trips for compute-sanitizer (memcheck / racecheck / synccheck): the
tile engine and the u32 engine, device and host I/O, cfg1, a cfg4 crop and a
cfg2 crop, plus a cfg3-shaped crop; each checked against the oracle so a
sanitizer run also proves the results.  Small sizes: the tools slow kernels
down by 10-100x."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS, eps_noa  # noqa: E402

cases = [("cfg1", None), ("cfg4", (180, 360)), ("cfg2", (12, 100, 100)), ("cfg3", (24, 64, 64))]
for engine in (0, 2):
    lopc.set_repair_engine(engine)
    for name, small in cases:
        cfg = CONFIGS[name]
        x = cfg.generate(small)
        eps = eps_noa(x, cfg.rel)
        ref = oracle.compress(x, eps)
        xt = torch.from_numpy(x).cuda()
        st = lopc.compress(xt, eps)  # device I/O
        y = lopc.decompress(st)
        torch.cuda.synchronize()
        ok_dev = st.cpu().numpy().tobytes() == ref and y.cpu().numpy().tobytes() == oracle.decompress(ref).tobytes()
        sh = lopc.compress(torch.from_numpy(x).pin_memory(), eps)  # host I/O (staged, pipelined decompress)
        yh = lopc.decompress(sh, out=torch.empty(x.shape, dtype=xt.dtype).pin_memory())
        ok_host = sh.numpy().tobytes() == ref and yh.numpy().tobytes() == oracle.decompress(ref).tobytes()
        print(f"engine {engine} {name} {x.shape}: device {'ok' if ok_dev else 'MISMATCH'}, "
              f"host {'ok' if ok_host else 'MISMATCH'}", flush=True)
lopc.set_repair_engine(0)

# slab mode (3 slabs of a cfg2 crop, halo rounds through device copies) on both engines
for engine in (0, 2):
    lopc.set_repair_engine(engine)
    x = CONFIGS["cfg2"].generate((24, 100, 100))
    eps = eps_noa(x, CONFIGS["cfg2"].rel)
    bounds = lopc.slab_partition(x.shape, torch.float32, 3)
    st = lopc.compress_slabs_local(torch.from_numpy(x).cuda(), eps, bounds)
    torch.cuda.synchronize()
    print(f"slab engine {engine}: {'ok' if st.cpu().numpy().tobytes() == oracle.compress(x, eps) else 'MISMATCH'}",
          flush=True)
lopc.set_repair_engine(0)

# corrupt streams: the decoder reads payloads in place (global memory), every
# read bounded by the payload length -- under memcheck no access may leave
# the stream's allocation, whatever the corruption (run with
# PYTORCH_NO_CUDA_MEMORY_CACHING=1 so each tensor is its own allocation)
rng = np.random.default_rng(7)
for name, small, dt in (("cfg2", (8, 100, 100), np.float32), ("cfg4", (90, 360), np.float64)):
    x = CONFIGS[name].generate(small).astype(dt)
    ref = oracle.compress(x, eps_noa(x, CONFIGS[name].rel))
    n_ok = n_err = 0
    for _ in range(40):
        b = bytearray(ref)
        for _ in range(int(rng.integers(1, 5))):
            pos = int(rng.integers(64, len(b)))
            b[pos] ^= int(rng.integers(1, 256))
        try:
            lopc.decompress(torch.from_numpy(np.frombuffer(bytes(b), np.uint8).copy()).cuda())
            torch.cuda.synchronize()
            n_ok += 1
        except lopc.LopcError:
            n_err += 1
    print(f"corrupt {name} {dt.__name__}: {n_ok} decoded, {n_err} rejected", flush=True)
