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
