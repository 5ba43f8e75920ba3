"""Fixed per-call cost of the C-ABI calls through the binding: wall time of
back-to-back compress / decompress calls on a tiny field (cfg1, 16 KiB) and
the device time of the same calls (CUDA events)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS, eps_noa  # noqa: E402

cfg = CONFIGS["cfg1"]
x = cfg.generate()
eps = eps_noa(x, cfg.rel)
xt = torch.from_numpy(x).cuda()
out = torch.empty(lopc.compress_bound(xt.shape, xt.dtype), dtype=torch.uint8, device="cuda")
y = torch.empty_like(xt)
for _ in range(20):
    st = lopc.compress(xt, eps, out=out)
    lopc.decompress(st, out=y)
torch.cuda.synchronize()
for name, fn in (("compress", lambda: lopc.compress(xt, eps, out=out)), ("decompress", lambda: lopc.decompress(st, out=y))):
    n = 500
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: wall {wall:.1f} us/call, device-event {e0.elapsed_time(e1) / n * 1e3:.1f} us/call")
