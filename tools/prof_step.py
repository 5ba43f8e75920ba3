"""One warm-up + one profiled compress/decompress step of a config (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS, eps_noa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if name == "cfg5":  # a 32-plane crop of one rank's cfg5 slab (f64, generated on the device), cfg5's eps
    from synth import turbulence as turb

    xt = turb.planes_torch(768, 800, 2048, 2048)
    lo, hi = turb.field_range(*turb.CFG5_DIMS)
    eps = turb.eps_noa_range(lo, hi, turb.CFG5_REL)
else:
    cfg = CONFIGS[name]
    x = cfg.generate()
    eps = eps_noa(x, cfg.rel)
    xt = torch.from_numpy(x).cuda()
for _ in range(2):
    st = lopc.compress(xt, eps)
    s = lopc.last_stats()
    y = lopc.decompress(st)
torch.cuda.synchronize()
print({k: s[k] for k in ("sweep_passes", "worklist_points", "inner_iters", "raised", "max_subbin", "pass_items")})
