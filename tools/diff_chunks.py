"""Debug: compare the GPU stream of a config with the oracle's chunk by chunk."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS, eps_noa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = CONFIGS[name]
x = cfg.generate()
eps = eps_noa(x, cfg.rel)
ref = oracle
g = lopc.compress(torch.from_numpy(x).cuda(), eps).cpu().numpy().tobytes()
r = ref.compress(x, eps)
print("len", len(g), len(r))
sg, sr = ref.chunk_sizes(g), ref.chunk_sizes(r)
og = 64 + 8 * len(sg) + np.concatenate([[0], np.cumsum(sg.sum(axis=1))])
orr = 64 + 8 * len(sr) + np.concatenate([[0], np.cumsum(sr.sum(axis=1))])
bad = 0
for c in range(len(sr)):
    for k in range(2):
        a0 = int(og[c] + (sg[c, 0] if k else 0))
        b0 = int(orr[c] + (sr[c, 0] if k else 0))
        pa, pb = g[a0:a0 + int(sg[c, k])], r[b0:b0 + int(sr[c, k])]
        if pa != pb:
            d = next((i for i in range(min(len(pa), len(pb))) if pa[i] != pb[i]), None)
            print(f"chunk {c} {'subs' if k else 'bins'} size gpu {sg[c, k]} ref {sr[c, k]} first diff {d}")
            bad += 1
            if bad > 12:
                sys.exit(0)
print("bad", bad)
