"""Tiny compress/decompress round trip (for compute-sanitizer runs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import random_field  # noqa: E402

for dims, dt in [((3, 4), "f32"), ((37, 41), "f32"), ((5, 6, 7), "f64"), ((20, 100, 100), "f32")]:
    x = random_field(dims, dt, "smooth", 1)
    xt = torch.from_numpy(x).cuda()
    st = lopc.compress(xt, 1e-3)
    torch.cuda.synchronize()
    print(dims, dt, "compressed", st.numel(), flush=True)
    y = lopc.decompress(st)
    torch.cuda.synchronize()
    print(dims, dt, "max err", float((y - xt).abs().max()), flush=True)
