"""One warm-up + one profiled compress/decompress of a cfg5 crop (f64,
2048 x 2048 x 16 planes of the turbulence field) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth import turbulence as turb  # noqa: E402

x = turb.planes_torch(0, 16, 2048, 2048)
lo, hi, _ = lopc.value_range(x)
eps = turb.eps_noa_range(lo, hi, 1e-5)
for _ in range(2):
    st = lopc.compress(x, eps)
    y = lopc.decompress(st)
torch.cuda.synchronize()
print(st.numel(), x.numel() * 8 / st.numel())
