"""Per-phase SM-cycle breakdown of the codec kernels (lopc_set_timing(2))."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2603_26968_b200 as lopc  # noqa: E402
from synth.fields import CONFIGS, eps_noa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[name]
x = cfg.generate()
eps = eps_noa(x, cfg.rel)
xt = torch.from_numpy(x).cuda()
st = lopc.compress(xt, eps)
lopc.decompress(st)
lopc.set_timing(2)
st = lopc.compress(xt, eps)
sc = lopc.last_stats()
y = lopc.decompress(st)
sd = lopc.last_stats()
enc = ["planes gather", "load+quantize", "a4 check", "BIT (both CTAs)", "bins RZE_1", "subs RZE_k", "subs RZE_1", "staging write"]
dec = {9: "bins load+RZE^-1", 10: "subs load+RZE^-1 x2", 11: "BIT^-1 (both CTAs)", 12: "NB^-1+scan"}
C = sc["n_chunks"]
print(f"{name}: chunks {C}; cycles per chunk (per CTA)")
for i, n in enumerate(enc):
    print(f"  enc {n:22s} {sc['phase_cycles'][i] / C:10.0f}")
for i, n in dec.items():
    print(f"  dec {n:22s} {sd['phase_cycles'][i] / C:10.0f}")
pc = sc["phase_cycles"]
if pc[8]:
    print(f"  k_tiles seeded visits {pc[8]}, with a change {pc[9]} ({100 * pc[9] / pc[8]:.1f}%), "
          f"levels run {pc[10] / pc[8]:.2f} per visit, levels below the first change {pc[11] / pc[8]:.2f} per visit")
print("  sweep pass end times (us):", [round(v, 1) for v in sc["pass_us"] if v], "items", sc["pass_items"][:10])
print(f"  sweep dense pass {sc['phase_cycles'][14] / 1e3:.1f} us, sparse passes {sc['phase_cycles'][15] / 1e3:.1f} us")
print({k: (sc[k], sd[k]) for k in ("ms_quant_repair", "ms_sweep", "ms_encode", "ms_place", "ms_decode")})
