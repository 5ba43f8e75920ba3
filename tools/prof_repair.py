import sys, torch
sys.path.insert(0, '.')
import paper_2603_26968_b200 as lopc
from synth.fields import CONFIGS, eps_noa
cfg = CONFIGS['cfg2']; x = cfg.generate(); eps = eps_noa(x, cfg.rel)
xt = torch.from_numpy(x).cuda()
for i in range(2):
    st = lopc.compress(xt, eps)
s = lopc.last_stats()
print({k: s[k] for k in ('sweep_passes','worklist_points','inner_iters','raised','max_subbin','n_tiles','pass_items')})
