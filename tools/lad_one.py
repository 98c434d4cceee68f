"""One l1_lad_solve at a config's coreset size (for ncu captures of lad_ipm_kernel)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import fctgen
import paper_1207_4684_b200 as fct

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = fctgen.CONFIGS[c]
n = min(cfg.n, 1 << 22)
X = torch.from_numpy(fctgen.matrix(cfg.kind, cfg.seed, cfg.n, cfg.d, 0, n)).cuda()
rng = np.random.default_rng(c)
idx = torch.from_numpy(np.sort(rng.choice(n, cfg.m, replace=False)).astype(np.int64)).cuda()
w = torch.from_numpy(1.0 / rng.uniform(0.05, 1.0, cfg.m)).cuda()
Z = fct.l1_coreset_gather(X, idx, w)
x, info = fct.l1_lad_solve(Z)
torch.cuda.synchronize()
print(info.cpu().numpy())
