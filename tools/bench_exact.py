"""Time l1_rownorm_exact (NEXT-1) at a config's full size: CUDA events on the current stream, inputs resident."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import fctgen
import paper_1207_4684_b200 as fct

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = fctgen.CONFIGS[c]
A = fctgen.matrix(cfg.kind, cfg.seed, cfg.n, cfg.d, 0, cfg.n)
rng = np.random.default_rng(0)
Rinv = np.triu(rng.standard_normal((cfg.d, cfg.d))) / np.sqrt(cfg.d) + np.eye(cfg.d)
Ad, Rd = torch.from_numpy(A).cuda(), torch.from_numpy(Rinv).cuda()
lam, tot = fct.l1_rownorm_exact(Ad, Rd)
for _ in range(3):
    fct.l1_rownorm_exact(Ad, Rd, lam, tot)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K):
    fct.l1_rownorm_exact(Ad, Rd, lam, tot)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
byt = cfg.n * (4 * cfg.d + 4)
print(json.dumps({"op": "l1_rownorm_exact", "config": c, "n": cfg.n, "d": cfg.d, "ms": ms,
                  "rows_per_s": cfg.n / (ms * 1e-3), "algorithmic_GBps": byt / (ms * 1e-3) / 1e9}))
