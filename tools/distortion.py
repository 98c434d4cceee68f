"""Empirical l1 distortion of the GPU sketch at a config's full size (the upper side is parity-unpinned
-- its O-constant is unknown -- so it is REPORTED against the constant-free yardstick d sqrt(s) log(r1 d) / 0.1).

Thm FCT1: ||A x||_1 <= ||Pi1 A x||_1 <= kappa ||A x||_1 for all x, w.h.p.  We draw X (d x 1000,
Gaussian), form A X and Y X on the GPU (fp64 measurement matmuls, not the product path) and report the ratios.
Also the conditioning of U = A R^-1 in the paper's kappa-bar-1 sense is not computed (needs d LPs, out of scope).
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import fctgen
import paper_1207_4684_b200 as fct

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nx = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
cfg = fctgen.CONFIGS[c]
inp = fctgen.make_inputs(cfg)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
A = dev(inp.A)
Y = fct.fct_sketch(A, dev(inp.signs), dev(inp.cauchy), dev(inp.hash), cfg.s, cfg.r1).double()
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(cfg.d, nx, dtype=torch.float64, device="cuda", generator=g)
ax = torch.zeros(nx, dtype=torch.float64, device="cuda")
for i in range(0, cfg.n, 1 << 22):
    ax += (A[i:i + (1 << 22)].double() @ X).abs().sum(dim=0)
yx = (Y @ X).abs().sum(dim=0)
r = (yx / ax).cpu().numpy()
yard = cfg.d * math.sqrt(cfg.s) * math.log(cfg.r1 * cfg.d) / 0.1
print(json.dumps({"op": "l1_distortion", "config": c, "n": cfg.n, "d": cfg.d, "s": cfg.s, "r1": cfg.r1, "x_draws": nx,
                  "ratio_min": float(r.min()), "ratio_median": float(np.median(r)), "ratio_max": float(r.max()),
                  "frac_lower_side_holds": float((r >= 1.0).mean()), "yardstick_d_sqrt_s_log_r1d_over_0.1": yard,
                  "max_over_yardstick": float(r.max() / yard)}))
