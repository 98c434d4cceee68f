"""Small end-to-end runs of every hot-path kernel for compute-sanitizer (memcheck / racecheck / synccheck):
the v5 sketch on the cfg-2/3/4 shapes (s = 256 / 1024), the v1 and generic sketches, K5, K2, NEXT-1, the fused
probs+sample, FCT2, multinomial sampling and the coreset solve, on a few thousand rows each."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import fctgen  # noqa: E402
import paper_1207_4684_b200 as fct  # noqa: E402

fct.load()
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
for c, n in ((2, 3 * 256 + 17), (3, 2 * 1024 + 5), (4, 2 * 1024 + 3)):
    cfg = fctgen.CONFIGS[c]
    inp = fctgen.make_inputs(cfg, n=n)
    A = dev(inp.A)
    Y = fct.fct_sketch(A, dev(inp.signs), dev(inp.cauchy), dev(inp.hash), cfg.s, cfg.r1)
    R, Rinv, info = fct.fct_condition(Y, check=False)
    lam, tot = fct.l1_rownorm(A, Rinv, dev(inp.pi2))
    lx, _ = fct.l1_rownorm_exact(A, Rinv)
    p, idx, w, cnt = fct.l1_probs_sample(lam, tot, cfg.m, cfg.seed)
    torch.cuda.synchronize()
    print(f"cfg {c}: n {n} info {int(info.item())} count {int(cnt.item())}", flush=True)
cfg = fctgen.CONFIGS[1]
inp = fctgen.make_inputs(cfg, n=4000)
Y = fct.fct_sketch(dev(inp.A), dev(inp.signs), dev(inp.cauchy), dev(inp.hash), cfg.s, cfg.r1)
im, wm, T = fct.l1_sample_multinomial(dev(np.abs(inp.A[:, 0])), 64, seed=3)
torch.cuda.synchronize()
print("cfg 1 (v1 / generic sketch, multinomial) ok", flush=True)
