"""Time l1_sample_multinomial (NEXT-4) at a config's n and m: CUDA events on the current stream, p resident."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import fctgen
import paper_1207_4684_b200 as fct

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = fctgen.CONFIGS[c]
g = torch.Generator(device="cuda").manual_seed(0)
p = torch.rand(cfg.n, device="cuda", generator=g, dtype=torch.float32) ** 4
p /= p.double().sum().float()
for _ in range(3):
    fct.l1_sample_multinomial(p, cfg.m, seed=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20
e0.record()
for _ in range(K):
    fct.l1_sample_multinomial(p, cfg.m, seed=1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
byt = cfg.n * 4 * 2 + cfg.n * 8 * 2 + cfg.m * 16   # p read twice (max, weights), uint64 CDF written + read, outputs
print(json.dumps({"op": "l1_sample_multinomial", "config": c, "n": cfg.n, "m": cfg.m, "ms": ms,
                  "rows_per_s": cfg.n / (ms * 1e-3), "approx_bytes": byt, "GBps": byt / (ms * 1e-3) / 1e9}))
