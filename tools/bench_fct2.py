"""Time the FCT2 sketch (NEXT-3) at a BASELINE config's n and d with the paper's FCT2 parameters
(s = r1 = ceil(2 d ln d), t = 2 d^2 -> power of two), C resident in HBM (r1 x n s / t)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import fctgen
import paper_1207_4684_b200 as fct
from oracle import fct2 as F   # parameter reading only

c = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = fctgen.CONFIGS[c]
n = rows or cfg.n
s, t, r1 = F.params(cfg.d)
A = torch.empty((n, cfg.d), dtype=torch.float32, device="cuda")
ch = 1 << 22
for r0 in range(0, n, ch):
    A[r0:r0 + ch] = torch.from_numpy(fctgen.matrix(cfg.kind, cfg.seed, max(cfg.n, n), cfg.d, r0, min(ch, n - r0))).cuda()
nb = -(-n // t)
K = nb * s
# C in HBM: generated on the host in row chunks (seeded Cauchy stream, as fctgen.fct2_inputs)
C = torch.empty((r1, K), dtype=torch.float32, device="cuda")
for r in range(r1):
    C[r] = torch.from_numpy(fctgen.cauchy(cfg.seed, fctgen.ST_FCT2_C, r * K, K)).cuda()
inp = fctgen.fct2_inputs(cfg.seed, t, t, s, 1)    # signs_t, sel (independent of n)
sg, sel = torch.from_numpy(inp.signs_t).cuda(), torch.from_numpy(inp.sel).cuda()
Y = fct.fct2_sketch(A, sg, sel, C, t, s, r1)
for _ in range(3):
    fct.fct2_sketch(A, sg, sel, C, t, s, r1, Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
k = 5
e0.record()
for _ in range(k):
    fct.fct2_sketch(A, sg, sel, C, t, s, r1, Y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / k
byt = n * cfg.d * 4 + r1 * K * 4
print(json.dumps({"op": "fct2_sketch", "config": c, "n": n, "d": cfg.d, "s": s, "t": t, "r1": r1, "K": K, "ms": ms,
                  "rows_per_s": n / (ms * 1e-3), "bytes_A_plus_C": byt, "GBps": byt / (ms * 1e-3) / 1e9,
                  "fma": r1 * K * cfg.d, "TFMA_per_s": r1 * K * cfg.d / (ms * 1e-3) / 1e12}))
