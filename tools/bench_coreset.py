"""NEXT-2 measurements on the GPU (not part of bench.py's step).

1. Time l1_coreset_gather + l1_lad_solve at the coreset sizes of the configs (m rows = the sampler's count for
   cfg m, q = cfg d), CUDA events on the current stream, inputs resident.
2. The relative-error-vs-sample-size trend of PAPER.md P:L1612-1614 ("the relative error is proportional to
   1/s") on cfg 2's planted l1 regression (n = 2^20 x 16, last column -b): the full LAD optimum x* is solved on
   the GPU (all n rows), then for each m the whole path (sketch -> condition -> row norms -> sample) and the
   coreset solve give x_hat; rel_err = f(x_hat)/f(x*) - 1 with f the full-data objective.
Writes JSON lines to stdout.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import fctgen
import paper_1207_4684_b200 as fct


def timed(fn, K=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K, out


def full_objective(X, x):
    """sum_i |X_i . [x; 1]| over all rows (fp64; measurement only)."""
    xx = torch.cat([x, torch.ones(1, dtype=torch.float64, device=x.device)])
    f = 0.0
    for i in range(0, X.shape[0], 1 << 22):
        f += (X[i:i + (1 << 22)].double() @ xx).abs().sum().item()
    return f


def solve_times():
    for c in (2, 3, 4, 5):
        cfg = fctgen.CONFIGS[c]
        n = min(cfg.n, 1 << 22)
        X = torch.from_numpy(fctgen.matrix(cfg.kind, cfg.seed, cfg.n, cfg.d, 0, n)).cuda()
        rng = np.random.default_rng(c)
        m = cfg.m
        idx = torch.from_numpy(np.sort(rng.choice(n, m, replace=False)).astype(np.int64)).cuda()
        w = torch.from_numpy(1.0 / rng.uniform(0.05, 1.0, m)).cuda()
        cnt = torch.tensor([m], dtype=torch.int64, device="cuda")
        Z = torch.empty((m, cfg.d), dtype=torch.float64, device="cuda")
        tg, _ = timed(lambda: fct.l1_coreset_gather(X, idx, w, cnt, Z=Z), K=20)
        ts, (x, info) = timed(lambda: fct.l1_lad_solve(Z, cnt), K=3)
        info = info.cpu().numpy()
        print(json.dumps({"op": "coreset_solve", "config": c, "m": m, "q": cfg.d, "gather_ms": tg, "solve_ms": ts,
                          "iterations": int(info[3]), "status": int(info[5]), "rel_gap": float(info[2]),
                          "ms_per_iteration": ts / max(1, info[3])}), flush=True)


def trend(seeds=5):
    cfg = fctgen.CONFIGS[2]
    inp = fctgen.make_inputs(cfg)
    X = torch.from_numpy(inp.A).cuda()
    sg, cd, hs, pi2 = (torch.from_numpy(a).cuda() for a in (inp.signs, inp.cauchy, inp.hash, inp.pi2))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    Zf = fct.l1_coreset_gather(X)
    e0.record()
    xs, info = fct.l1_lad_solve(Zf, None, max_iter=200)
    e1.record()
    torch.cuda.synchronize()
    info = info.cpu().numpy()
    fstar = full_objective(X, xs)
    print(json.dumps({"op": "full_lad", "config": 2, "n": cfg.n, "q": cfg.d, "ms": e0.elapsed_time(e1),
                      "iterations": int(info[3]), "status": int(info[5]), "f_star": fstar}), flush=True)
    for m in (128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536):
        errs, counts = [], []
        for sd in range(seeds):
            P = fct.Pipeline(cfg.n, cfg.d, cfg.s, cfg.r1, cfg.k, m, seed=100 + sd)
            P.run(X, sg, cd, hs, pi2)
            x, inf = fct.l1_coreset_regression(X, P.idx, P.weight, P.count)
            inf = inf.cpu().numpy()
            counts.append(int(P.count.item()))
            errs.append(full_objective(X, x) / fstar - 1.0 if inf[5] == 0 else float("inf"))
        q1, med, q3 = np.percentile(errs, [25, 50, 75])
        print(json.dumps({"op": "coreset_trend", "config": 2, "m": m, "mean_count": float(np.mean(counts)),
                          "rel_err_q1": q1, "rel_err_median": med, "rel_err_q3": q3, "m_x_median": m * med,
                          "seeds": seeds}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "solve"):
        solve_times()
    if what in ("all", "trend"):
        trend()
