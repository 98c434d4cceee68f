"""K1 sweep: fct_sketch time on a cfg-shaped problem for scatter modes and L2-offload fractions.
Inputs are generated on the device (timing only; parity lives in tests/).  CUDA events on the launching
stream, median of K launches.  Usage: python tools/bench_sketch.py CFG [ROWS] [modes] [fracs]"""
import json
import os
import statistics
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)

CFG = {3: (1 << 24, 32, 1024, 1024), 4: (1 << 26, 64, 1024, 4096), 5: (1 << 25, 100, 2048, 8192)}


def child(cfg, rows, mode, frac, K=8):
    import torch
    import paper_1207_4684_b200 as fct
    from paper_1207_4684_b200 import _lib
    if os.environ.get("FCT_LIB"):
        _lib._lib = _lib.load(os.environ["FCT_LIB"])   # A/B against another build of the library
    _lib.load()
    n, d, s, r1 = CFG[cfg]
    n = rows or n
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((n, d), device="cuda", generator=g)
    sg = (torch.randint(0, 2, (n,), device="cuda", generator=g, dtype=torch.int8) * 2 - 1).to(torch.int8)
    c = torch.empty(2 * n, device="cuda").cauchy_(generator=g)
    h = torch.randint(0, r1, (2 * n,), device="cuda", generator=g, dtype=torch.int32)
    for _ in range(2):
        Y = fct.fct_sketch(A, sg, c, h, s, r1)
    ts = []
    for _ in range(K):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        Y = fct.fct_sketch(A, sg, c, h, s, r1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    alg = n * (4 * d + 1 + 8 + 8) + 4 * r1 * d
    print(json.dumps({"lib": os.environ.get("FCT_LIB", "libfct.so"), "cfg": cfg, "n": n, "mode": mode, "l2_frac": frac, "ms": ms,
                      "GBps_alg": alg / ms / 1e6, "frac_copy_peak": alg / ms / 1e6 / 6540.8}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], float(sys.argv[5]))
        sys.exit(0)
    cfg = int(sys.argv[1])
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["cas", "exch"]
    fracs = [float(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0.0, 0.25, 0.5]
    for m in modes:
        for f in fracs:
            env = dict(os.environ, FCT_SKETCH_SCATTER=m, FCT_SKETCH_L2=str(f))
            subprocess.run([sys.executable, __file__, "--child", str(cfg), str(rows), m, str(f)], env=env)
