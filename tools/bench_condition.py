"""K5 timing: fct_condition on a cfg-shaped Y (r1 x d), CUDA events on the launching stream, median of 50."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1207_4684_b200 as fct  # noqa: E402

fct.load()
out = []
for r1, d in [(64, 8), (256, 16), (1024, 32), (4096, 64), (8192, 100), (8192, 128)]:
    Y = torch.from_numpy(np.random.default_rng(1).standard_normal((r1, d)).astype(np.float32)).cuda()
    for _ in range(5):
        fct.fct_condition(Y, check=False)
    ts = []
    for _ in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)   # keep the GPU busy so the host enqueues ahead: device time only
        e0.record()
        _, _, info = fct.fct_condition(Y, check=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    out.append({"r1": r1, "d": d, "us_median": statistics.median(ts), "us_min": min(ts), "info": int(info.item())})
    if os.environ.get("FCT_COND_TIMING"):
        # phase timestamps written by CTA 0 (globaltimer, ns) at the start of the condition workspace's tail
        from paper_1207_4684_b200 import api
        ws = api.workspace(0, "condition")
        nb = api._lib_().fct_condition_workspace_bytes(r1, d)
        ts_raw = ws.view(torch.uint8)[nb - 512:nb].view(torch.int64).cpu().numpy()
        out[-1]["phase_us"] = [round((int(b) - int(a_)) / 1e3, 2) for a_, b in zip(ts_raw[:56], ts_raw[1:56]) if b > a_]
        if ts_raw[61] > 0:
            out[-1]["inverse_cycles_per_step"] = round(int(ts_raw[60]) / int(ts_raw[61]), 1)
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps(out[-1]), flush=True)
