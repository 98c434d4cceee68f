"""Per-CUDA-source-line warp-instructions and stall samples for one kernel (needs -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: [0, 0, ""])
reasons = defaultdict(lambda: defaultdict(int))
fname = "?"
h = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        si = h.index("Warp Stall Sampling (All Samples)")
        ei = h.index("Instructions Executed")
        st_cols = [(j, c) for j, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if h is None or len(r) != len(h) or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    try:
        agg[key][0] += int(r[ei] or 0)
        agg[key][1] += int(r[si] or 0)
    except ValueError:
        continue
    for j, c in st_cols:
        try:
            reasons[key][c[6:]] += int(r[j] or 0)
        except ValueError:
            pass
    if not agg[key][2]:
        agg[key][2] = r[1].strip()[:90]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp-instructions {ti:.4g}, stall samples {ts}")
for (f, ln), (i, s, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    rs = sorted(reasons[(f, ln)].items(), key=lambda x: -x[1])[:3]
    rtxt = " ".join(f"{k}:{100*v/max(s,1):.0f}" for k, v in rs if v)
    print(f"{100*s/ts:5.1f}%s {100*i/ti:5.1f}%i {f}:{ln:<5d} {t[:60]:60s} [{rtxt}]")
