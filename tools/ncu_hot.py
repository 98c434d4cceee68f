"""Summarise an ncu report's source page: top CUDA lines / SASS instructions by warp-stall samples.
usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [cuda|sass] [top]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
mode = sys.argv[3] if len(sys.argv) > 3 else "cuda"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", mode, "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] in ("Address", "Line", "#") and len(r) > 3)
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
src = h.index("Source")
data = []
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    try:
        data.append((int(r[si] or 0), int(r[ei] or 0), r[0], r[src].strip()[:110]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"total samples {tot}, warp-instructions {toti}")
for s, e, a, t in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{100*s/tot:5.1f}% {100*e/toti:5.1f}%i {a:>6} {t}")
