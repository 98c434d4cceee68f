"""Instruction mix of one kernel from an ncu report: warp-instructions and stall samples per opcode.
usage: python tools/ncu_ops.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
si, ei, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
agg = defaultdict(lambda: [0, 0])
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    t = r[src].split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op = op.split(".")[0]
    agg[op][0] += int(r[ei] or 0)
    agg[op][1] += int(r[si] or 0)
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"warp-instructions {ti:.4g}, stall samples {ts}")
for op, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{op:10s} inst {i:11.4g} ({100*i/ti:5.1f}%)  stall {100*s/ts:5.1f}%")
