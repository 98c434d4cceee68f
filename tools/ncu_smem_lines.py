"""Shared-memory wavefronts per CUDA source line (ncu source page, cuda+sass view).
usage: python tools/ncu_smem_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, fname, out = None, "?", []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        h = r
    elif h and len(r) == len(h) and r[0].isdigit():
        g = lambda c: int(float(r[h.index(c)] or 0)) if r[h.index(c)] not in ("-", "") else 0
        w = g("L1 Wavefronts Shared")
        if w:
            out.append((w, g("L1 Wavefronts Shared Excessive"), g("L1 Wavefronts Shared Ideal"), fname, r[0], r[1].strip()[:80]))
tot = sum(o[0] for o in out) or 1
print(f"total shared wavefronts {tot:.4e}, excessive {sum(o[1] for o in out) / tot * 100:.1f} %")
for w, ex, ide, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{w / tot * 100:5.1f}%  {w:.3e} wf  excess {ex / w * 100:4.0f}%  {f}:{ln}  {src}")
