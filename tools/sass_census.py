"""SASS census of libfct.so: per kernel, the instructions that prove the Blackwell-native paths (tcgen05 MMA
UTC*MMA, TMEM LDTM/STTM, TMA UTMALDG / UBLKCP, mbarrier SYNCS.*) and the scatter / reduction primitives
(ATOMS.EXCH / CAS, REDG).  usage: python tools/sass_census.py [libfct.so] > profiles/r02_sass_census.txt"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1207_4684_b200/libfct.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
GROUPS = OrderedDict([
    ("UTCMMA", r"^UTC\w*MMA"), ("LDTM", r"^LDTM"), ("STTM", r"^STTM"), ("UTMALDG", r"^UTMALDG"),
    ("UBLKCP", r"^UBLKCP"), ("SYNCS(mbar)", r"^SYNCS"), ("ATOMS.EXCH", r"^ATOMS\.EXCH"), ("ATOMS.CAS", r"^ATOMS\.CAS"),
    ("REDG", r"^REDG"), ("DFMA", r"^DFMA"), ("F2F.F64.F32", r"^F2F\.F64\.F32"), ("FADD2/FFMA2", r"^F(ADD|FMA|MUL)2"),
    ("total", r".")])
kernels, cur = OrderedDict(), None
for ln in txt.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        kernels[cur] = Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
    if cur and m:
        op = m.group(1)
        for g, pat in GROUPS.items():
            if re.match(pat, op):
                kernels[cur][g] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(anonymous namespace\)::", "", d)
    return re.sub(r"\(.*\)$", "", d)[:70]


cols = list(GROUPS)
print("static SASS instruction counts per kernel (cuobjdump -sass " + lib + ")")
print(f"{'kernel':70s} " + " ".join(f"{c:>11s}" for c in cols))
for k, cnt in kernels.items():
    print(f"{short(k):70s} " + " ".join(f"{cnt[c]:11d}" for c in cols))
