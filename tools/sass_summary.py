"""Opcode evidence from the built objects (cuobjdump -sass): per kernel family, counts of the
Blackwell-native instructions (tcgen05 MMA UTC*MMA, TMEM loads LDTM, TMA UTMALDG / UBLKCP,
mbarrier SYNCS.*) and of the legacy tensor path (HMMA, should be 0).
usage: python tools/sass_summary.py [objects...]  (default: paper_2605_19150_b200/build/*.o)"""
import glob
import os
import re
import subprocess
import sys
from collections import Counter, defaultdict

OPS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCOMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "HMMA",
       "BAR.SYNC", "LDS", "STS", "LDG", "STG"]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
objs = sys.argv[1:] or sorted(glob.glob(os.path.join(root, "paper_2605_19150_b200", "build", "*.o")))
fam = defaultdict(Counter)
nk = Counter()
for o in objs:
    txt = subprocess.run(["cuobjdump", "-sass", o], capture_output=True, text=True).stdout
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            dem = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            cur = re.sub(r"<.*", "", dem).replace("void ", "")
            nk[cur] += 1
            continue
        if cur is None:
            continue
        ins = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not ins:
            continue
        op = ins.group(1)
        for k in OPS:
            if op == k or op.startswith(k + "."):
                fam[cur][k] += 1
                break
print(f"{'kernel family':44s} {'inst':>4s} " + " ".join(f"{k:>8s}" for k in OPS))
for k in sorted(fam):
    print(f"{k[:44]:44s} {nk[k]:4d} " + " ".join(f"{fam[k][o]:8d}" for o in OPS))
