"""SASS evidence of the hand-written sm_100a paths: per kernel of libumapb200.so, the counts of the
tcgen05 / TMA / TMEM / packed-fp32 instructions (cuobjdump -sass; B200_PROFILING.md mnemonics:
UTCHMMA = tcgen05.mma, UTMALDG = TMA tensor load, UBLKCP = bulk copy, LDTM = tcgen05.ld).
    python tools/sass_counts.py [lib.so] > profiles/sass_<tag>.txt"""
import collections
import os
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "paper_2008_00325_b200", "libumapb200.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "SYNCS", "FADD2", "FMUL2", "FFMA2", "ATOMS", "RED", "MUFU",
       "HMMA"]
print(f"# {os.path.basename(lib)}: sm_100a SASS instruction counts per kernel (static, cuobjdump)")
arch = re.findall(r"arch = (sm_\w+)", txt)
print(f"# arch: {sorted(set(arch))}")
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    if not name.startswith("_ZN8umapb200"):
        continue
    c = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)((?:\.[A-Z0-9_]+)*)", line)
        if m and m.group(1) in OPS:
            c[m.group(1) + (".2CTA" if ".2CTA" in m.group(2) else "")] += 1
    if c:
        dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dn = dn.replace("umapb200::(anonymous namespace)::", "").split("(")[0]
        print(f"{dn:60s} " + " ".join(f"{k}={v}" for k, v in sorted(c.items())))
