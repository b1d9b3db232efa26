#!/usr/bin/env python3
"""SASS mnemonics per kernel of libturboreg.so (cuobjdump -sass; sm_100a): the evidence that the dense SC^2
block runs on tcgen05 (UTC*MMA, LDTM/STTM) with TMA (UTMALDG), scoring on the bulk-copy engine (UBLKCP),
the FP-heavy loops on packed f32x2 (FFMA2/FADD2/FMUL2).  usage: python tools/sass_evidence.py > out.txt"""
import os
import re
import subprocess
import sys
from collections import Counter, OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2507_01439_b200", "lib", "libturboreg.so")
WATCH = ("UTCIMMA", "UTCOMMA", "UTCQMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP",
         "UBLKPF", "FFMA2", "FADD2", "FMUL2", "LDGSTS", "HMMA", "SYNCS")
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
per = OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        op = m.group(1)
        for w in WATCH:
            if op == w or op.startswith(w):
                per[cur][w] += 1
print(f"SASS mnemonics per kernel in {os.path.relpath(LIB, ROOT)} (cuobjdump -sass; sm_100a)")
print("UTC*MMA = tcgen05.mma (UTCIMMA kind::i8, UTCOMMA kind::mxf4 block-scaled), LDTM/STTM = tcgen05.ld/st,")
print("UTMALDG = TMA tensor load, UBLKCP = bulk async copy, UBLKPF = bulk L2 prefetch, UTCBAR = tcgen05.commit,")
print("SYNCS = mbarrier ops, FFMA2/FADD2/FMUL2 = packed f32x2 FP ops, LDGSTS = cp.async.")
hmma = sum(c["HMMA"] for c in per.values())
print(f"HMMA (legacy mma.sync) instructions in the library: {hmma}\n")
for k, c in per.items():
    if c:
        print(k)
        print("    " + ", ".join(f"{w} x{c[w]}" for w in WATCH if c[w]))
