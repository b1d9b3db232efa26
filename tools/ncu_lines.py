#!/usr/bin/env python3
"""Aggregate ncu 'cuda,sass' source-page CSV per CUDA source line: stall samples and executed instructions.
usage: ncu -i X.ncu-rep [-k ...] --page source --csv --print-source cuda,sass | python tools/ncu_lines.py [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(sys.stdin))
top = int(sys.argv[1]) if len(sys.argv) > 1 else 30
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
i_line, i_src, i_stall, i_exec = 0, 1, h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg = defaultdict(lambda: [0, 0, ""])
cur = None
for r in rows[hdr + 1:]:
    if len(r) <= i_exec:
        continue
    if r[i_line]:
        cur = r[i_line]
        agg[cur][2] = r[i_src]
    try:
        agg[cur][0] += int(r[i_stall] or 0)
        agg[cur][1] += int(r[i_exec] or 0)
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts} instructions {ti}")
for line, (s, e, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% stall {100*e/ti:5.1f}% inst  L{line}: {src.strip()[:100]}")
