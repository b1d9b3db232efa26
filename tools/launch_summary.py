#!/usr/bin/env python3
"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per kernel launches, mean duration
and share of the library's kernel time.  usage: python tools/launch_summary.py launches.csv "<header line>" > out.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
iu = h.index("Metric Unit") if "Metric Unit" in h else None
agg = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].replace("void ", "").replace("trk::", "").strip()
    name = name[:name.index("(")] if name.startswith("k_") and "(" in name and "<" not in name.split("(")[0] else name
    name = name.split(">(")[0] + ">" if ">(" in name else name
    v = float(r[iv].replace(",", ""))
    u = r[iu] if iu is not None else "ns"
    v = v / 1000.0 if u in ("ns", "nsecond") else v * 1000.0 if u in ("ms", "msecond") else v
    agg[name].append(v)
mine = {k: v for k, v in agg.items() if k.startswith("k_")}
tot = sum(sum(v) for v in mine.values()) or 1.0
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"{'kernel':22s} {'launches':>8s} {'mean_us':>9s}   share_of_our_kernels")
for k, v in sorted(mine.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:22s} {len(v):8d} {sum(v)/len(v):9.1f}   {100*sum(v)/tot:5.1f}%")
others = {k: v for k, v in agg.items() if not k.startswith("k_")}
if others:
    print("other kernels (torch / flush):", ", ".join(f"{k} x{len(v)}" for k, v in sorted(others.items())))
