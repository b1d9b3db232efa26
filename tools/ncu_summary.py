#!/usr/bin/env python3
"""Summarise an ncu report for profiles/: per kernel launch duration, DRAM bytes, SM/tensor/L2 throughput,
occupancy, IPC.  usage: python tools/ncu_summary.py report.ncu-rep out_prefix [pairs_per_launch]
With pairs_per_launch, also writes <dir of out_prefix>/ncu_traffic.json (DRAM bytes per pair per kernel),
which bench.py reads for the roofline "traffic" field."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name-base", "function"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
units = rows[1]
want = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active": "tc_inst_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "launch__registers_per_thread": "registers",
    "sm__ops_path_tensor_src_int8.sum": "tensor_int8_ops",
    "sm__ops_path_tensor_src_int8.sum.per_second": "tensor_int8_ops_per_s",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "mem_tensor_active_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_inst_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_inst_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
}
idx = {k: hdr.index(k) for k in want if k in hdr}
ki = hdr.index("Kernel Name")
per = defaultdict(list)
for r in rows[2:]:
    if len(r) <= ki:
        continue
    d = {}
    for k, i in idx.items():
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if u == "ns":
            v /= 1000.0
        elif u == "us" or u == "usecond":
            pass
        elif u == "ms" or u == "msecond":
            v *= 1000.0
        if u in ("Kbyte", "KB"):
            v *= 1e3
        elif u in ("Mbyte", "MB"):
            v *= 1e6
        elif u in ("Gbyte", "GB"):
            v *= 1e9
        d[want[k]] = v
    per[r[ki]].append(d)
summary = {}
for k, lst in per.items():
    avg = {m: sum(x.get(m, 0.0) for x in lst) / len(lst) for m in set().union(*lst)}
    avg["launches_captured"] = len(lst)
    avg["dram_bytes"] = avg.get("dram_read", 0.0) + avg.get("dram_write", 0.0)
    summary[k] = avg
json.dump(summary, open(out + ".json", "w"), indent=1, sort_keys=True)
with open(out + ".txt", "w") as f:
    for k, v in sorted(summary.items(), key=lambda kv: -kv[1].get("duration", 0)):
        f.write(f"{k:22s} dur {v.get('duration', 0):9.1f} us  dram {v['dram_bytes']/1e6:9.2f} MB  "
                f"sm {v.get('sm_throughput_pct', 0):5.1f}%  tensor {v.get('tensor_pipe_pct', 0):5.1f}%  "
                f"occ {v.get('occupancy_pct', 0):5.1f}%  ipc {v.get('ipc', 0):4.2f}  regs {v.get('registers', 0):.0f}"
                + (f"  int8 {v['tensor_int8_ops']/1e9:.1f} Gop" if v.get("tensor_int8_ops") else "")
                + f"  issue {v.get('issue_active_pct', 0):5.1f}%  fma {v.get('fma_pipe_pct', 0):5.1f}%"
                + f"  alu {v.get('alu_pipe_pct', 0):5.1f}%  l2hit {v.get('l2_hit_pct', 0):5.1f}%"
                + f"  dram {v.get('dram_pct', 0):5.1f}%  inst {v.get('inst_executed', 0)/1e6:.1f}M\n")
print(open(out + ".txt").read())

if len(sys.argv) > 3:
    import os

    pairs = int(sys.argv[3])
    tr = {}
    for k, v in summary.items():
        name = k.split("<")[0].split("(")[0].replace("void ", "").strip()
        tr[name] = {"dram_bytes_per_pair": v["dram_bytes"] / pairs, "pairs_in_capture": pairs,
                    "source": os.path.relpath(out + ".json", os.path.dirname(os.path.dirname(os.path.abspath(out))) + "/..")}
    json.dump(tr, open(os.path.join(os.path.dirname(out), "ncu_traffic.json"), "w"), indent=1, sort_keys=True)
