#!/bin/bash
# Round evidence for profiles/<round>/ (run on the GPU box from the repo root; outputs in gpurun_out/):
#   bench line, ncu launch list of the bench command, ncu --set full of the top kernels.
# Each ncu pass runs only after the same command has exited 0 without ncu.
set -e
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1
python tools/perf_probe.py --pairs 203 --cfg E > gpurun_out/perf.json
ncu --set full --import-source on --clock-control none \
    -k regex:"k_compat|k_sc2_mma|k_score|k_sc2|k_pgs|k_degree|k_expand|k_hist|k_collect" -c 10 \
    -o gpurun_out/prof_full -f python tools/perf_probe.py --pairs 203 --cfg E > gpurun_out/ncu_full.log 2>&1
