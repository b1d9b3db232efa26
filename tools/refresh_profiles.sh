#!/bin/bash
# Round evidence for profiles/<round>/ (run on the GPU box from the repo root; outputs in gpurun_out/<round>/).
# One ncu pass per gpurun call:
#   tools/refresh_profiles.sh r02 ll     bench line + ncu launch list of the bench command
#   tools/refresh_profiles.sh r02 full   ncu --set full of every kernel >= ~1 % of the step
# Each ncu pass runs only after the same command has exited 0 without ncu.
set -e
R=${1:-r02}
MODE=${2:-ll}
O=gpurun_out/$R
mkdir -p $O
if [ "$MODE" = ll ]; then
    python bench.py > $O/bench.json 2> $O/bench.err
    CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-context"
    $CMD > $O/plain_ll.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_ll.log 2>&1
else
    CMD2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-context"
    $CMD2 > $O/plain_full.log 2>&1 && \
    ncu --set full --import-source on --clock-control none \
        -k regex:"k_compat|k_sc2|k_score|k_pgs|k_degree|k_expand|k_hist|k_collect" -c 11 \
        -o $O/prof_full -f $CMD2 > $O/ncu_full.log 2>&1
fi
