#!/usr/bin/env bash
# ncu evidence for the headline config (run under gpurun; one GPU):
#  1. the launch list of one cfg5 mm_layout (every launch with its device time:
#     kernel shares of the step; cold-cache and serialised, so shares, not absolutes)
#  2. --set full of kernel (c), (a) and (d) at the FINEST level: the finest level
#     runs last, so the LAST launch of each kernel in one layout is the finest
#     level's last sweep (skip = launches of the kernel in one layout - 1)
# Usage: bash tools/profile_round.sh r02 cfg5 15
set -e
tag=${1:-r02}; cfg=${2:-cfg5}; K=${3:-15}
out=gpurun_out
python tools/layout_once.py "$cfg" --count > "$out/${tag}_counts_${cfg}.json"
cnt() { python -c "import json;print(json.load(open('$out/${tag}_counts_${cfg}.json'))['$1'])"; }
nc=$(cnt repulse_coarse); ng=$(cnt gather_update); nd=$(cnt centroid)
python tools/layout_once.py "$cfg" > "$out/${tag}_plain_${cfg}.log" 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$out/${tag}_launches_${cfg}.csv" \
    python tools/layout_once.py "$cfg" > "$out/${tag}_ncu_launches_${cfg}.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_repulse$' -s $((nc - 1)) -c 1 \
    -o "$out/prof_${tag}_repulse_coarse_${cfg}" python tools/layout_once.py "$cfg" > "$out/${tag}_ncu_c.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_gather$' -s $((ng - 1)) -c 1 \
    -o "$out/prof_${tag}_gather_${cfg}" python tools/layout_once.py "$cfg" > "$out/${tag}_ncu_a.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_centroid$' -s $((nd - 1)) -c 1 \
    -o "$out/prof_${tag}_centroid_${cfg}" python tools/layout_once.py "$cfg" > "$out/${tag}_ncu_d.log" 2>&1
echo done
