#!/bin/bash
# serialised per-launch device times of one standalone panel (ncu launch list)
T=${1:-x}; O=gpurun_out; mkdir -p $O
for cfg in "2048 132" "8192 100" "12288 100"; do
  set -- $cfg
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${T}_panel_${1}_${2}.csv python scripts/panel_probe.py $1 $2 1024 > /dev/null 2>&1
done
