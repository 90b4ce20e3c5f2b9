#!/bin/bash
# Round bench + evidence: default bench line, then the launch list of a
# one-step run of the same command under ncu (serialised, cold cache).
T=${1:-r02}; O=gpurun_out; mkdir -p $O
s0=$(date +%s); timeout 1500 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo rc=$? wall_s=$(( $(date +%s) - s0 )) >> $O/${T}_bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file $O/${T}_launches.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 \
  --skip-native --sweep-k "" --size-sweep "" > $O/${T}_launches_bench.log 2>&1
python scripts/launch_summary.py $O/${T}_launches.csv > $O/${T}_launches.txt 2>&1
