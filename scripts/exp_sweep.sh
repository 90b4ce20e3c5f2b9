#!/bin/bash
# interleaved A/B of many settings at n=32768 (2 reps each) + n=16384 once
T=${1:-x}; shift; O=gpurun_out
for rep in 1 2; do
  for envs in "$@"; do
    echo "== $envs rep=$rep $(env $envs timeout 200 python scripts/panel_breakdown.py 32768 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
  done
done
for envs in "$@"; do
  echo "== $envs $(env $envs timeout 200 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
done
