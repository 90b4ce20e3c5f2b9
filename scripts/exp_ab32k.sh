#!/bin/bash
# interleaved A/B of LU factor time at n=32768 k=7 (reps x settings)
T=${1:-x}; shift; O=gpurun_out
for rep in 1 2 3; do
  for envs in "$@"; do
    echo "== $envs rep=$rep $(env $envs timeout 200 python scripts/panel_breakdown.py 32768 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
  done
done
