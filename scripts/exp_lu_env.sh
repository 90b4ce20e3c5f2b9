#!/bin/bash
# LU factor time at the bench sizes under a list of env settings (A/B tuning)
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
for envs in "$@"; do
  for n in 8192 16384 32768; do
    echo "== $envs n=$n" >> $O/${T}_env.log
    env $envs timeout 300 python scripts/panel_breakdown.py $n 1024 7 2>&1 | head -1 >> $O/${T}_env.log
  done
done
