#!/bin/bash
# LU k-sweep at n=16384 and n=32768 k=7 under env settings (A/B)
T=${1:-x}; shift; O=gpurun_out
for envs in "$@"; do
  for k in 3 5 7 9; do echo "== $envs k=$k $(env $envs timeout 200 python scripts/panel_breakdown.py 16384 1024 $k 2>&1 | head -1)" >> $O/${T}_ks.log; done
  echo "== $envs $(env $envs timeout 200 python scripts/panel_breakdown.py 32768 1024 7 2>&1 | head -1)" >> $O/${T}_ks.log
done
