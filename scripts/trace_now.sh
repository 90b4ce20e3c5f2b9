#!/bin/bash
# per-step LU timelines (OZ_LU_TRACE) at the bench sizes, current defaults
T=${1:-x}; O=gpurun_out; mkdir -p $O
for n in 32768 16384; do
  OZ_LU_TRACE=1 timeout 300 python scripts/panel_breakdown.py $n 1024 7 > $O/${T}_trace_$n.log 2>&1
done
