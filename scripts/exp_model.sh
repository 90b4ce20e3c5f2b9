#!/bin/bash
# LU trace with current defaults, then an A/B over look-ahead panel-model constants
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
OZ_LU_TRACE=1 timeout 300 python scripts/panel_breakdown.py 32768 1024 7 > $O/${T}_trace_32768.log 2>&1
bash scripts/exp_ab32k.sh $T "$@"
for e in "$@"; do
  echo "== $e $(env $e timeout 300 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
done
