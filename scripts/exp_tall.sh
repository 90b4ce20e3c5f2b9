#!/bin/bash
# tall register leaf variants: tests, standalone tall panels, LU A/B
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_panel_leaf.py tests/test_gpu_lu.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
for e in OZ_PANEL_LEAF_TALL=1; do
  env $e timeout 300 python scripts/panel_probe.py 30720,24576,20480 16,20,28 1024 > $O/${T}_probe_${e#*=}.log 2>&1
done
bash scripts/exp_ab32k.sh $T "$@"
for e in "$@"; do
  echo "== $e $(env $e timeout 300 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
done
