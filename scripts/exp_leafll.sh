#!/bin/bash
# grid register leaf with tagged-word (LL) records: tests, standalone panels, LU
T=${1:-x}; shift; O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_panel_leaf.py tests/test_gpu_lu.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
timeout 300 python scripts/panel_probe.py 12288,16384,30720 32,100 1024 > $O/${T}_probe.log 2>&1
OZ_PANEL_TIMING=1 timeout 300 python scripts/panel_probe.py 16384 32 1024 > $O/${T}_probe_timing.log 2>&1
bash scripts/exp_ab32k.sh $T "OZ_X=1"
echo "== $(timeout 300 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
