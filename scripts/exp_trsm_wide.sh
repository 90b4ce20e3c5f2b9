#!/bin/bash
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 300 python scripts/trsm_wide_probe.py > $O/${T}_trsm_wide.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:trsm_unit \
  --log-file $O/${T}_trsm_wide_launches.csv python scripts/trsm_wide_probe.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_lu.py tests/test_gpu_hpl2d.py -q -x -p no:cacheprovider > $O/${T}_tests.log 2>&1
bash scripts/exp_ab32k.sh $T "OZ_X=1"
echo "== $(timeout 300 python scripts/panel_breakdown.py 16384 1024 7 2>&1 | head -1)" >> $O/${T}_ab.log
