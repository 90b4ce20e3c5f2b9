#!/bin/bash
O=gpurun_out; mkdir -p $O
for cfg in "64 64" "300 64" "1000 64" "4096 64" "4096 1024" "2048 1024" "1000 256"; do
  timeout 120 python scripts/leaf_ab.py $cfg >> $O/r02f_leaf_ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_lu.py -q -x -p no:cacheprovider > $O/r02f_gpu_lu.log 2>&1; echo rc=$? >> $O/r02f_gpu_lu.log
timeout 300 python scripts/panel_probe.py 2048,4096,8192,16384 32,148 1024 > $O/r02f_panel_probe.log 2>&1
OZ_PANEL_LEAF=0 timeout 300 python scripts/panel_probe.py 2048,4096,8192,16384 32,148 1024 > $O/r02f_panel_probe_old.log 2>&1
timeout 300 python scripts/probe.py lu 16384 1024 > $O/r02f_lu.log 2>&1
