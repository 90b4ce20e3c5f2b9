#!/bin/bash
# leaf tuning loop: A/B bits, panel timing, one ncu capture of the register leaf
T=${1:-x}; O=gpurun_out; mkdir -p $O
for cfg in "300 64" "4096 1024" "1000 256" "8000 512"; do
  timeout 120 python scripts/leaf_ab.py $cfg >> $O/${T}_leaf_ab.log 2>&1
done
timeout 300 python scripts/panel_probe.py 2048,4096,8192,16384 32,148 1024 > $O/${T}_panel_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_leaf -s 5 -c 1 -o $O/${T}_leaf python scripts/panel_probe.py 2048 148 1024 > $O/${T}_ncu.log 2>&1
ncu -i $O/${T}_leaf.ncu-rep --page source --csv > $O/${T}_leaf_src.csv 2>/dev/null
