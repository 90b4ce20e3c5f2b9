#!/bin/bash
O=gpurun_out; mkdir -p $O
./scripts/exch_mb > $O/r02i_exch.log 2>&1
for cfg in "300 64" "4096 1024" "2048 1024" "1000 256" "8000 512" "12000 256"; do
  timeout 120 python scripts/leaf_ab.py $cfg >> $O/r02i_leaf_ab.log 2>&1
done
timeout 300 python scripts/panel_probe.py 2048,4096,8192,16384 32,148 1024 > $O/r02i_panel_probe.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:panel_leaf -s 5 -c 1 -o $O/r02i_leaf python scripts/panel_probe.py 2048 148 1024 > $O/r02i_ncu.log 2>&1
