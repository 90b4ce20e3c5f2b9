#!/bin/bash
# ncu --set full of one grid register-leaf launch: 64-column/256-row (m=12288 on 100 SMs)
# and the tall 16-column/1024-row variant (m=20480 on 20 SMs)
T=${1:-x}; O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_leaf_kernel -s 4 -c 1 \
  -o $O/${T}_leaf64 python scripts/panel_probe.py 12288 100 1024 > $O/${T}_leaf64.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:panel_leaf_kernel -s 4 -c 1 \
  -o $O/${T}_leaf16 python scripts/panel_probe.py 20480 20 1024 > $O/${T}_leaf16.log 2>&1
